"""Print device memory after each setup step of a config (diagnostics)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1807_10749_b200 import configs  # noqa: E402
from paper_1807_10749_b200.engine import ENGINES  # noqa: E402
from paper_1807_10749_b200.lowering import lowered  # noqa: E402
from paper_1807_10749_b200.plan import split_requests  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
free = lambda: round(torch.cuda.mem_get_info()[0] / 1e9, 2)
circ, plan, req, pre = configs.build(name)
print("after build", free())
eng = ENGINES.get(0, "c64")
print("after create", free())
eng.load_program(lowered(circ, plan.cut))
print("after load", free())
eng.set_requests(*split_requests(circ.n_qubits, plan.cut.block_a, plan.cut.block_b, req))
print("after requests", free())
eng.set_option("mem_budget_mb", 100000)
r = eng.run(plan.x_p, pre[:1], 0, plan.branch_space)
print("after run", free(), r.stats)

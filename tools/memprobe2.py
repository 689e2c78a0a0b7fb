"""Replicates bench.py's setup order and prints free device memory (diagnostics)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1807_10749_b200 import configs  # noqa: E402
from paper_1807_10749_b200.engine import ENGINES  # noqa: E402
from paper_1807_10749_b200.lowering import lowered  # noqa: E402
from paper_1807_10749_b200.plan import split_requests  # noqa: E402

free = lambda: round(torch.cuda.mem_get_info()[0] / 1e9, 2)
torch.cuda.set_device(0)
print("start", free())
circ, plan, req, pre = configs.build("cfg5")
eng = ENGINES.get(0, "c64")
eng.set_stream(torch.cuda.current_stream().cuda_stream)
eng.load_program(lowered(circ, plan.cut))
eng.set_requests(*split_requests(circ.n_qubits, plan.cut.block_a, plan.cut.block_b, req))
out = torch.zeros(2 * req.size, dtype=torch.float64, device="cuda:0")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda:0")
print("before run", free())
try:
    r = eng.run(plan.x_p, pre[:1], 0, plan.branch_space, out_device_ptr=out.data_ptr(), want_host=False)
    print("after run", free(), r.stats["ms_total"])
except Exception as e:
    print("ERR", e, free())

"""Wall vs device time per gs_run for a config (diagnostics)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_1807_10749_b200 import configs  # noqa: E402
from paper_1807_10749_b200.engine import ENGINES  # noqa: E402
from paper_1807_10749_b200.lowering import lowered  # noqa: E402
from paper_1807_10749_b200.plan import split_requests  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
circ, plan, req, pre = configs.build(name)
eng = ENGINES.get(0, "c64")
eng.load_program(lowered(circ, plan.cut))
eng.set_requests(*split_requests(circ.n_qubits, plan.cut.block_a, plan.cut.block_b, req))
for i in range(5):
    t = time.perf_counter()
    r = eng.run(plan.x_p, pre, 0, plan.branch_space)
    wall = (time.perf_counter() - t) * 1e3
    print(f"wall {wall:.3f} ms  device {r.stats['ms_total']:.3f} ms  launches {r.stats['n_launches']} nodes {r.stats['n_nodes']}")

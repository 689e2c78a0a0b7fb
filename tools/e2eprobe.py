"""Where the end-to-end run_batched time goes (diagnostics)."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_1807_10749_b200 import configs  # noqa: E402
from paper_1807_10749_b200.amplitudes import AmplitudeBatch  # noqa: E402
from paper_1807_10749_b200.engine import ENGINES  # noqa: E402
from paper_1807_10749_b200.lowering import lowered  # noqa: E402
from paper_1807_10749_b200.pathsum import run_batched  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
window = int(sys.argv[2]) if len(sys.argv) > 2 else 32
circ, plan, req, pre = configs.build(name)
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    ENGINES.get(0, "c64").set_option(k, int(v))
for s in range(3):
    run_batched(circ, plan, req, prefixes=pre[s * window:(s + 1) * window])
T = {}


def tick(k, t0):
    T.setdefault(k, []).append((time.perf_counter() - t0) * 1e3)
    return time.perf_counter()


for s in range(3, 23):
    w = pre[s * window:(s + 1) * window]
    t_all = t = time.perf_counter()
    prog = lowered(circ, plan.cut)
    idx = np.asarray(req, dtype=np.int64).ravel()
    eng = ENGINES.get(0, "c64")
    eng.load_program(prog)
    t = tick("prep", t)
    eng.set_requests_global(idx, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
    t = tick("set_requests_global", t)
    out = AmplitudeBatch.zeros(idx)
    t = tick("zeros", t)
    r = eng.run(plan.x_p, w, 0, plan.branch_space, out=out.amps)
    t = tick("run", t)
    T.setdefault("run.device", []).append(r.stats["ms_total"])
    T.setdefault("run.enqueue", []).append(r.stats["host_ms_enqueue"])
    tick("total", t_all)
    t = time.perf_counter()
    run_batched(circ, plan, req, prefixes=w)
    tick("run_batched", t)
for k, v in T.items():
    print(f"{k:22s} median {np.median(v):8.3f} ms  max {np.max(v):8.3f}")

"""Time the GPU full-state engine (statevec.run_full) on the config circuits.

    python tools/fullprobe.py [cfg2 cfg3 ...]

Prints the device time of gs_run_full (passes + scale, CUDA events inside the
library), the number of passes and the achieved pass bandwidth (one read + one
write of the 2^n-amplitude state per pass)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1807_10749_b200 import configs  # noqa: E402
from paper_1807_10749_b200.engine import ENGINES  # noqa: E402
from paper_1807_10749_b200.lowering import lowered  # noqa: E402
from paper_1807_10749_b200.statevec import full_cut  # noqa: E402

for name in sys.argv[1:] or ["cfg2"]:
    circ, _, _, _ = configs.build(name, n_req=4)
    n = circ.n_qubits
    if n > 31:
        print(name, "skipped:", n, "qubits")
        continue
    eng = ENGINES.get(0, "c64")
    eng.load_program(lowered(circ, full_cut(circ)))
    eng.run_full()  # warm-up (JIT, buffers)
    best = None
    for _ in range(5):
        t = time.perf_counter()
        r = eng.run_full()
        wall = time.perf_counter() - t
        st = r.stats
        if best is None or st["ms_total"] < best[0]["ms_total"]:
            best = (st, wall)
    st, wall = best
    passes = st["n_pass_launches"]
    gbs = passes * 16.0 * (1 << n) / (st["ms_total"] / 1e3) / 1e9
    print(f"{name}: {n} qubits, {len(circ.gates)} gates, {passes} passes, device {st['ms_total']:.3f} ms "
          f"({gbs:.0f} GB/s over passes), with the 2^{n} download {wall * 1e3:.1f} ms")

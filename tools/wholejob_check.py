"""Whole-job cross-check of the leaf forms (cfg4: all 335,544 retained prefixes x 8 branches,
10^6 bitstrings): the default (Pauli-sibling fused pass) twice -- bitwise equal -- against
the 8-slot fused pass (pf_pauli=0) and the separate leaf passes + projected gather
(proj_fuse=0).  Prints relative L2 differences as one JSON line.

    python tools/wholejob_check.py [cfg4]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1807_10749_b200 import configs  # noqa: E402
from paper_1807_10749_b200.engine import ENGINES  # noqa: E402
from paper_1807_10749_b200.lowering import lowered  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
circ, plan, req, pre = configs.build(name)
eng = ENGINES.get(0, "c64")
out, secs = {}, {}
for key, opts in (("pauli", {}), ("pauli_again", {}), ("slots", {"pf_pauli": 0}), ("separate", {"proj_fuse": 0})):
    for k, v in opts.items():
        eng.set_option(k, v)
    eng.load_program(lowered(circ, plan.cut))
    eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
    t = time.perf_counter()
    out[key] = eng.run(plan.x_p, plan.retained, 0, plan.branch_space).amps
    secs[key] = time.perf_counter() - t
    for k in opts:
        eng.set_option(k, 1)


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


print(json.dumps({
    "config": name, "paths": int(len(plan.retained) * plan.branch_space), "requests": int(len(req)),
    "seconds": {k: round(v, 2) for k, v in secs.items()},
    "bitwise_repeat": bool(np.array_equal(out["pauli"], out["pauli_again"])),
    "relL2_pauli_vs_slots": rel(out["pauli"], out["slots"]),
    "relL2_pauli_vs_separate": rel(out["pauli"], out["separate"]),
    "relL2_slots_vs_separate": rel(out["slots"], out["separate"]),
    "sum_abs2": float(np.sum(np.abs(out["pauli"]) ** 2)),
}))

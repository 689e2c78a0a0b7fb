import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long CPU oracle runs")


def load_amps(case):
    path = os.path.join(GOLDEN, "amps", f"{case}.npz")
    if not os.path.exists(path):
        # every fixture is committed: a missing one is a broken checkout, not a reason to skip parity
        pytest.fail(f"golden fixture tests/golden/amps/{case}.npz is missing (tests/golden/make_golden.py writes it)")
    with np.load(path, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def plans_golden():
    with open(os.path.join(GOLDEN, "plans.json")) as fh:
        return json.load(fh)


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    den = float(np.linalg.norm(b))
    return float(np.linalg.norm(a - b)) / (den if den > 0 else 1.0)


def small_case(case):
    """(circuit, plan, requests, golden dict) for a tests/golden/amps small case."""
    from paper_1807_10749_b200 import Cut, make_plan, parse_circuit

    g = load_amps(case)
    text = str(g["text"])
    n = int(text.split("\n", 1)[0])
    circ = parse_circuit(text)
    cut = None
    if "cut" in g and g["cut"].size:
        a = tuple(int(v) for v in g["cut"])
        b = tuple(q for q in range(n) if q not in a)
        cut = Cut("s", 0, a, b)
    plan = make_plan(circ, fidelity=1.0, cut=cut, x_p=int(g["x_p"]), x_b=int(g["x_b"]))
    return circ, plan, g["requests"], g

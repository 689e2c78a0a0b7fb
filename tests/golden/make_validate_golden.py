"""Golden verifier rounds from the reference.

Build container only (imports the read-only reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_validate_golden.py

Writes tests/golden/validate.json: the reference test's circuits (2x7, depth
24, v2 rules, seeds 3 and 4 -- ``test_validate.py:23-36``) as serialized
text, the verifier cut, the calibrated delta, and the reference's round
results (f_e, f1_realized, passed) for the honest / random / under-fidelity
claimants at the seeds its tests use.
"""
from __future__ import annotations

import json
import os
import sys

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from gridsim.benchgen import GenSpec, generate  # noqa: E402
from gridsim.circuit import serialize_circuit  # noqa: E402
from gridsim.validate import (  # noqa: E402
    calibrate_delta, claimant_round, issue_challenge, verifier_cut, verifier_round,
)

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    circ = generate(GenSpec(2, 7, 24, "v2", seed=3))
    other = generate(GenSpec(2, 7, 24, "v2", seed=4))
    vcut = verifier_cut(circ)
    delta = calibrate_delta(circ, k=2048, rounds=6, seed=5, cut=vcut)
    rounds = []
    for engine, seed, f1, fid, cseed, path_seed in (
        ("exact", 21, 0.15, 1.0, 0, 91),
        ("random", 22, 0.15, 1.0, 8, 92),
        ("hybrid", 23, 0.2, 0.01, 9, 93),
        ("hybrid", 24, 0.2, 0.3, 10, 94),
    ):
        ch = issue_challenge(circ, k=2048, delta=delta, seed=seed, f1=f1)
        resp = claimant_round(circ, ch, engine=engine, fidelity=fid, seed=cseed)
        res = verifier_round(circ, ch, resp, path_seed=path_seed, cut=vcut)
        rounds.append({"engine": engine, "seed": seed, "f1": f1, "fidelity": fid, "claimant_seed": cseed,
                       "path_seed": path_seed, "f_e": res.f_e, "f1_realized": res.f1_realized,
                       "passed": res.passed})
    out = {
        "circuit": serialize_circuit(circ),
        "other": serialize_circuit(other),
        "verifier_cut": {"orientation": vcut.orientation, "position": vcut.position,
                         "a": list(vcut.block_a), "b": list(vcut.block_b)},
        "delta": delta,
        "rounds": rounds,
    }
    with open(os.path.join(HERE, "validate.json"), "w") as fh:
        json.dump(out, fh, indent=1)
        fh.write("\n")
    print(json.dumps({"delta": delta, "rounds": rounds}, indent=1))


if __name__ == "__main__":
    main()

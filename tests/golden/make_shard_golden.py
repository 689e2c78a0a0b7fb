"""Shard-file fixtures from the reference orchestrator (run in the build container).

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_shard_golden.py

Writes tests/golden/shard_hashes.json (reference plan_hash / request_hash /
job filenames for cfg1 and cfg3 with 1,024 challenge requests) and
tests/golden/shards/cfg1/: the shard files the reference's own worker writes
for cfg1's first four prefixes (orchestrator._worker via run_campaign-free
direct call), so the GPU side can be checked to read, merge and resume them.
"""
import json
import os
import shutil
import sys

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import gridsim.orchestrator as orch  # noqa: E402
import gridsim.pathsum as ps  # noqa: E402
from gridsim.benchgen import GenSpec, generate  # noqa: E402
from gridsim.validate import challenge_indices  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = {"cfg1": (4, 4, 16, "v1", 1.0), "cfg3": (6, 6, 28, "v1", 0.1)}
N_REQ = 1024


def main():
    out = {}
    for name, (r, c, d, ver, f) in CASES.items():
        circ = generate(GenSpec(r, c, d, ver, include_final_h=True, seed=0))
        plan = ps.make_plan(circ, fidelity=f, seed=0, workers=1)
        req = challenge_indices(circ.n_qubits, N_REQ, 12345)
        jobs = orch.shard(circ, plan, req)
        out[name] = {
            "n_req": N_REQ,
            "plan_hash": orch.plan_hash(circ, plan, req),
            "request_hash": orch.request_hash(req),
            "filenames_head": [j.filename for j in jobs[:8]],
            "n_jobs": len(jobs),
        }
        if name == "cfg1":
            d_out = os.path.join(HERE, "shards", "cfg1")
            shutil.rmtree(d_out, ignore_errors=True)
            os.makedirs(d_out)
            orch._worker(circ, plan, req, jobs[:4], {j.prefix: 0 for j in jobs}, d_out, {})
    with open(os.path.join(HERE, "shard_hashes.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1)[:800])


if __name__ == "__main__":
    main()

"""Campaign shard files: the reference's file names, hashes,
header and verified merge, so GPU jobs and reference CPU workers share one
shard directory.  Pinned against tests/golden/shard_hashes.json and the shard
files the reference's own worker wrote (tests/golden/make_shard_golden.py).
"""
import json
import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN, load_amps, rel_l2
from paper_1807_10749_b200 import configs
from paper_1807_10749_b200.amplitudes import AmplitudeBatch, write_amplitudes
from paper_1807_10749_b200.shards import (
    SHARD_DIGITS,
    MergeError,
    merge,
    plan_hash,
    request_hash,
    shard,
    status,
)

REF_SHARDS = os.path.join(GOLDEN, "shards", "cfg1")


def _golden():
    with open(os.path.join(GOLDEN, "shard_hashes.json")) as fh:
        return json.load(fh)


@pytest.mark.parametrize("name", ["cfg1", "cfg3"])
def test_hashes_and_names_match_reference(name):
    g = _golden()[name]
    circ, plan, req, _ = configs.build(name, n_req=g["n_req"])
    assert request_hash(req) == g["request_hash"]
    assert plan_hash(circ, plan, req) == g["plan_hash"]
    jobs = shard(circ, plan, req)
    assert len(jobs) == g["n_jobs"]
    assert [j.filename for j in jobs[:8]] == g["filenames_head"]


def _cpu_job(circ, plan, req, job, d):
    """A CPU worker (the oracle standing in for the reference's) writing one shard."""
    from oracle import pathsum_oracle as oracle

    amps = oracle.run_batched(circ, plan, req, np.array([job.prefix]))
    header = {"plan": job.plan_hash, "circuit": job.circuit_hash, "requests": job.request_hash,
              "prefix": str(job.prefix), "attempt": "1", "seconds": "0.0"}
    write_amplitudes(os.path.join(d, job.filename), AmplitudeBatch(req, amps), digits=SHARD_DIGITS, header=header)


def test_merge_reference_and_cpu_shards(tmp_path):
    circ, plan, req, _ = configs.build("cfg1", n_req=1024)
    d = str(tmp_path)
    for f in os.listdir(REF_SHARDS):
        shutil.copy(os.path.join(REF_SHARDS, f), d)
    st = status(circ, plan, req, d)
    assert len(st.done) == 4 and len(st.pending) == 12 and not st.complete
    with pytest.raises(MergeError):
        merge(circ, plan, req, d)  # missing shards
    jobs = shard(circ, plan, req)
    for job in jobs[4:]:
        _cpu_job(circ, plan, req, job, d)
    assert status(circ, plan, req, d).complete
    total = merge(circ, plan, req, d)
    want = load_amps("cfg1")
    assert np.array_equal(total.indices, want["requests"])
    assert rel_l2(total.amps, want["amps_c64"]) <= 1e-6
    # a duplicate (renamed copy) and a foreign-request shard are refused
    src = os.path.join(d, jobs[0].filename)
    shutil.copy(src, os.path.join(d, "zz_copy.amp"))
    with pytest.raises(MergeError):
        merge(circ, plan, req, d)
    os.remove(os.path.join(d, "zz_copy.amp"))
    other = req.copy()
    other[0] ^= 1
    write_amplitudes(os.path.join(d, jobs[1].filename), AmplitudeBatch(other, np.zeros(other.size)),
                     digits=SHARD_DIGITS, header={"plan": jobs[1].plan_hash, "circuit": jobs[1].circuit_hash,
                                                  "requests": jobs[1].request_hash, "prefix": "1"})
    with pytest.raises(MergeError):
        merge(circ, plan, req, d)


@pytest.mark.gpu
def test_gpu_jobs_resume_a_reference_campaign(tmp_path):
    """GPU jobs fill the shards the reference's worker has not written; the merge
    equals the reference's run_approx; a second call writes nothing."""
    from paper_1807_10749_b200.pathsum import run_approx
    from paper_1807_10749_b200.shards import run_shard_jobs

    circ, plan, req, _ = configs.build("cfg1", n_req=1024)
    d = str(tmp_path)
    for f in os.listdir(REF_SHARDS):
        shutil.copy(os.path.join(REF_SHARDS, f), d)
    written = run_shard_jobs(circ, plan, req, d)
    assert sorted(written) == sorted(int(p) for p in plan.retained[4:])
    assert run_shard_jobs(circ, plan, req, d) == []
    total = merge(circ, plan, req, d)
    assert rel_l2(total.amps, load_amps("cfg1")["amps_c64"]) <= 1e-5
    assert rel_l2(total.amps, run_approx(circ, plan, req).amps) <= 1e-5

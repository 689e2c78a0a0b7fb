"""Campaign shard files written by GPU jobs.

The reference coordinates a truncated path sum as one job per retained
prefix whose result is a text shard file (``gridsim/orchestrator.py``:
``plan_hash`` / ``request_hash`` / ``ShardJob`` ``:44-85``, the worker
``:133-159``, ``status`` ``:126-130``, the verified merge ``:291-343``).
Those names, hashes, the scan and the merge are the reference's own and are
re-exported from ``gridsim.orchestrator`` unchanged.  What this module adds
is the GPU worker:

* :func:`run_shard_jobs` evaluates every pending job of a campaign (file
  absent or not matching the campaign) on the B200 -- one prefix, all its
  branches, through one loaded program and one device request split -- and
  commits each shard by atomic rename with the reference worker's header
  keys and 17-digit format, so GPU jobs and the reference's CPU workers fill
  one shard directory and an interrupted campaign resumes on either side.

Our circuits are converted to ``gridsim`` circuits through the shared text
format (identical ``circuit_hash``).  Needs ``gridsim`` importable (or
installed under ``baseline/_ref``).  The coordinator (retry rounds, forked
workers) stays the reference's and out of scope here.
"""
from __future__ import annotations

import os
import time

import numpy as np

from .gridsim_engine import load_gridsim, to_gridsim

_orch = load_gridsim("orchestrator")
_sv = load_gridsim("statevec")

SHARD_DIGITS = _orch.SHARD_DIGITS
CampaignError = _orch.CampaignError
MergeError = _orch.MergeError
CampaignStatus = _orch.CampaignStatus
ShardJob = _orch.ShardJob
request_hash = _orch.request_hash


def plan_hash(circuit, plan, requests) -> str:
    return _orch.plan_hash(to_gridsim(circuit), plan, requests)


def shard(circuit, plan, requests) -> list:
    return _orch.shard(to_gridsim(circuit), plan, requests)


def status(circuit, plan, requests, shard_dir: str):
    return _orch.status(to_gridsim(circuit), plan, requests, shard_dir)


def merge(circuit, plan, requests, shard_dir: str):
    return _orch.merge(to_gridsim(circuit), plan, requests, shard_dir)


def _committed(shard_dir: str, job, req: np.ndarray) -> bool:
    """True when ``job``'s file exists, parses and matches the campaign (the
    reference's notion of a finished job, ``orchestrator.py:88-103``)."""
    try:
        batch, header = _sv.read_amplitudes(os.path.join(shard_dir, job.filename))
    except (OSError, ValueError):
        return False
    want = {"plan": job.plan_hash, "circuit": job.circuit_hash, "requests": job.request_hash,
            "prefix": str(job.prefix)}
    return all(header.get(k) == v for k, v in want.items()) and np.array_equal(batch.indices, req)


def run_shard_jobs(circuit, plan, requests, shard_dir: str, prefixes=None, device: int = 0,
                   dtype="c64") -> list:
    """GPU worker: evaluate and commit every pending job (optionally only ``prefixes``).

    Returns the prefixes written.  Valid files already present are left alone,
    so calling it again after an interruption resumes the campaign.
    """
    os.makedirs(shard_dir, exist_ok=True)
    req = np.asarray(requests, dtype=np.int64)
    jobs = shard(circuit, plan, req)
    if prefixes is not None:
        keep = {int(p) for p in prefixes}
        jobs = [j for j in jobs if j.prefix in keep]
    todo = [j for j in jobs if not _committed(shard_dir, j, req)]
    if not todo:
        return []
    from .engine import ENGINES

    eng = ENGINES.get(device, dtype)
    with eng.lock:
        return _run_jobs(circuit, plan, req, shard_dir, todo, device, dtype)


def _run_jobs(circuit, plan, req, shard_dir, todo, device, dtype):
    from .pathsum import _engine_for

    eng, idx = _engine_for(circuit, plan, req, device, dtype)
    done = []
    for job in todo:
        t0 = time.perf_counter()
        amps = eng.run(plan.x_p, [job.prefix], 0, plan.branch_space).amps
        header = {"plan": job.plan_hash, "circuit": job.circuit_hash,
                  "requests": job.request_hash, "prefix": str(job.prefix), "attempt": "1",
                  "seconds": f"{time.perf_counter() - t0:.6f}"}
        final = os.path.join(shard_dir, job.filename)
        tmp = f"{final}.tmp.{os.getpid()}"
        _sv.write_amplitudes(tmp, _sv.AmplitudeBatch(idx, amps), digits=SHARD_DIGITS,
                             header=header)
        os.replace(tmp, final)
        done.append(job.prefix)
    return done

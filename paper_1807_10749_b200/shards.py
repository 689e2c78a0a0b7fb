"""Campaign shard files written by GPU jobs.

The reference coordinates a truncated path sum as one job per retained
prefix whose result is a text shard file (``orchestrator.py:44-85`` names and
hashes, ``:133-159`` the worker, ``:315-356`` the verified merge; the file
format is ``write_amplitudes`` with 17 significant digits, ``statevec.py:
479-511``, ``orchestrator.py:28``).  This module produces and consumes the
same files, so GPU jobs and the reference's CPU workers can fill one shard
directory, and a campaign interrupted on either side resumes on the other:

* ``plan_hash`` / ``request_hash`` / ``ShardJob.filename`` are the
  reference's digests (pinned against reference-computed values in
  ``tests/golden/shard_hashes.json``);
* ``run_shard_jobs`` is the GPU worker: every pending job (file absent or not
  matching the campaign) is evaluated by the CUDA engine -- one prefix, all its
  branches -- and committed by atomic rename, with the reference's header keys;
* ``status`` and ``merge`` re-implement the reference's scan and verified
  fold (ascending prefix order, complex128), raising ``MergeError`` for
  missing, foreign, duplicated or inconsistent shards.

The coordinator (retry rounds, forked CPU workers, reports) stays out of
scope: it is control plane, not the path sum.
"""
from __future__ import annotations

import hashlib
import os
import time
from dataclasses import dataclass

import numpy as np

from .amplitudes import AmplitudeBatch, read_amplitudes, write_amplitudes
from .circuit import Circuit, circuit_hash
from .plan import SimPlan

SHARD_DIGITS = 17


class CampaignError(RuntimeError):
    def __init__(self, message: str, failed=()):
        super().__init__(message)
        self.failed = tuple(int(p) for p in failed)


class MergeError(CampaignError):
    pass


def request_hash(requests) -> str:
    """Order-sensitive digest of the requested basis indices (``orchestrator.py:44-47``)."""
    data = np.ascontiguousarray(requests, dtype=np.int64)
    return hashlib.sha256(data.tobytes()).hexdigest()[:16]


def plan_hash(circuit: Circuit, plan: SimPlan, requests) -> str:
    """Digest binding a campaign to circuit, plan and requests (``orchestrator.py:50-63``)."""
    parts = [
        circuit_hash(circuit),
        plan.cut.orientation,
        str(plan.cut.position),
        repr(float(plan.fidelity)),
        str(plan.x_p),
        str(plan.x_b),
        str(plan.seed),
        ",".join(str(r) for r in plan.radices),
        request_hash(requests),
    ]
    return hashlib.sha256("|".join(parts).encode()).hexdigest()[:16]


@dataclass(frozen=True)
class ShardJob:
    prefix: int
    plan_hash: str
    circuit_hash: str
    request_hash: str

    @property
    def filename(self) -> str:
        return f"{self.plan_hash}.{self.prefix:08x}.amp"


def shard(circuit: Circuit, plan: SimPlan, requests) -> list[ShardJob]:
    """One job per retained prefix (``orchestrator.py:80-85``)."""
    fp = plan_hash(circuit, plan, requests)
    ch = circuit_hash(circuit)
    rh = request_hash(requests)
    return [ShardJob(int(p), fp, ch, rh) for p in plan.retained]


def _header_ok(header: dict, job: ShardJob) -> bool:
    return (
        header.get("plan") == job.plan_hash
        and header.get("circuit") == job.circuit_hash
        and header.get("requests") == job.request_hash
        and header.get("prefix") == str(job.prefix)
    )


def shard_done(shard_dir: str, job: ShardJob, requests) -> bool:
    """A job is done iff its file parses, matches the hashes and the request list."""
    try:
        batch, header = read_amplitudes(os.path.join(shard_dir, job.filename))
    except (OSError, ValueError):
        return False
    return _header_ok(header, job) and np.array_equal(batch.indices, np.asarray(requests, dtype=np.int64))


@dataclass
class CampaignStatus:
    plan_hash: str
    total: int
    done: tuple
    pending: tuple

    @property
    def complete(self) -> bool:
        return not self.pending


def status(circuit: Circuit, plan: SimPlan, requests, shard_dir: str) -> CampaignStatus:
    jobs = shard(circuit, plan, requests)
    done, pending = [], []
    for job in jobs:
        (done if shard_done(shard_dir, job, requests) else pending).append(job.prefix)
    return CampaignStatus(jobs[0].plan_hash, len(jobs), tuple(done), tuple(pending))


def run_shard_jobs(circuit: Circuit, plan: SimPlan, requests, shard_dir: str, prefixes=None,
                   device: int = 0, dtype="c64") -> list:
    """GPU worker: evaluate and commit every pending job (optionally only ``prefixes``).

    Returns the prefixes written.  Valid files already present are left alone,
    so calling it again after an interruption resumes the campaign.
    """
    from .pathsum import _engine_for

    os.makedirs(shard_dir, exist_ok=True)
    req = np.asarray(requests, dtype=np.int64)
    jobs = shard(circuit, plan, req)
    if prefixes is not None:
        wanted = {int(p) for p in prefixes}
        jobs = [j for j in jobs if j.prefix in wanted]
    pending = [j for j in jobs if not shard_done(shard_dir, j, req)]
    if not pending:
        return []
    eng, idx = _engine_for(circuit, plan, req, device, dtype)
    written = []
    for job in pending:
        start = time.perf_counter()
        amps = eng.run(plan.x_p, [job.prefix], 0, plan.branch_space).amps
        seconds = time.perf_counter() - start
        header = {
            "plan": job.plan_hash,
            "circuit": job.circuit_hash,
            "requests": job.request_hash,
            "prefix": str(job.prefix),
            "attempt": "1",
            "seconds": f"{seconds:.6f}",
        }
        final = os.path.join(shard_dir, job.filename)
        tmp = f"{final}.tmp.{os.getpid()}"
        write_amplitudes(tmp, AmplitudeBatch(idx, amps), digits=SHARD_DIGITS, header=header)
        os.replace(tmp, final)
        written.append(job.prefix)
    return written


def merge(circuit: Circuit, plan: SimPlan, requests, shard_dir: str) -> AmplitudeBatch:
    """Verified fold of every shard of this campaign, ascending prefix order
    (``orchestrator.py:315-356``)."""
    jobs = shard(circuit, plan, requests)
    fp = jobs[0].plan_hash
    by_prefix = {job.prefix: job for job in jobs}
    req = np.asarray(requests, dtype=np.int64)
    found, amps = {}, {}
    for name in sorted(os.listdir(shard_dir)):
        if not name.endswith(".amp"):
            continue
        try:
            batch, header = read_amplitudes(os.path.join(shard_dir, name))
        except (OSError, ValueError) as exc:
            raise MergeError(f"unreadable shard file {name}: {exc}")
        if header.get("plan") != fp:
            continue  # another campaign sharing the directory
        try:
            prefix = int(header["prefix"])
        except (KeyError, ValueError):
            raise MergeError(f"shard file {name} lacks a readable prefix header")
        if prefix in found:
            raise MergeError(f"duplicate shard for prefix {prefix}: {found[prefix]} and {name}")
        job = by_prefix.get(prefix)
        if job is None:
            raise MergeError(f"shard file {name} claims prefix {prefix}, not in this plan")
        if not _header_ok(header, job):
            raise MergeError(f"shard file {name} does not match the campaign hashes")
        if not np.array_equal(batch.indices, req):
            raise MergeError(f"shard file {name} answers different request indices")
        found[prefix] = name
        amps[prefix] = batch.amps
    missing = sorted(p for p in by_prefix if p not in found)
    if missing:
        shown = ", ".join(str(p) for p in missing[:16])
        raise MergeError(f"{len(missing)} shards missing: prefixes {shown}", failed=missing)
    total = AmplitudeBatch.zeros(req)
    for prefix in sorted(found):
        total.amps += amps[prefix]
    return total

"""Parity at the benchmark's own scale (VERDICT r01 "missing" #3).

The committed config goldens cover a few prefixes x 4,096 requests.  Here the
CUDA path runs with its default options on the BASELINE request counts -- all
10^6 bitstrings of config 4, all 10^5 of config 3 -- so the device request
split, the request sort, the grouped/projected gathers and the reduction run at
full size, and is compared with the CPU oracle (a numpy restatement of the
reference ``run_batched``, ``pathsum.py:574-640``, bit-exact with the reference
on cfg4) computed in the same test over host worker processes.

The bench window itself (256 prefixes per step for cfg4) is checked through a
size-independent property: one call over the window equals the sum of calls
over a partition of it (linearity, ``orchestrator.py:340-342`` fold).
"""
import numpy as np
import pytest

from conftest import rel_l2
from paper_1807_10749_b200 import configs

pytestmark = pytest.mark.gpu

C64_TOL = 1e-5


@pytest.fixture(scope="module")
def ps():
    from paper_1807_10749_b200 import engine, pathsum

    if engine.device_count() < 1:
        pytest.fail("no CUDA device visible to libgridsim_b200.so")
    return pathsum


def _spread(retained, n_lead, n_spread, seed):
    """Leading contiguous prefixes (shared tree nodes, aligned sibling blocks)
    plus a seeded spread across the whole retained set (other digit values)."""
    rng = np.random.default_rng(seed)
    spread = rng.choice(np.arange(n_lead, retained.size), size=n_spread, replace=False)
    return np.concatenate([retained[:n_lead], retained[np.sort(spread)]])


@pytest.mark.parametrize("name,n_lead,n_spread", [("cfg4", 4, 4), ("cfg3", 8, 8)])
def test_full_request_set_vs_oracle(ps, name, n_lead, n_spread):
    from oracle import pathsum_oracle as oracle

    circ, plan, req, _ = configs.build(name)
    assert req.size == configs.CONFIGS[name].n_req
    pre = _spread(plan.retained, n_lead, n_spread, seed=7)
    got = ps.run_batched(circ, plan, req, prefixes=pre).amps
    want = oracle.run_batched_pool(circ, plan, req, pre)
    assert np.linalg.norm(want) > 0
    assert rel_l2(got, want) <= C64_TOL
    # same prefixes, default entry point, request order reversed: same per-request values
    rev = ps.run_batched(circ, plan, req[::-1], prefixes=pre).amps
    assert rel_l2(rev[::-1], got) <= 1e-12


@pytest.mark.parametrize("name,window,parts", [("cfg4", 256, 8), ("cfg3", 128, 4)])
def test_bench_window_linearity(ps, name, window, parts):
    """The bench's step (one run_batched over ``window`` prefixes, all requests)
    equals the sum of the runs over a contiguous partition of the window."""
    circ, plan, req, _ = configs.build(name)
    pre = plan.retained[:window]
    whole = ps.run_batched(circ, plan, req, prefixes=pre).amps
    split = sum(ps.run_batched(circ, plan, req, prefixes=p).amps for p in np.array_split(pre, parts))
    assert np.linalg.norm(whole) > 0
    assert rel_l2(whole, split) <= 1e-10

"""GPU parity: the CUDA path through the C ABI vs the reference's own outputs.

Bars (BASELINE.json north_star): complex64 within 1e-5 relative L2 of the
reference run_approx / run_batched / run_path; complex128 within 1e-10 of the
reference with DTYPE rebound to complex128; path enumeration and subset are
bit-exact (the plan is the reference's, tests/test_plan.py).
"""
import numpy as np
import pytest

from conftest import load_amps, rel_l2, small_case
from paper_1807_10749_b200 import configs, make_plan

pytestmark = pytest.mark.gpu

C64_TOL = 1e-5
C128_TOL = 1e-10
SMALL = ["s3x4v2", "s3x4v1", "s4x4v2", "stair3x4", "iswap2x3", "iswap3x3", "fsim3x4", "fsim2x4"]


@pytest.fixture(scope="module")
def ps():
    from paper_1807_10749_b200 import engine, pathsum

    if engine.device_count() < 1:
        pytest.fail("no CUDA device visible to libgridsim_b200.so")
    return pathsum


def _engine(dtype="c64"):
    from paper_1807_10749_b200.engine import ENGINES

    return ENGINES.get(0, dtype)


@pytest.fixture(params=[0, 5, 4])
def tile_bits(request):
    """0 = default tile; 5/4 force multi-pass schedules with out-of-tile diagonal ops."""
    eng64, eng128 = _engine("c64"), _engine("c128")
    for e in (eng64, eng128):
        e.set_option("tile_bits", request.param)
    yield request.param
    for e in (eng64, eng128):
        e.set_option("tile_bits", 0)


def test_cz2_known_answer(ps):
    circ, plan, idx, g = small_case("cz2")
    np.testing.assert_allclose(ps.run_approx(circ, plan, idx).amps, [0.5, 0.5, 0.5, -0.5], atol=1e-7)
    np.testing.assert_allclose(ps.run_prefix_tree(circ, plan, 0, idx).amps, g["path0"], atol=1e-7)
    np.testing.assert_allclose(ps.run_prefix_tree(circ, plan, 1, idx).amps, g["path1"], atol=1e-7)


@pytest.mark.parametrize("case", SMALL)
def test_small_cases(ps, case, tile_bits):
    circ, plan, idx, g = small_case(case)
    assert rel_l2(ps.run_approx(circ, plan, idx).amps, g["amps_c64"]) <= C64_TOL
    assert rel_l2(ps.run_approx(circ, plan, idx, dtype="c128").amps, g["amps_c128"]) <= C128_TOL
    for pid, want in zip(g["path_ids"], g["path_amps"]):
        assert rel_l2(ps.run_path(circ, plan, int(pid), idx).amps, want) <= C64_TOL


@pytest.mark.parametrize("name", ["cfg1", "cfg1v2"])
def test_cfg1(ps, name, tile_bits):
    g = load_amps(name)
    circ, plan, req, _ = configs.build(name)
    assert rel_l2(ps.run_approx(circ, plan, req).amps, g["amps_c64"]) <= C64_TOL
    assert rel_l2(ps.run_approx(circ, plan, req, dtype="c128").amps, g["amps_c128"]) <= C128_TOL
    assert rel_l2(ps.run_approx(circ, plan, req).amps, g["full_c64"]) <= C64_TOL
    for pid, want in zip(g["path_ids"], g["path_amps"]):
        assert rel_l2(ps.run_path(circ, plan, int(pid), req).amps, want) <= C64_TOL
    pq = make_plan(circ, fidelity=0.25, seed=5)
    assert rel_l2(ps.run_approx(circ, pq, req).amps, g["f025_amps"]) <= C64_TOL


@pytest.mark.parametrize("name", ["cfg2", "cfg2v2", "cfg2h", "cfg3", "cfg3v2", "cfg4"])
def test_config_windows(ps, name):
    g = load_amps(name)
    circ, plan, _, _ = configs.build(name, n_req=4)
    req = g["requests"]
    got = ps.run_batched(circ, plan, req, prefixes=g["prefixes"]).amps
    assert rel_l2(got, g["amps_c64"]) <= C64_TOL
    if "amps_c128" in g:
        got = ps.run_batched(circ, plan, req, prefixes=g["prefixes_c128"], dtype="c128").amps
        assert rel_l2(got, g["amps_c128"]) <= C128_TOL
    if "path_ids" in g:
        for pid, want in zip(g["path_ids"], g["path_amps"]):
            assert rel_l2(ps.run_path(circ, plan, int(pid), req).amps, want) <= C64_TOL


def test_split_invariance_and_order(ps):
    circ, plan, req, _ = configs.build("cfg1v2")
    base = ps.run_approx(circ, make_plan(circ, x_b=0), req).amps
    for x_p in (0, 2, 5, 8):
        got = ps.run_approx(circ, make_plan(circ, x_p=x_p), req).amps
        assert rel_l2(got, base) <= 1e-6
    fwd = ps.run_batched(circ, plan, req, prefixes=plan.retained).amps
    bwd = ps.run_batched(circ, plan, req, prefixes=plan.retained[::-1]).amps
    assert rel_l2(fwd, bwd) <= 1e-12


def test_linearity_and_duplicates(ps):
    """Sum over a prefix set = sum of the sums over a partition; duplicates count twice."""
    circ, plan, req, _ = configs.build("cfg2")
    pre = plan.retained[:512]
    whole = ps.run_batched(circ, plan, req, prefixes=pre).amps
    parts = sum(ps.run_batched(circ, plan, req, prefixes=p).amps for p in np.array_split(pre, 3))
    assert rel_l2(parts, whole) <= 1e-10
    dup = ps.run_batched(circ, plan, req, prefixes=np.concatenate([pre[:7], pre[:7]])).amps
    one = ps.run_batched(circ, plan, req, prefixes=pre[:7]).amps
    assert rel_l2(dup, 2 * one) <= 1e-12


def test_cfg2_full_job_is_exact_state(ps):
    """f = 1: all 262,144 paths of config 2 sum to the exact amplitudes."""
    g = load_amps("cfg2_full")
    circ, plan, req, _ = configs.build("cfg2")
    got = ps.run_approx(circ, plan, req).amps
    assert rel_l2(got, g["exact"]) <= C64_TOL


def test_errors(ps):
    circ, plan, req, _ = configs.build("cfg1")
    with pytest.raises(ValueError):
        ps.run_approx(circ, plan, req, engine="nope")
    with pytest.raises(IndexError):
        ps.run_approx(circ, plan, [1 << 16])
    with pytest.raises(ValueError):
        ps.run_batched(circ, plan, req, prefixes=[plan.prefix_space])
    with pytest.raises(ValueError):
        ps.run_path(circ, plan, plan.path_space, req)
    empty = ps.run_approx(circ, plan, np.array([], dtype=np.int64))
    assert empty.amps.shape == (0,)
    none = ps.run_batched(circ, plan, req, prefixes=np.array([], dtype=np.int64))
    assert np.all(none.amps == 0)


@pytest.mark.parametrize("name", ["cfg5", "cfg5f"])
def test_cfg5_full_size_c64_matches_c128(ps, name):
    """28|28 halves (2 GiB each): the complex64 specialised kernels agree with the
    complex128 kernels on the same leading path and branch set, and summing a
    prefix's branches equals the sum of its single paths (linearity)."""
    circ, plan, _, pre = configs.build(name, n_req=4)
    from paper_1807_10749_b200 import challenge_indices

    req = challenge_indices(circ.n_qubits, 2048, 12345)
    pid = int(pre[0]) * plan.branch_space
    p64 = ps.run_path(circ, plan, pid, req).amps
    p128 = ps.run_path(circ, plan, pid, req, dtype="c128").amps
    assert np.linalg.norm(p128) > 0
    assert rel_l2(p64, p128) <= C64_TOL
    nb = min(plan.branch_space, 4)
    singles = sum(ps.run_path(circ, plan, pid + b, req).amps for b in range(nb))
    if nb == plan.branch_space:
        tree = ps.run_prefix_tree(circ, plan, int(pre[0]), req).amps
        assert rel_l2(tree, singles) <= 1e-6


@pytest.mark.parametrize("name", ["cfg5", "cfg5f"])
def test_cfg5_reference_paths(ps, name):
    """Per-path parity with the reference at 28|28 (tests/golden/amps/<name>.npz,
    produced by the reference's run_path in the build container)."""
    g = load_amps(name)
    circ, plan, _, _ = configs.build(name, n_req=4)
    for pid, want in zip(g["path_ids"], g["path_amps"]):
        assert rel_l2(ps.run_path(circ, plan, int(pid), g["requests"]).amps, want) <= C64_TOL


@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg2h"])
def test_fused_leaf_gather_option(ps, name):
    """fuse_gather=1 (gather inside the last B-side leaf pass) gives the same sums."""
    g = load_amps(name)
    circ, plan, _, _ = configs.build(name, n_req=4)
    eng = _engine("c64")
    eng.set_option("fuse_gather", 1)
    try:
        got = ps.run_batched(circ, plan, g["requests"], prefixes=g["prefixes"]).amps
    finally:
        eng.set_option("fuse_gather", 0)
    assert rel_l2(got, g["amps_c64"]) <= C64_TOL


def test_async_run_stream_order(ps):
    """async_run=1: back-to-back runs into a device buffer, read after one sync,
    equal the synchronous results (staging ring reuse across queued runs)."""
    import torch

    from paper_1807_10749_b200.lowering import lowered

    circ, plan, req, pre = configs.build("cfg3", n_req=64)
    eng = _engine("c64")
    eng.load_program(lowered(circ, plan.cut))
    eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
    wins = [pre[i * 96:(i + 1) * 96] for i in range(6)]
    want = [ps.run_batched(circ, plan, req, prefixes=w).amps for w in wins]
    eng.load_program(lowered(circ, plan.cut))
    eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
    outs = [torch.zeros(2 * req.size, dtype=torch.float64, device="cuda:0") for _ in wins]
    stream = torch.cuda.Stream()
    eng.set_stream(stream.cuda_stream)
    eng.set_option("async_run", 1)
    try:
        for w, o in zip(wins, outs):
            eng.run(plan.x_p, w, 0, plan.branch_space, out_device_ptr=o.data_ptr(), want_host=False)
        stream.synchronize()
    finally:
        eng.set_option("async_run", 0)
        eng.set_stream(None)
    for o, w in zip(outs, want):
        got = o.cpu().numpy().view(np.complex128)
        assert rel_l2(got, w) <= 1e-12


def test_run_batched_call_matches_two_calls(ps):
    """gs_run_batched (requests staged while the tree is enqueued) equals
    gs_set_requests_global + gs_run, and a bad index raises before output."""
    from paper_1807_10749_b200.lowering import lowered

    circ, plan, req, pre = configs.build("cfg3", n_req=4096)
    eng = _engine("c64")
    eng.load_program(lowered(circ, plan.cut))
    ba, bb = plan.cut.block_a, plan.cut.block_b
    one = eng.run_batched(req, circ.n_qubits, ba, bb, plan.x_p, pre[:64], 0, plan.branch_space).amps.copy()
    eng.set_requests_global(req, circ.n_qubits, ba, bb)
    two = eng.run(plan.x_p, pre[:64], 0, plan.branch_space).amps
    assert np.array_equal(one, two)
    bad = req.copy()
    bad[7] = -1
    with pytest.raises(IndexError):
        eng.run_batched(bad, circ.n_qubits, ba, bb, plan.x_p, pre[:64], 0, plan.branch_space)
    again = eng.run_batched(req, circ.n_qubits, ba, bb, plan.x_p, pre[:64], 0, plan.branch_space).amps
    assert np.array_equal(again, one)


def test_pipelined_result_download(ps):
    """d2h_chunk_mb > 0: chunked download through the pinned bounce buffer gives
    the same host result as the direct copy."""
    circ, plan, req, pre = configs.build("cfg3")
    eng = _engine("c64")
    want = ps.run_batched(circ, plan, req, prefixes=pre[:8]).amps
    eng.set_option("d2h_chunk_mb", 1)
    try:
        got = ps.run_batched(circ, plan, req, prefixes=pre[:8]).amps
    finally:
        eng.set_option("d2h_chunk_mb", 0)
    assert req.size * 16 > (1 << 20)  # more than one chunk
    assert np.array_equal(got, want)


@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg5"])
def test_sorted_request_gather_is_bitwise_equal(ps, name):
    """sort_requests=1 (the HBM gathers read requests sorted by A index, results
    folded back to request order) gives exactly the unsorted sums, through all
    three request-loading entry points."""
    from paper_1807_10749_b200.lowering import lowered
    from paper_1807_10749_b200.plan import split_requests

    circ, plan, req, pre = configs.build(name, n_req=20000)
    window = pre[:2] if name == "cfg5" else pre[:16]
    branch_hi = 2 if name == "cfg5" else plan.branch_space
    eng = _engine("c64")
    eng.load_program(lowered(circ, plan.cut))
    ba, bb = plan.cut.block_a, plan.cut.block_b
    outs = {}
    for srt in (0, 1):
        eng.set_option("sort_requests", srt)
        try:
            a = eng.run_batched(req, circ.n_qubits, ba, bb, plan.x_p, window, 0, branch_hi).amps.copy()
            eng.set_requests_global(req, circ.n_qubits, ba, bb)
            b = eng.run(plan.x_p, window, 0, branch_hi).amps
            ia, ib = split_requests(circ.n_qubits, ba, bb, req)
            eng.set_requests(ia, ib)
            c = eng.run(plan.x_p, window, 0, branch_hi).amps
        finally:
            eng.set_option("sort_requests", 1)
        assert np.array_equal(a, b) and np.array_equal(a, c)
        outs[srt] = a
    assert np.array_equal(outs[0], outs[1])
    assert np.abs(outs[1]).max() > 0


@pytest.mark.parametrize("name", ["cfg3", "cfg4"])
def test_quad_gather_matches_thread_per_request(ps, name):
    """quad_gather=1 (4 lanes per request in the grouped gather, fp64 partials
    joined by shuffles) agrees with one thread per request to fp64 rounding."""
    g = load_amps(name)
    circ, plan, _, _ = configs.build(name, n_req=4)
    eng = _engine("c64")
    got = {}
    for q in (0, 1):
        eng.set_option("quad_gather", q)
        try:
            got[q] = ps.run_batched(circ, plan, g["requests"], prefixes=g["prefixes"]).amps
        finally:
            eng.set_option("quad_gather", 1)
    assert rel_l2(got[1], got[0]) <= 1e-13
    assert rel_l2(got[1], g["amps_c64"]) <= C64_TOL


@pytest.mark.parametrize("name", ["cfg2h", "cfg3", "cfg4", "cfg5"])
def test_pipelined_pass_kernels_bitwise(ps, name):
    """pipeline=1 (persistent pass kernels prefetching the next tile with
    cp.async) runs the same arithmetic: bitwise equal sums."""
    from paper_1807_10749_b200.lowering import lowered

    circ, plan, req, pre = configs.build(name, n_req=4096)
    window = pre[:2] if name == "cfg5" else pre[:8]
    branch_hi = 2 if name == "cfg5" else plan.branch_space
    eng = _engine("c64")
    got = {}
    eng.set_option("proj_fuse", 0)  # the same leaf path both times (the fused pass is never pipelined)
    try:
        for pipe in (0, 1):
            eng.set_option("pipeline", pipe)
            try:
                eng.load_program(lowered(circ, plan.cut))
                eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
                got[pipe] = eng.run(plan.x_p, window, 0, branch_hi).amps
            finally:
                eng.set_option("pipeline", 0)
    finally:
        eng.set_option("proj_fuse", 1)
    assert np.array_equal(got[0], got[1])
    assert np.abs(got[1]).max() > 0


@pytest.mark.parametrize("name", ["cfg1", "cfg2h", "cfg3", "cfg4"])
def test_parent_dedupe_bitwise(ps, name):
    """dedupe_parent=1 (sibling slots load their shared parent tile once, via
    shared memory) computes bitwise the same sums as every slot loading it."""
    from paper_1807_10749_b200.lowering import lowered

    circ, plan, req, pre = configs.build(name, n_req=4096)
    eng = _engine("c64")
    got = {}
    for d in (0, 1):
        eng.set_option("dedupe_parent", d)
        try:
            eng.load_program(lowered(circ, plan.cut))
            eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
            # an odd branch range: sibling groups that do not share a parent too
            got[d] = (eng.run(plan.x_p, pre[:12], 0, plan.branch_space).amps,
                      eng.run(plan.x_p, pre[:5], 1, plan.branch_space - 1).amps)
        finally:
            eng.set_option("dedupe_parent", 1)
    for a, b in zip(got[0], got[1]):
        assert np.array_equal(a, b) and np.abs(a).max() > 0


@pytest.mark.parametrize("name", ["cfg5", "cfg5f"])
def test_tail_gather_matches_tail_pass(ps, name):
    """tail_gather=1 (the leaf's small last pass evaluated per request inside
    the gather, fp64) agrees with running that pass (fp32) to rounding."""
    from paper_1807_10749_b200.lowering import lowered

    circ, plan, req, pre = configs.build(name, n_req=4096)
    eng = _engine("c64")
    got = {}
    for t in (0, 1):
        eng.set_option("tail_gather", t)
        try:
            eng.load_program(lowered(circ, plan.cut))
            if t:
                assert sum(eng.describe()["tail"]) > 0
            eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
            got[t] = eng.run(plan.x_p, pre[:1], 0, 2).amps
        finally:
            eng.set_option("tail_gather", 1)
    assert rel_l2(got[1], got[0]) <= 1e-6


@pytest.mark.parametrize("case", SMALL)
def test_tail_gather_small_cases(ps, case):
    """Small circuits forced onto the path-major gather with 5-qubit tiles (multi-pass
    leaf levels, tails of 1-3 qubits incl. diagonal ops on outside bits) vs the reference."""
    circ, plan, req, g = small_case(case)
    eng = _engine("c64")
    opts = {"smem_gather": 0, "grouped_leaf": 0, "tile_bits": 5}
    try:
        for k, v in opts.items():
            eng.set_option(k, v)
        got = ps.run_approx(circ, plan, req).amps
    finally:
        eng.set_option("smem_gather", 1)
        eng.set_option("grouped_leaf", 1)
        eng.set_option("tile_bits", 0)
    assert rel_l2(got, g["amps_c64"]) <= C64_TOL


@pytest.mark.parametrize("name", ["cfg1", "cfg2h", "cfg3", "cfg4", "cfg5"])
def test_uniform_chunks_bitwise(ps, name):
    """uniform_chunks=1 (full fan-out chunks compute parent/digits from the slot)
    gives bitwise the node-table results, incl. partial branch ranges."""
    from paper_1807_10749_b200.lowering import lowered

    circ, plan, req, pre = configs.build(name, n_req=4096)
    window = pre[:2] if name == "cfg5" else pre[:9]
    eng = _engine("c64")
    got = {}
    for u in (0, 1):
        eng.set_option("uniform_chunks", u)
        try:
            eng.load_program(lowered(circ, plan.cut))
            eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
            got[u] = (eng.run(plan.x_p, window, 0, plan.branch_space).amps,
                      eng.run(plan.x_p, window, 1, plan.branch_space - 1).amps)
        finally:
            eng.set_option("uniform_chunks", 1)
    for a, b in zip(got[0], got[1]):
        assert np.array_equal(a, b) and np.abs(a).max() > 0


@pytest.mark.parametrize("name", ["cfg2h", "cfg3", "cfg4"])
def test_four_register_bit_passes(ps, name):
    """reg_bits=4 (512-thread CTAs, 16 amplitudes per thread, specialised too)
    matches the reference windows."""
    g = load_amps(name)
    circ, plan, _, _ = configs.build(name, n_req=4)
    eng = _engine("c64")
    eng.set_option("reg_bits", 4)
    eng.set_option("jit_min_blocks", 2)
    try:
        got = ps.run_batched(circ, plan, g["requests"], prefixes=g["prefixes"]).amps
    finally:
        eng.set_option("reg_bits", 6)
        eng.set_option("jit_min_blocks", 3)
    assert rel_l2(got, g["amps_c64"]) <= C64_TOL


@pytest.mark.parametrize("name", ["cfg4", "cfg4v2", "cfg3v2"])
def test_projected_leaf_side(ps, name):
    """proj_leaf=1: the projector-only leaf side (CZ cut, A side) is read from its
    parent state in the gather (no leaf pass); equal to running the leaf pass."""
    from paper_1807_10749_b200.lowering import lowered

    circ, plan, req, pre = configs.build(name, n_req=4096)
    eng = _engine("c64")
    got = {}
    for pj in (0, 1):
        eng.set_option("proj_leaf", pj)
        try:
            eng.load_program(lowered(circ, plan.cut))
            assert eng.describe()["proj_side"] == (0 if pj else -1)
            eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
            got[pj] = (eng.run(plan.x_p, pre[:9], 0, plan.branch_space).amps,
                       eng.run(plan.x_p, pre[:5], 1, plan.branch_space - 1).amps)
        finally:
            eng.set_option("proj_leaf", 1)
    for a, b in zip(got[0], got[1]):
        assert rel_l2(b, a) <= 1e-6 and np.abs(a).max() > 0


@pytest.mark.parametrize("name", ["cfg4", "cfg3v2"])
def test_projected_leaf_permuted_parents(ps, name):
    """proj_perm=1 (parents of the projected side stored with the sibling-run
    qubits at the lowest address bits) gives the default sums."""
    from paper_1807_10749_b200.lowering import lowered

    circ, plan, req, pre = configs.build(name, n_req=4096)
    eng = _engine("c64")
    got = {}
    for pm in (0, 1):
        eng.set_option("proj_perm", pm)
        try:
            eng.load_program(lowered(circ, plan.cut))
            if pm:
                assert eng.describe()["proj_swaps"] > 0
            eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
            got[pm] = eng.run(plan.x_p, pre[:17], 0, plan.branch_space).amps
        finally:
            eng.set_option("proj_perm", 0)
    assert rel_l2(got[1], got[0]) <= 1e-12 and np.abs(got[0]).max() > 0


@pytest.mark.parametrize("name", ["cfg4", "cfg3v2"])
def test_projected_leaf_linearity_and_duplicates(ps, name):
    """With the projected leaf side (cfg4 / cfg3v2 A side): partition linearity,
    duplicate prefixes counting twice (leaf weights), and agreement with the
    reference window."""
    circ, plan, req, _ = configs.build(name, n_req=8192)
    pre = plan.retained[:40]
    whole = ps.run_batched(circ, plan, req, prefixes=pre).amps
    parts = sum(ps.run_batched(circ, plan, req, prefixes=p).amps for p in np.array_split(pre, 3))
    assert rel_l2(parts, whole) <= 1e-10
    dup = ps.run_batched(circ, plan, req, prefixes=np.concatenate([pre[:5], pre[:5]])).amps
    one = ps.run_batched(circ, plan, req, prefixes=pre[:5]).amps
    assert rel_l2(dup, 2 * one) <= 1e-12
    g = load_amps(name)
    got = ps.run_batched(circ, plan, g["requests"], prefixes=g["prefixes"]).amps
    assert rel_l2(got, g["amps_c64"]) <= C64_TOL


def test_projected_leaf_side_complex128(ps):
    """The projected leaf side in complex128 mode (interpreted passes, fp64 parents):
    equal to running the leaf pass to fp64 rounding, and to complex64 within 1e-5."""
    from paper_1807_10749_b200.lowering import lowered

    circ, plan, req, pre = configs.build("cfg4", n_req=4096)
    eng = _engine("c128")
    got = {}
    for pj in (0, 1):
        eng.set_option("proj_leaf", pj)
        try:
            eng.load_program(lowered(circ, plan.cut))
            assert eng.describe()["proj_side"] == (0 if pj else -1)
            eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
            got[pj] = eng.run(plan.x_p, pre[:6], 0, plan.branch_space).amps
        finally:
            eng.set_option("proj_leaf", 1)
    assert rel_l2(got[1], got[0]) <= 1e-12 and np.abs(got[0]).max() > 0
    c64 = ps.run_batched(circ, plan, req, prefixes=pre[:6]).amps
    assert rel_l2(c64, got[1]) <= C64_TOL


@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg2h"])
def test_grouped_sibling_pair_stores(ps, name):
    """slot_store16=1 (leaf slot bit 0 in a register: two sibling leaves per
    16-byte store) writes the same leaves: bitwise equal sums."""
    from paper_1807_10749_b200.lowering import lowered

    circ, plan, req, pre = configs.build(name, n_req=4096)
    eng = _engine("c64")
    got = {}
    for v in (0, 1):
        eng.set_option("slot_store16", v)
        try:
            eng.load_program(lowered(circ, plan.cut))
            eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
            got[v] = (eng.run(plan.x_p, pre[:9], 0, plan.branch_space).amps,
                      eng.run(plan.x_p, pre[:5], 1, plan.branch_space - 1).amps)
        finally:
            eng.set_option("slot_store16", 0)
    for a, b in zip(got[0], got[1]):
        assert np.array_equal(a, b) and np.abs(a).max() > 0


def test_pinned_result_buffers(ps):
    """run_batched results live in reused page-locked buffers: a result stays
    valid (and distinct) while referenced, and released buffers are reused."""
    import gc

    from paper_1807_10749_b200 import engine

    circ, plan, req, pre = configs.build("cfg3", n_req=4096)
    a = ps.run_batched(circ, plan, req, prefixes=pre[:4]).amps
    a_copy = a.copy()
    b = ps.run_batched(circ, plan, req, prefixes=pre[4:8]).amps
    assert a.ctypes.data != b.ctypes.data
    assert np.array_equal(a, a_copy)  # not overwritten by the second call
    c = ps.run_batched(circ, plan, req, prefixes=pre[:4]).amps
    assert np.array_equal(c, a_copy)
    ptr = b.ctypes.data
    del b
    gc.collect()
    d = ps.run_batched(circ, plan, req, prefixes=pre[4:8]).amps
    assert d.ctypes.data == ptr  # the released block came back
    assert isinstance(d.base, engine._PinnedBlock)


@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg2h", "cfg5"])
def test_sunk_trailing_passes(ps, name):
    """sink_ops (a level's small trailing pass moved behind the next level's cross
    terms, where it commutes) reorders commuting ops only: equal sums."""
    from paper_1807_10749_b200.lowering import lowered

    circ, plan, req, pre = configs.build(name, n_req=4096)
    window = pre[:2] if name == "cfg5" else pre[:9]
    branch_hi = 2 if name == "cfg5" else plan.branch_space
    eng = _engine("c64")
    got = {}
    for v in (0, 12):
        eng.set_option("sink_ops", v)
        try:
            eng.load_program(lowered(circ, plan.cut))
            eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
            got[v] = eng.run(plan.x_p, window, 0, branch_hi).amps
        finally:
            eng.set_option("sink_ops", 12)
    assert rel_l2(got[12], got[0]) <= 1e-6 and np.abs(got[0]).max() > 0


@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg3v2"])
def test_overlapped_gathers_bitwise(ps, name):
    """overlap_gather=1 (each leaf chunk's gather on a second stream while the
    next chunk's leaf passes run; double-buffered leaves, partials, tables) gives
    bitwise the serial sums, including many small chunks and back-to-back runs."""
    from paper_1807_10749_b200.lowering import lowered

    circ, plan, req, pre = configs.build(name, n_req=4096)
    eng = _engine("c64")
    got = {}
    for v in (0, 1):
        eng.set_option("overlap_gather", v)
        eng.set_option("max_chunk", 24)  # many leaf chunks per run
        try:
            eng.load_program(lowered(circ, plan.cut))
            eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
            got[v] = [eng.run(plan.x_p, pre[k * 7:(k + 1) * 7], 0, plan.branch_space).amps for k in range(3)]
            got[v].append(eng.run(plan.x_p, pre[:5], 1, plan.branch_space - 1).amps)
        finally:
            eng.set_option("overlap_gather", 0)
            eng.set_option("max_chunk", 1 << 20)
    for a, b in zip(got[0], got[1]):
        assert np.array_equal(a, b) and np.abs(a).max() > 0


@pytest.mark.parametrize("name", ["cfg4", "cfg4v2", "cfg3v2"])
def test_fused_projected_leaf_pass(ps, name):
    """proj_fuse=1 (default): the grouped side's last leaf pass does the
    projected-side gather itself (no leaf state reaches HBM).  Equal to the
    separate leaf pass + projected gather (proj_fuse=0) to complex64 rounding of
    the projected amplitudes, for each epilogue unroll, partial last groups,
    branch sub-ranges and duplicate prefixes; and to the reference window."""
    from paper_1807_10749_b200.lowering import lowered

    circ, plan, req, pre = configs.build(name, n_req=20000)
    eng = _engine("c64")
    got = {}
    DEFAULTS = {"proj_fuse": 1, "pf_tail": 0, "pf_min_blocks": 3, "tile_major": 2, "pf_pauli": 1}
    try:
        # "fused" is the default: the Pauli-sibling form (one base state per leaf group, siblings read
        # as Pauli images); "slots" is the 8-slot form it replaces
        for key, opts in (("sep", {"proj_fuse": 0}), ("fused", {}), ("slots", {"pf_pauli": 0}),
                          ("tail", {"pf_tail": 1, "pf_pauli": 0}),
                          ("mb0", {"pf_min_blocks": 0}), ("tilemajor", {"tile_major": 1})):
            for k, v in opts.items():
                eng.set_option(k, v)
            eng.load_program(lowered(circ, plan.cut))
            assert eng.describe()["proj_fused"] == (0 if key == "sep" else 1)
            assert (eng.describe()["pauli"] is not None) == (key in ("fused", "mb0", "tilemajor"))
            eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
            got[key] = (eng.run(plan.x_p, pre[:9], 0, plan.branch_space).amps,
                        eng.run(plan.x_p, pre[:5], 1, plan.branch_space - 1).amps,
                        eng.run(plan.x_p, np.concatenate([pre[:3], pre[:3]]), 0, plan.branch_space).amps)
            for k in opts:
                eng.set_option(k, DEFAULTS[k])
    finally:
        for k, v in DEFAULTS.items():
            eng.set_option(k, v)
    for key in ("fused", "slots", "tail", "mb0", "tilemajor"):
        for a, b in zip(got["sep"], got[key]):
            assert np.abs(a).max() > 0
            assert rel_l2(b, a) <= 2e-6, key
    g = load_amps(name) if name != "cfg4v2" else None
    if g is not None:
        got = ps.run_batched(circ, plan, g["requests"], prefixes=g["prefixes"]).amps
        assert rel_l2(got, g["amps_c64"]) <= C64_TOL


@pytest.mark.parametrize("name", ["cfg3", "cfg4", "cfg5"])
def test_tile_major_cta_order_bitwise(ps, name):
    """tile_major (CTA launch order of the passes below the root) changes only which
    CTA runs when: bitwise equal sums."""
    from paper_1807_10749_b200.lowering import lowered

    circ, plan, req, pre = configs.build(name, n_req=4096)
    window = pre[:2] if name == "cfg5" else pre[:8]
    eng = _engine("c64")
    got = {}
    try:
        for tm in (0, 1):
            eng.set_option("tile_major", tm)
            eng.load_program(lowered(circ, plan.cut))
            eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
            got[tm] = eng.run(plan.x_p, window, 0, plan.branch_space).amps
    finally:
        eng.set_option("tile_major", 2)
    assert np.array_equal(got[0], got[1]) and np.abs(got[0]).max() > 0


@pytest.mark.parametrize("name", ["cfg2h", "cfg5", "s3x4v1", "s3x4v2", "s4x4v2", "stair3x4"])
def test_pauli_sibling_leaves_path_major(ps, name):
    """Path-major gathers (half-states outside the grouped layout's range): with
    pf_pauli=1 the I/Z side of a CZ cut evolves ONE base state per parent without
    cross terms and the gather reads each leaf as its Pauli image (flipped index,
    sign, phase).  Equal to evolving every leaf (pf_pauli=0) to complex64
    rounding, on whole jobs, branch sub-ranges, single paths and duplicate
    prefixes; small circuits also against the reference's amplitudes."""
    from paper_1807_10749_b200.lowering import lowered

    small = name not in ("cfg2h", "cfg5")
    if small:
        circ, plan, req, g = small_case(name)
        pre = plan.retained
    else:
        circ, plan, req, pre = configs.build(name, n_req=4096)
        pre = pre[:2] if name == "cfg5" else pre
    eng = _engine("c64")
    forced = {"smem_gather": 0, "grouped_leaf": 0} if small else {}
    got = {}
    try:
        for k, v in forced.items():
            eng.set_option(k, v)
        for pauli in (0, 1):
            eng.set_option("pf_pauli", pauli)
            eng.load_program(lowered(circ, plan.cut))
            d = eng.describe()  # (s4x4v2's B-side leaf level is not Pauli-compatible: a T behind an X^1/2)
            assert d["psib_side"] == (1 if pauli and d["pauli_sides"][1] else -1)
            assert d["pauli_sides"][1] == (0 if name == "s4x4v2" else 1)
            eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
            bs = plan.branch_space
            got[pauli] = (eng.run(plan.x_p, pre, 0, bs).amps,
                          eng.run(plan.x_p, pre[:1], bs // 2, bs // 2 + 1).amps,
                          eng.run(plan.x_p, pre[-1:], 1 if bs > 2 else 0, bs - 1 if bs > 2 else bs).amps,
                          eng.run(plan.x_p, np.concatenate([pre[:2], pre[:1]]), 0, bs).amps)
    finally:
        eng.set_option("pf_pauli", 1)
        eng.set_option("smem_gather", 1)
        eng.set_option("grouped_leaf", 1)
    assert np.abs(got[0][0]).max() > 0
    for a, b in zip(got[0], got[1]):  # (a single path can be exactly zero: a projector on a |0> qubit)
        assert rel_l2(b, a) <= 2e-6
    if small:
        assert rel_l2(got[1][0], g["amps_c64"]) <= C64_TOL


@pytest.mark.parametrize("name", ["cfg2h", "cfg3", "cfg4", "cfg5", "s4x4v2", "fsim3x4"])
def test_runtime_sign_variables_bitwise(ps, name):
    """jit_rsign (±1 factors chosen by thread / tile bits or digits carried as sign
    variables and folded into the next butterfly's FFMA2s) changes no bit of the
    complex64 results, whatever the cap on live variables: a·(±1) is exact."""
    from paper_1807_10749_b200.lowering import lowered

    if name in ("s4x4v2", "fsim3x4"):
        circ, plan, req, _ = small_case(name)
        pre = plan.retained
    else:
        circ, plan, req, pre = configs.build(name, n_req=4096)
        pre = pre[:2] if name == "cfg5" else pre[:8]
    eng = _engine("c64")
    got = {}
    try:
        for key, (on, cap) in {"off": (0, 8), "cap1": (1, 1), "cap3": (1, 3), "cap8": (1, 8), "cap32": (1, 32)}.items():
            eng.set_option("jit_rsign", on)
            eng.set_option("jit_rsign_max", cap)
            eng.load_program(lowered(circ, plan.cut))
            eng.set_requests_global(req, circ.n_qubits, plan.cut.block_a, plan.cut.block_b)
            got[key] = eng.run(plan.x_p, pre, 0, plan.branch_space).amps
    finally:
        eng.set_option("jit_rsign", 0)
        eng.set_option("jit_rsign_max", 8)
    assert np.abs(got["off"]).max() > 0
    for key in ("cap1", "cap3", "cap8", "cap32"):
        assert np.array_equal(got[key], got["off"]), key

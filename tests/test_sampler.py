"""Amplitude consumers: rejection sampling, tail mass,
fidelity.

CPU tests pin ``oracle/sampler_oracle.py`` against numpy's own Philox bit
generator (the reference's random source, ``sampler.py:76-79``) and, when
``/root/reference`` is present, against the reference sampler itself.  GPU
tests check the CUDA kernels (``csrc/sampler.cu``, through the C ABI) against
the pinned oracle: bit-exact for indices and accept decisions, 1e-12 relative
for the fp64 sums (summation order differs from numpy's pairwise sums).
"""
import os
import sys

import numpy as np
import pytest

from oracle import sampler_oracle as so

REF_SRC = "/root/reference/pkg/src"


def _ref_sampler():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference sources not present (GPU box)")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from gridsim import sampler

    return sampler


# ---- oracle pins (CPU) ------------------------------------------------------------
@pytest.mark.parametrize("seed", [0, 7, 2**40 + 3, 2**62 + 5])
@pytest.mark.parametrize("lane", [0, 1, 2])
def test_oracle_philox_matches_numpy(seed, lane):
    g = np.random.Generator(np.random.Philox(key=[seed, lane]))
    raw = g.bit_generator.random_raw(41)
    assert np.array_equal(raw, so.words64(seed, lane, 0, 41))
    assert np.array_equal(raw[6:33], so.words64(seed, lane, 6, 27))


@pytest.mark.parametrize("n", [1, 5, 20, 32, 33, 49, 63])
@pytest.mark.parametrize("offset", [0, 1, 3, 8, 17])
def test_oracle_committed_indices_match_numpy(n, offset):
    # the reference's draw: a fresh Philox stream, skipped to `offset`
    count = 29
    g = np.random.Generator(np.random.Philox(key=[11, 0]))
    full = g.integers(0, 1 << n, size=offset + count, dtype=np.int64)
    assert np.array_equal(full[offset:], so.committed_indices(n, count, 11, offset))


def test_oracle_uniforms_match_numpy():
    g = np.random.Generator(np.random.Philox(key=[5, 1]))
    assert np.array_equal(g.random(1001), so.uniforms(5, 1, 1001))


@pytest.mark.parametrize("size", [2, 3, 1000, 12345, 3_000_001])
def test_oracle_bounded_draws_match_numpy(size):
    # size 3,000,001: threshold / 2^32 ~ 7e-4, so the rejection path runs
    count = 200_000
    g = np.random.Generator(np.random.Philox(key=[9, 2]))
    ref = g.integers(0, size, size=count)
    assert np.array_equal(ref, so.bounded32(9, 2, size, count))


def test_oracle_matches_reference_sampler():
    S = _ref_sampler()
    rng = np.random.default_rng(1)
    for mode in ("basic", "frugal"):
        req = S.SampleRequest(n_qubits=12, count=400, seed=3, mode=mode)
        idx = S.committed_indices(req)
        assert np.array_equal(idx, so.committed_indices(12, req.batch_size, 3))
        p = rng.exponential(size=idx.size) / 2**12
        ref = S.sample(req, idx, p)
        got = so.sample(mode, 12, req.probs_per_sample, 3, idx, p)
        assert np.array_equal(ref.indices, got[0])
        assert ref.accepted_count == got[1] and ref.measured_tail_mass == got[2]
    for size in (1, 2, 7, 12345):
        p = rng.exponential(size=size) / 2**10
        t = S.tail_mass(p, 10, resamples=40, seed=9)
        est, sig = so.tail_mass(p, 10, 10, 40, 9)
        assert t.estimate == est
        assert sig == pytest.approx(t.sigma, rel=1e-12, abs=1e-300)


def test_host_request_validation():
    from paper_1807_10749_b200 import sampler as B

    with pytest.raises(B.SamplingError):
        B.SampleRequest(n_qubits=0, count=1)
    with pytest.raises(B.SamplingError):
        B.SampleRequest(n_qubits=4, count=1, mode="weird")
    with pytest.raises(B.SamplingError):
        B.plan_basic(4, 0.0)
    assert B.plan_basic(49, 1e-3) == _plan_basic_formula(49, 1e-3)
    assert B.SampleRequest(n_qubits=20, count=3, mode="basic").batch_size == 3 * B.plan_basic(20, 1e-3)
    assert B.frugal_tv_bound(10) == pytest.approx(2.0 * np.exp(-10 / (1 - np.exp(-10))))


def _plan_basic_formula(n, eps):
    import math

    return max(1, math.ceil(n * math.log(2.0) + math.log(1.0 / eps)))


# ---- device kernels vs the pinned oracle (GPU) -------------------------------------
def _chaotic(n_entries, n_qubits, seed):
    rng = np.random.default_rng(seed)
    return rng.exponential(size=n_entries) / float(1 << n_qubits)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 12, 32, 33, 53])
@pytest.mark.parametrize("offset", [0, 1, 5, 12345])
def test_device_committed_indices(n, offset):
    from paper_1807_10749_b200 import sampler as B

    req = B.SampleRequest(n_qubits=n, count=1000, seed=17)
    got = B.committed_indices(req, offset)
    assert np.array_equal(got, so.committed_indices(n, req.batch_size, 17, offset))


@pytest.mark.gpu
@pytest.mark.parametrize("mode", ["basic", "frugal"])
@pytest.mark.parametrize("n_qubits,count", [(12, 1), (16, 500), (25, 20000)])
def test_device_sample_bit_exact(mode, n_qubits, count):
    from paper_1807_10749_b200 import sampler as B

    req = B.SampleRequest(n_qubits=n_qubits, count=count, mode=mode, seed=4)
    idx = B.committed_indices(req)
    p = _chaotic(idx.size, n_qubits, 2)
    p[::97] = 0.0
    p[1::101] = req.probs_per_sample / float(1 << n_qubits)  # exactly at the cap: kept
    got = B.sample(req, idx, p)
    ref_idx, ref_count, ref_tail = so.sample(mode, n_qubits, req.probs_per_sample, 4, idx, p)
    assert got.accepted_count == ref_count
    assert np.array_equal(got.indices, ref_idx)
    assert got.measured_tail_mass == pytest.approx(ref_tail, rel=1e-12, abs=1e-300)


@pytest.mark.gpu
def test_device_sample_edges():
    from paper_1807_10749_b200 import sampler as B

    req = B.SampleRequest(n_qubits=10, count=50, seed=1)
    idx = B.committed_indices(req)
    # uniform state: accepts about one in M', no tail
    uni = np.full(idx.size, 1.0 / 1024)
    s = B.sample_frugal(req, idx, uni)
    assert s.measured_tail_mass == 0.0
    assert np.array_equal(s.indices, so.sample("frugal", 10, 10, 1, idx, uni)[0])
    # all-zero probabilities accept nothing
    assert B.sample_frugal(req, idx, np.zeros(idx.size)).accepted_count == 0
    # capped probability accepts everything
    assert B.sample_frugal(req, idx, np.full(idx.size, 1.0)).accepted_count == idx.size
    with pytest.raises(B.SamplingError):
        B.sample_frugal(req, idx[:-1], uni[:-1])
    with pytest.raises(B.SamplingError):
        B.sample_frugal(req, idx, -uni)
    with pytest.raises(B.SamplingError):
        B.sample_frugal(req, idx[:10], uni)


@pytest.mark.gpu
@pytest.mark.parametrize("size,resamples", [(1, 10), (2, 20), (12345, 100), (3_000_001, 3)])
def test_device_tail_mass(size, resamples):
    from paper_1807_10749_b200 import sampler as B

    p = _chaotic(size, 20, 5)
    got = B.tail_mass(p, 20, m_star=3, resamples=resamples, seed=8)
    est, sig = so.tail_mass(p, 20, 3, resamples, 8)
    assert got.estimate == pytest.approx(est, rel=1e-12, abs=1e-300)
    assert got.sigma == pytest.approx(sig, rel=1e-9, abs=1e-15)
    with pytest.raises(B.SamplingError):
        B.tail_mass(np.zeros(0), 20)


@pytest.mark.gpu
def test_device_inputs_stay_on_device():
    import torch

    from paper_1807_10749_b200 import sampler as B

    req = B.SampleRequest(n_qubits=20, count=3000, seed=6)
    idx = B.committed_indices(req)
    amps = (np.random.default_rng(3).standard_normal((idx.size, 2)) / 1024.0).view(np.complex128).ravel()
    p_host = B.probabilities(amps)
    # CUDA hypot vs libm hypot: a few ulp apart at most
    np.testing.assert_allclose(p_host, np.abs(amps) ** 2, rtol=8e-16 * 4, atol=0)
    d_amps = torch.from_numpy(amps.view(np.float64).copy()).cuda()
    np.testing.assert_array_equal(B.probabilities(d_amps), p_host)
    d_p = torch.from_numpy(p_host).cuda()
    d_idx = torch.from_numpy(idx).cuda()
    a = B.sample_frugal(req, d_idx, d_p)
    b = B.sample_frugal(req, idx, p_host)
    assert np.array_equal(a.indices, b.indices) and a.measured_tail_mass == b.measured_tail_mass


@pytest.mark.gpu
def test_device_fidelity():
    from paper_1807_10749_b200 import sampler as B
    from paper_1807_10749_b200.amplitudes import AmplitudeBatch, estimate_fidelity

    rng = np.random.default_rng(0)
    idx = np.arange(100_000, dtype=np.int64)
    r = rng.standard_normal(idx.size) + 1j * rng.standard_normal(idx.size)
    c = 0.3 * r + rng.standard_normal(idx.size) + 1j * rng.standard_normal(idx.size)
    ref = AmplitudeBatch(idx, r)
    cand = AmplitudeBatch(idx, c)
    assert B.estimate_fidelity_device(ref, cand) == pytest.approx(estimate_fidelity(ref, cand), rel=1e-12)
    assert B.estimate_fidelity_device(ref, ref) == pytest.approx(1.0, rel=1e-14)
    with pytest.raises(ValueError):
        B.estimate_fidelity_device(ref, AmplitudeBatch(idx, np.zeros(idx.size)))


def test_abi_argument_errors_without_a_device():
    """Argument checks happen before any device work, so they run on CPU."""
    import ctypes

    from paper_1807_10749_b200 import sampler as B

    out = np.empty(4, dtype=np.int64)
    assert B.LIB.gs_committed_indices(0, 0, 1, 0, 4, out.ctypes.data) == -1
    assert b"n_qubits" in B.LIB.gs_sampler_last_error()
    assert B.LIB.gs_committed_indices(0, 10, 1, -1, 4, out.ctypes.data) == -1
    assert B.LIB.gs_committed_indices(0, 10, 1, 0, 0, out.ctypes.data) == 0  # empty: no work
    n = ctypes.c_int64(0)
    t = ctypes.c_double(0)
    p = np.zeros(7)
    assert B.LIB.gs_sample(0, 1, 10, 10, 1, 7, out.ctypes.data, p.ctypes.data, out.ctypes.data,
                           ctypes.byref(n), ctypes.byref(t)) == -1
    assert b"not a multiple" in B.LIB.gs_sampler_last_error()
    assert B.LIB.gs_sample(0, 2, 10, 1, 1, 7, out.ctypes.data, p.ctypes.data, out.ctypes.data,
                           ctypes.byref(n), ctypes.byref(t)) == -1
    assert B.LIB.gs_tail_mass(0, 10, 10, 0, 1, 7, p.ctypes.data, ctypes.byref(t), ctypes.byref(t)) == -1
    assert B.LIB.gs_fidelity(0, 0, p.ctypes.data, p.ctypes.data, ctypes.byref(t)) == -1
    with pytest.raises(B.SamplingError):
        B.committed_indices(B.SampleRequest(n_qubits=10, count=1), offset=-1)
    with pytest.raises(B.SamplingError):
        B.tail_mass(np.zeros((2, 2)), 10)


@pytest.mark.gpu
def test_device_sampling_statistics():
    """The reference's statistical checks (test_sampler.py:120-140) on the device path."""
    from paper_1807_10749_b200 import sampler as B

    req = B.SampleRequest(16, count=1000, m_star=10, seed=4)
    idx = B.committed_indices(req)
    probs = np.random.default_rng(11).exponential(1.0 / (1 << 16), size=idx.size)
    assert abs(B.sample_frugal(req, idx, probs).accepted_count - 1000) < 300
    # one acceptance stream for both modes: every basic accept is a frugal accept when M' < M
    req_b = B.SampleRequest(12, count=200, mode="basic", epsilon=1e-3, seed=9)
    m = B.plan_basic(12, 1e-3)
    idx = B.committed_indices(req_b)
    probs = np.random.default_rng(1).exponential(1.0 / 4096, size=idx.size)
    basic = B.sample_basic(req_b, idx, probs)
    req_f = B.SampleRequest(12, count=200 * m // 10, mode="frugal", m_star=10, seed=9)
    frugal = B.sample_frugal(req_f, idx[: req_f.batch_size], probs[: req_f.batch_size])
    assert basic.accepted_count <= frugal.accepted_count
    assert set(basic.indices.tolist()) <= set(frugal.indices.tolist()) | set(idx[req_f.batch_size:].tolist())
    assert B.SampleSet(np.array([5]), 4, 1, 0.0).bitstrings == ["0101"]

"""CPU oracle for the amplitude consumers.

TEST INFRASTRUCTURE ONLY: imported by ``tests/`` (and nothing on the product
path).  It restates, in vectorised numpy, the counter-based random streams
and the reductions of the reference sampler so the CUDA kernels in
``paper_1807_10749_b200/csrc/sampler.cu`` can be checked draw by draw:

* Philox4x64-10 as numpy's ``np.random.Philox`` runs it (key = [seed, lane],
  the counter's word 0 is incremented *before* each block, 4 uint64 outputs
  per block; ``next_uint32`` hands out the low then the high half of a word),
  reference ``sampler.py:76-79``;
* ``committed_indices`` (``sampler.py:83-102``): Lemire bounded draws over a
  power-of-two range never reject, so draw i is ``word32(i) >> (32 - n)``
  (n <= 32) or ``word64(i) >> (64 - n)`` (n > 32);
* ``sample_basic`` / ``sample_frugal`` (``sampler.py:135-165``): acceptance
  stream lane 1, ``random()`` = ``(word64 >> 11) * 2**-53``;
* ``tail_mass`` bootstrap picks (``sampler.py:177-203``): lane 2, Lemire
  32-bit bounded draws with rejection.

Pinned against numpy itself in ``tests/test_sampler_oracle.py`` (numpy is the
reference's own dependency, ``pkg/pyproject.toml``).
"""
from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2E7470EE14C6C93)
M1 = np.uint64(0xCA5A826395121157)
W0 = np.uint64(0x9E3779B97F4A7C15)
W1 = np.uint64(0xBB67AE8584CAA73B)
_LO = np.uint64(0xFFFFFFFF)
_32 = np.uint64(32)


def _mulhilo(a: np.uint64, b: np.ndarray):
    """64x64 -> (hi, lo) with uint64 arrays (numpy has no 128-bit multiply)."""
    a_lo, a_hi = a & _LO, a >> _32
    b_lo, b_hi = b & _LO, b >> _32
    ll = a_lo * b_lo
    lh = a_lo * b_hi
    hl = a_hi * b_lo
    hh = a_hi * b_hi
    mid = (ll >> _32) + (lh & _LO) + (hl & _LO)
    hi = hh + (lh >> _32) + (hl >> _32) + (mid >> _32)
    lo = a * b
    return hi, lo


def philox_blocks(seed: int, lane: int, first_block: int, n_blocks: int) -> np.ndarray:
    """Output words of counter blocks ``first_block .. first_block+n_blocks-1``
    (block b runs with counter b+1), shape ``(n_blocks, 4)`` uint64."""
    with np.errstate(over="ignore"):
        c0 = np.arange(first_block + 1, first_block + 1 + n_blocks, dtype=np.uint64)
        c1 = np.zeros_like(c0)
        c2 = np.zeros_like(c0)
        c3 = np.zeros_like(c0)
        k0 = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        k1 = np.uint64(lane)
        for r in range(10):
            if r:
                k0 = k0 + W0
                k1 = k1 + W1
            hi0, lo0 = _mulhilo(M0, c0)
            hi1, lo1 = _mulhilo(M1, c2)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return np.stack([c0, c1, c2, c3], axis=1)


def words64(seed: int, lane: int, start: int, count: int) -> np.ndarray:
    b0, b1 = start // 4, (start + count + 3) // 4
    w = philox_blocks(seed, lane, b0, max(b1 - b0, 0)).reshape(-1)
    return w[start - 4 * b0: start - 4 * b0 + count]


def words32(seed: int, lane: int, start: int, count: int) -> np.ndarray:
    w0, w1 = start // 2, (start + count + 1) // 2
    w = words64(seed, lane, w0, w1 - w0)
    halves = np.stack([w & _LO, w >> _32], axis=1).reshape(-1).astype(np.uint64)
    return halves[start - 2 * w0: start - 2 * w0 + count]


def committed_indices(n_qubits: int, count: int, seed: int, offset: int = 0) -> np.ndarray:
    if n_qubits <= 32:
        w = words32(seed, 0, offset, count)
        return (w >> np.uint64(32 - n_qubits)).astype(np.int64)
    w = words64(seed, 0, offset, count)
    return (w >> np.uint64(64 - n_qubits)).astype(np.int64)


def uniforms(seed: int, lane: int, count: int) -> np.ndarray:
    return (words64(seed, lane, 0, count) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def sample(mode: str, n_qubits: int, per_sample: int, seed: int, indices, probs):
    """(accepted indices, count, tail) of sample_basic / sample_frugal."""
    probs = np.asarray(probs, dtype=np.float64)
    indices = np.asarray(indices, dtype=np.int64)
    n_states = 1 << n_qubits
    u = uniforms(seed, 1, probs.size)
    if mode == "basic":
        cap = per_sample / n_states
        accept = (probs <= cap) & (u < probs * n_states / per_sample)
        tail = float(probs[probs > cap].sum() * n_states / probs.size)
    else:
        accept = u < np.minimum(1.0, probs * n_states / per_sample)
        tail = float(probs[probs > per_sample / n_states].sum() * n_states / probs.size)
    return indices[accept], int(accept.sum()), tail


def bounded32(seed: int, lane: int, size: int, count: int) -> np.ndarray:
    """``integers(0, size, count)`` for 1 < size <= 2^32 (Lemire, rejection)."""
    rng_excl = np.uint64(size)
    threshold = np.uint64(((1 << 32) - size) % size)
    out = np.empty(0, dtype=np.int64)
    start = 0
    while out.size < count:
        need = count - out.size
        chunk = need + need // 1024 + 64
        w = words32(seed, lane, start, chunk)
        m = w * rng_excl
        ok = (m & _LO) >= threshold
        out = np.concatenate([out, (m[ok] >> _32).astype(np.int64)])
        start += chunk
    return out[:count]


def tail_mass(probs, n_qubits: int, m_star: int, resamples: int, seed: int):
    probs = np.asarray(probs, dtype=np.float64)
    n_states = float(1 << n_qubits)
    threshold = m_star / n_states
    contrib = np.where(probs > threshold, probs, 0.0)
    scale = n_states / probs.size
    estimate = float(contrib.sum() * scale)
    if probs.size == 1:
        picks = np.zeros((resamples, 1), dtype=np.int64)
    else:
        picks = bounded32(seed, 2, probs.size, resamples * probs.size).reshape(resamples, probs.size)
    boots = contrib[picks].sum(axis=1) * scale
    return estimate, float(boots.std())

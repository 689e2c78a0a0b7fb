"""Rejection sampling, tail mass and fidelity on the device.

Mirrors the reference sampler (``pkg/src/gridsim/sampler.py``): the same
names, arguments, result types and ``SamplingError`` behaviour, with the
per-entry work -- the committed index batch (``committed_indices``
``sampler.py:83-102``), the acceptance draws (``sample_basic`` /
``sample_frugal`` ``:135-165``), the tail-mass estimate and its bootstrap
(``tail_mass`` ``:177-203``) -- done by the CUDA kernels in
``csrc/sampler.cu`` through the C ABI (``include/gridsim_b200.h``).  The
random streams are numpy's Philox4x64-10 (key ``[seed, lane]``) regenerated
on the device counter by counter, so indices and accept decisions are
bit-identical to the reference's.  ``estimate_fidelity_device`` is
``pathsum.py:648-664`` on the device.

Inputs may be numpy arrays (copied in) or CUDA tensors (read in place, e.g.
the amplitudes of a ``run_batched`` whose output stayed on the device).
There is no CPU fallback: without the library this module does not import.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from .amplitudes import AmplitudeBatch
from .engine import LIB

DEFAULT_FRUGAL_M = 10
BOOTSTRAP_RESAMPLES = 100

_P = ctypes.c_void_p
LIB.gs_sampler_last_error.restype = ctypes.c_char_p
LIB.gs_committed_indices.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64, ctypes.c_int64,
                                     ctypes.c_int64, _P]
LIB.gs_sample.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64,
                          ctypes.c_int64, _P, _P, _P, ctypes.POINTER(ctypes.c_int64),
                          ctypes.POINTER(ctypes.c_double)]
LIB.gs_tail_mass.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64,
                             ctypes.c_int64, _P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
LIB.gs_fidelity.argtypes = [ctypes.c_int32, ctypes.c_int64, _P, _P, ctypes.POINTER(ctypes.c_double)]
LIB.gs_probabilities.argtypes = [ctypes.c_int32, ctypes.c_int64, _P, _P]


class SamplingError(ValueError):
    pass


def _check(code: int):
    if code != 0:
        msg = LIB.gs_sampler_last_error().decode()
        if code == -1:
            raise SamplingError(msg)
        raise RuntimeError(msg)


_TORCH_DTYPE_NAMES = {np.dtype(np.int64): "torch.int64", np.dtype(np.float64): "torch.float64",
                      np.dtype(np.complex128): "torch.complex128"}


def _device_tensor(x, dtype, device: int | None = None):
    """Check a CUDA tensor handed to the sampler kernels: element type, layout and
    device must be what the kernel reads (a float32/int32/complex64 tensor would
    be read with 8/16-byte strides past its end), and the producer's queued work
    must be complete -- the sampler runs on its own stream."""
    want = _TORCH_DTYPE_NAMES[np.dtype(dtype)]
    if str(x.dtype) != want:
        raise SamplingError(f"device tensor has dtype {x.dtype}, the sampler needs {want}")
    if not x.is_contiguous():
        raise SamplingError("device tensor must be contiguous")
    if device is not None and x.device.index is not None and x.device.index != device:
        raise SamplingError(f"tensor is on cuda:{x.device.index}, the request names device {device}")
    import torch

    torch.cuda.current_stream(x.device).synchronize()
    return x


def _addr(x, dtype, device: int | None = None):
    """(pointer, keep-alive, length) of a numpy array or a CUDA tensor."""
    if hasattr(x, "data_ptr") and getattr(x, "is_cuda", False):
        x = _device_tensor(x, dtype, device)
        return x.data_ptr(), x, x.numel()
    arr = np.ascontiguousarray(x, dtype=dtype)
    return arr.ctypes.data, arr, arr.size


def _seed(seed: int) -> int:
    return int(seed) & 0xFFFFFFFFFFFFFFFF


def plan_basic(n_qubits: int, epsilon: float) -> int:
    """M = ceil(n ln 2 + ln(1/eps)) (reference ``sampler.py:26-38``)."""
    if n_qubits < 0:
        raise SamplingError(f"negative qubit count {n_qubits}")
    if not 0.0 < epsilon <= 1.0:
        raise SamplingError(f"epsilon must be in (0, 1], got {epsilon}")
    m = math.ceil(n_qubits * math.log(2.0) + math.log(1.0 / epsilon))
    return max(1, m)


@dataclass(frozen=True)
class SampleRequest:
    """Reference ``sampler.py:41-73``."""

    n_qubits: int
    count: int
    mode: str = "frugal"
    epsilon: float = 1e-3
    m_star: int = DEFAULT_FRUGAL_M
    seed: int = 0
    device: int = 0

    def __post_init__(self):
        if self.n_qubits < 1:
            raise SamplingError(f"need at least 1 qubit, got {self.n_qubits}")
        if self.count < 1:
            raise SamplingError(f"sample count must be >= 1, got {self.count}")
        if self.mode not in ("basic", "frugal"):
            raise SamplingError(f"unknown mode {self.mode!r}")
        if not 0.0 < self.epsilon < 1.0:
            raise SamplingError(f"epsilon must be in (0, 1), got {self.epsilon}")
        if self.m_star < 1:
            raise SamplingError(f"M' must be >= 1, got {self.m_star}")

    @property
    def n_states(self) -> int:
        return 1 << self.n_qubits

    @property
    def probs_per_sample(self) -> int:
        if self.mode == "basic":
            return plan_basic(self.n_qubits, self.epsilon)
        return self.m_star

    @property
    def batch_size(self) -> int:
        return self.count * self.probs_per_sample


def committed_indices(req: SampleRequest, offset: int = 0) -> np.ndarray:
    """Reference ``sampler.py:83-102``, drawn on the device."""
    if offset < 0:
        raise SamplingError(f"negative chunk offset {offset}")
    if req.n_qubits > 63:
        raise SamplingError("committed indices are int64: at most 63 qubits")
    out = np.empty(req.batch_size, dtype=np.int64)
    _check(LIB.gs_committed_indices(req.device, req.n_qubits, _seed(req.seed), offset, out.size, out.ctypes.data))
    return out


@dataclass
class SampleSet:
    indices: np.ndarray
    n_qubits: int
    accepted_count: int
    measured_tail_mass: float

    @property
    def bitstrings(self) -> list:
        fmt = f"0{self.n_qubits}b"
        return [format(int(i), fmt) for i in self.indices]


def _check_batch(indices, probs, per_sample: int):
    is_dev = hasattr(probs, "is_cuda") and probs.is_cuda
    if not is_dev:
        probs = np.asarray(probs, dtype=np.float64)
    if not (hasattr(indices, "is_cuda") and indices.is_cuda):
        indices = np.asarray(indices, dtype=np.int64)
    if tuple(indices.shape) != tuple(probs.shape) or len(probs.shape) != 1:
        raise SamplingError("indices and probs must be parallel 1-d arrays")
    n = int(probs.shape[0])
    if n == 0 or n % per_sample:
        raise SamplingError(f"batch of {n} is not a multiple of {per_sample} probabilities per sample")
    if bool((probs < 0).any()):
        raise SamplingError("negative probability in batch")
    return indices, probs, n


def _sample(req: SampleRequest, mode: int, per_sample: int, indices, probs) -> SampleSet:
    indices, probs, n = _check_batch(indices, probs, per_sample)
    ip, ikeep, _ = _addr(indices, np.int64, req.device)
    pp, pkeep, _ = _addr(probs, np.float64, req.device)
    out = np.empty(n, dtype=np.int64)
    count = ctypes.c_int64(0)
    tail = ctypes.c_double(0.0)
    _check(LIB.gs_sample(req.device, mode, req.n_qubits, per_sample, _seed(req.seed), n, ip, pp,
                         out.ctypes.data, ctypes.byref(count), ctypes.byref(tail)))
    del ikeep, pkeep
    return SampleSet(out[: count.value].copy(), req.n_qubits, int(count.value), float(tail.value))


def sample_basic(req: SampleRequest, indices, probs) -> SampleSet:
    """Reference ``sampler.py:135-150``."""
    return _sample(req, 0, plan_basic(req.n_qubits, req.epsilon), indices, probs)


def sample_frugal(req: SampleRequest, indices, probs) -> SampleSet:
    """Reference ``sampler.py:153-165``."""
    return _sample(req, 1, req.m_star, indices, probs)


def sample(req: SampleRequest, indices, probs) -> SampleSet:
    if req.mode == "basic":
        return sample_basic(req, indices, probs)
    return sample_frugal(req, indices, probs)


@dataclass
class TailEstimate:
    estimate: float
    sigma: float
    threshold: float
    resamples: int


def tail_mass(probs, n_qubits: int, m_star: int = DEFAULT_FRUGAL_M, resamples: int = BOOTSTRAP_RESAMPLES,
              seed: int = 0, device: int = 0) -> TailEstimate:
    """Reference ``sampler.py:177-203``."""
    if not (hasattr(probs, "is_cuda") and probs.is_cuda):
        probs = np.asarray(probs, dtype=np.float64)
    if len(probs.shape) != 1 or int(probs.shape[0]) == 0:
        raise SamplingError("need a non-empty 1-d probability batch")
    pp, keep, n = _addr(probs, np.float64, device)
    est = ctypes.c_double(0.0)
    sig = ctypes.c_double(0.0)
    _check(LIB.gs_tail_mass(device, n_qubits, m_star, resamples, _seed(seed), n, pp, ctypes.byref(est),
                            ctypes.byref(sig)))
    del keep
    return TailEstimate(float(est.value), float(sig.value), m_star / float(1 << n_qubits), resamples)


def frugal_tv_bound(m_star: int = DEFAULT_FRUGAL_M) -> float:
    """Reference ``sampler.py:206-208``."""
    return 2.0 * math.exp(-m_star / (1.0 - math.exp(-m_star)))


def probabilities(amps, device: int = 0) -> np.ndarray:
    """``np.abs(amps) ** 2`` (reference ``cli.py:228``) on the device."""
    if not (hasattr(amps, "is_cuda") and amps.is_cuda):
        amps = np.ascontiguousarray(amps, dtype=np.complex128)
        ap, keep, n = amps.ctypes.data, amps, amps.size
    else:
        # complex128 tensor, or float64 (re, im) pairs
        if amps.is_complex():
            keep = _device_tensor(amps, np.complex128, device)
            n = amps.numel()
        else:
            keep = _device_tensor(amps, np.float64, device)
            if amps.numel() % 2:
                raise SamplingError("float64 (re, im) pairs need an even element count")
            n = amps.numel() // 2
        ap = keep.data_ptr()
    out = np.empty(n, dtype=np.float64)
    _check(LIB.gs_probabilities(device, n, ap, out.ctypes.data))
    del keep
    return out


def estimate_fidelity_device(reference: AmplitudeBatch, candidate: AmplitudeBatch, device: int = 0) -> float:
    """``estimate_fidelity`` (reference ``pathsum.py:648-664``) on the device."""
    if len(reference.indices) == 0:
        raise ValueError("empty amplitude batch")
    if not np.array_equal(reference.indices, candidate.indices):
        raise ValueError("fidelity estimate needs matching index sets")
    r = np.ascontiguousarray(reference.amps, dtype=np.complex128)
    c = np.ascontiguousarray(candidate.amps, dtype=np.complex128)
    out = ctypes.c_double(0.0)
    code = LIB.gs_fidelity(device, r.size, r.ctypes.data, c.ctypes.data, ctypes.byref(out))
    if code != 0:
        raise ValueError(LIB.gs_sampler_last_error().decode())
    return float(out.value)

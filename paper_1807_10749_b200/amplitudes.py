"""Amplitude batches, the result type of the hot path.

Mirrors ``AmplitudeBatch`` (reference ``statevec.py:449-476``: int64 indices,
complex128 amplitudes in request order), ``estimate_fidelity``
(``pathsum.py:648-664``) and the amplitude text format
(``statevec.py:479-511``: ``index_hex re im`` lines, ``# key value`` header).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ACC_DTYPE = np.complex128


@dataclass
class AmplitudeBatch:
    indices: np.ndarray  # int64
    amps: np.ndarray  # complex128

    def __post_init__(self):
        self.indices = np.asarray(self.indices, dtype=np.int64)
        self.amps = np.asarray(self.amps, dtype=ACC_DTYPE)
        if self.indices.shape != self.amps.shape:
            raise ValueError("indices and amplitudes differ in length")

    @classmethod
    def zeros(cls, indices) -> "AmplitudeBatch":
        idx = np.asarray(indices, dtype=np.int64)
        return cls(idx, np.zeros(idx.shape, dtype=ACC_DTYPE))

    def copy(self) -> "AmplitudeBatch":
        return AmplitudeBatch(self.indices.copy(), self.amps.copy())


def estimate_fidelity(reference: AmplitudeBatch, candidate: AmplitudeBatch) -> float:
    """``|<r|c>|^2 / (<r|r><c|c>)`` over a shared index set, in fp64."""
    if len(reference.indices) == 0:
        raise ValueError("empty amplitude batch")
    if not np.array_equal(reference.indices, candidate.indices):
        raise ValueError("fidelity estimate needs matching index sets")
    r = reference.amps.astype(ACC_DTYPE)
    c = candidate.amps.astype(ACC_DTYPE)
    rr = float(np.vdot(r, r).real)
    cc = float(np.vdot(c, c).real)
    if rr == 0 or cc == 0:
        raise ValueError("zero-norm batch in fidelity estimate")
    return float(abs(np.vdot(r, c)) ** 2 / (rr * cc))


def write_amplitudes(path, batch: AmplitudeBatch, digits: int = 9, header: dict | None = None) -> None:
    fmt = f"%x %.{digits - 1}e %.{digits - 1}e\n"
    with open(path, "w") as fh:
        for key, value in (header or {}).items():
            fh.write(f"# {key} {value}\n")
        for i, a in zip(batch.indices, batch.amps):
            fh.write(fmt % (i, a.real, a.imag))


def read_amplitudes(path):
    header, idx, amps = {}, [], []
    with open(path) as fh:
        for lineno, raw in enumerate(fh, start=1):
            line = raw.strip()
            if not line:
                continue
            if line.startswith("#"):
                kv = line[1:].strip().split(None, 1)
                if len(kv) == 2:
                    header[kv[0]] = kv[1]
                continue
            parts = line.split()
            if len(parts) != 3:
                raise ValueError(f"amplitude line {lineno}: expected 3 fields, got {raw!r}")
            idx.append(int(parts[0], 16))
            amps.append(complex(float(parts[1]), float(parts[2])))
    return AmplitudeBatch(np.array(idx, dtype=np.int64), np.array(amps, dtype=ACC_DTYPE)), header

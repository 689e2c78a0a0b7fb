"""Seeded request (bitstring) sets.

``challenge_indices`` restates the reference's verifier index generator
(``validate.py:72-86``): k distinct sorted basis indices of an n-qubit space
from ``default_rng(index_seed)``.  BASELINE configs draw their bitstrings
with it (seed 12345).
"""
from __future__ import annotations

import numpy as np


class ValidationError(ValueError):
    pass


def challenge_indices(n_qubits: int, k: int, index_seed: int) -> np.ndarray:
    space = 1 << n_qubits
    if k > space:
        raise ValidationError(f"cannot pick {k} distinct indices from {space} states")
    rng = np.random.default_rng(index_seed)
    if k == space:
        return np.arange(space, dtype=np.int64)
    if k > space // 4 and space <= (1 << 24):
        return np.sort(rng.choice(space, size=k, replace=False).astype(np.int64))
    chosen = set()
    while len(chosen) < k:
        chosen.update(int(v) for v in rng.integers(0, space, size=k - len(chosen)))
    return np.array(sorted(chosen), dtype=np.int64)

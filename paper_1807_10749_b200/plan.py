"""Path-space planning: Schmidt terms of cross gates, the prefix/branch split,
the seeded retained-prefix subset and the request bit split.

Host-side mirror of the planning half of the reference ``gridsim/pathsum.py``.
The GPU engine consumes a :class:`SimPlan`; it never re-derives one, so path
enumeration and subset selection are bit-exact by construction as long as
these functions reproduce the reference (pinned by ``tests/test_plan.py``
against plans the reference itself produced, ``tests/golden/``).

* ``schmidt_decompose`` -- ``pathsum.py:92-119`` (term order defines digits)
* ``split_requests``    -- ``pathsum.py:122-140``
* ``path_digits`` / ``path_id`` -- ``pathsum.py:219-236``
* ``SimPlan``           -- ``pathsum.py:246-274``
* ``retained_prefixes`` -- ``pathsum.py:277-291`` (numpy PCG64 streams)
* ``make_plan``         -- ``pathsum.py:294-329`` and ``_default_branch_digits``
  ``pathsum.py:332-344``
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .circuit import (Circuit, CircuitError, Cut, GateKind, as_kind, choose_cut, gate_block,
                      gate_matrix, kind_name)

_P0 = np.diag([1.0, 0.0]).astype(np.complex128)
_P1 = np.diag([0.0, 1.0]).astype(np.complex128)
_Z = np.diag([1.0, -1.0]).astype(np.complex128)
_I2 = np.eye(2, dtype=np.complex128)
_RAISE = np.array([[0, 1], [0, 0]], dtype=np.complex128)  # |0><1|
_LOWER = np.array([[0, 0], [1, 0]], dtype=np.complex128)  # |1><0|

SVD_REL_CUTOFF = 1e-7  # reference _SVD_TOL, pathsum.py:52


@dataclass
class TermDecomposition:
    """``U = sum_k kron(L_k, R_k)``; ``terms[k] = (L_k, R_k)`` (``pathsum.py:55-64``)."""

    kind: GateKind
    terms: list

    @property
    def rank(self) -> int:
        return len(self.terms)


def _operator_svd_terms(u: np.ndarray) -> list:
    """Operator-Schmidt terms of a generic 4x4 via SVD of the realigned matrix.

    Realign ``U[(i1 i2),(j1 j2)] -> R[(i1 j1),(i2 j2)]``; each kept singular
    triple gives ``(sqrt(s) * left, sqrt(s) * right)``.  Order: descending
    singular value (rounded to 12 digits), exact ties broken by the rounded
    entries of L then R -- the reference's ordering (``pathsum.py:72-89``).
    """
    r = np.asarray(u, dtype=np.complex128).reshape(2, 2, 2, 2).transpose(0, 2, 1, 3).reshape(4, 4)
    left, sing, right = np.linalg.svd(r)
    kept = np.flatnonzero(sing > SVD_REL_CUTOFF * sing[0])
    terms = []
    for k in kept:
        scale = math.sqrt(sing[k])
        terms.append((scale * left[:, k].reshape(2, 2), scale * right[k, :].reshape(2, 2)))

    def order(pos):
        lo, ro = terms[pos]
        flat = np.concatenate([lo.ravel(), ro.ravel()])
        return (-round(sing[kept[pos]], 12),) + tuple(
            (round(v.real, 12), round(v.imag, 12)) for v in flat
        )

    return [terms[pos] for pos in sorted(range(len(terms)), key=order)]


def schmidt_decompose(gate) -> TermDecomposition:
    """Operator decomposition of a two-qubit gate, ``Gate``, ``GateKind`` or 4x4.

    CZ -> ``[(P0, I), (P1, Z)]`` and iSWAP -> the four projector/ladder terms,
    exactly; anything else through :func:`_operator_svd_terms`.
    """
    kind, matrix = None, None
    if hasattr(gate, "kind") and hasattr(gate, "qubits"):  # a gate record (ours or gridsim's)
        kind, matrix = as_kind(gate.kind), gate_matrix(gate)
    elif hasattr(gate, "value") or isinstance(gate, str):  # a gate kind
        kind = as_kind(gate)
    else:
        matrix = np.asarray(gate, dtype=np.complex128)
        if matrix.shape != (4, 4):
            raise ValueError(f"expected a 4x4 matrix, got {matrix.shape}")
    if kind is GateKind.CZ:
        return TermDecomposition(kind, [(_P0, _I2), (_P1, _Z)])
    if kind is GateKind.ISWAP:
        return TermDecomposition(
            kind, [(_P0, _P0), (_P1, _P1), (1j * _RAISE, _LOWER), (1j * _LOWER, _RAISE)]
        )
    if matrix is None:
        from .circuit import GATE_TABLE

        matrix = GATE_TABLE[kind_name(kind)][1]
        if matrix is None or matrix.shape != (4, 4):
            raise ValueError(f"{kind_name(kind)!r} is not a two-qubit gate with a fixed matrix")
    return TermDecomposition(kind or GateKind.GENERIC_2Q, _operator_svd_terms(matrix))


def split_requests(n_qubits: int, block_a, block_b, indices):
    """Global basis indices -> (idx_a, idx_b) block-local indices.

    Global bit ``n-1-q`` (qubit q) goes to local bit ``n_blk-1-j`` where q is
    the j-th qubit of its block (ascending).  ``IndexError`` when an index is
    outside ``[0, 2^n)`` (``pathsum.py:122-140``).
    """
    idx = np.asarray(indices, dtype=np.int64)
    if idx.size and (idx.min() < 0 or idx.max() >= (1 << n_qubits)):
        raise IndexError("request index outside the state space")
    halves = []
    for block in (block_a, block_b):
        width = len(block)
        local = np.zeros(idx.shape, dtype=np.int64)
        # runs of consecutive qubits are runs of consecutive bits: one shift+mask each
        j = 0
        while j < width:
            k = j
            while k + 1 < width and block[k + 1] == block[k] + 1:
                k += 1
            run = k - j + 1
            src = n_qubits - 1 - block[k]  # global bit of the run's lowest bit
            dst = width - 1 - k            # local bit of the run's lowest bit
            local |= ((idx >> src) & ((1 << run) - 1)) << dst
            j = k + 1
        halves.append(local)
    return halves[0], halves[1]


def path_digits(path_id_value: int, radices) -> tuple:
    """Big-endian mixed-radix digits; digit k picks the term of cross gate k."""
    rest = int(path_id_value)
    out = []
    for base in reversed(tuple(radices)):
        rest, d = divmod(rest, base)
        out.append(d)
    if rest:
        raise ValueError("path id outside the path space")
    return tuple(reversed(out))


def path_id(digits, radices) -> int:
    value = 0
    for d, base in zip(digits, radices):
        if not 0 <= d < base:
            raise ValueError(f"digit {d} outside radix {base}")
        value = value * base + d
    return value


def space_size(radices) -> int:
    return math.prod(int(r) for r in radices)


@dataclass
class SimPlan:
    """One truncated hybrid run: cut, radices, split and retained prefixes."""

    cut: Cut
    fidelity: float
    radices: tuple
    x_p: int
    x_b: int
    d_p: int
    d_b: int
    seed: int
    retained: np.ndarray  # sorted int64 prefix ids

    @property
    def x(self) -> int:
        return len(self.radices)

    @property
    def prefix_space(self) -> int:
        return space_size(self.radices[: self.x_p])

    @property
    def branch_space(self) -> int:
        return space_size(self.radices[self.x_p :])

    @property
    def path_space(self) -> int:
        return space_size(self.radices)

    @property
    def n_paths(self) -> int:
        return len(self.retained) * self.branch_space


def retained_prefixes(prefix_space: int, fidelity: float, seed: int) -> np.ndarray:
    """``max(1, round(f*space))`` distinct prefixes, sorted, from ``default_rng(seed)``.

    Same draw sequence as the reference: the full range when everything is
    kept, ``choice(replace=False)`` above a quarter of the space, otherwise
    rejection-sampled batches of ``integers`` (``pathsum.py:277-291``).
    """
    m = max(1, round(fidelity * prefix_space))
    if m > prefix_space:
        raise CircuitError(f"cannot retain {m} of {prefix_space} prefixes")
    rng = np.random.default_rng(seed)
    if m == prefix_space:
        return np.arange(prefix_space, dtype=np.int64)
    if m > prefix_space // 4:
        return np.sort(rng.choice(prefix_space, size=m, replace=False).astype(np.int64))
    picked = set()
    while len(picked) < m:
        picked.update(int(v) for v in rng.integers(0, prefix_space, size=m - len(picked)))
    return np.array(sorted(picked), dtype=np.int64)


def cross_gates(circuit: Circuit, cut: Cut) -> list:
    return [g for g in circuit.gates if len(g.qubits) == 2 and gate_block(g, cut) == "cross"]


def _auto_branch_digits(circuit: Circuit, cut: Cut, cross: list, workers: int) -> int:
    """Smallest x_b whose branch work covers the checkpoint copy 32x (``pathsum.py:332-344``)."""
    x = len(cross)
    cap = x - max(0, math.ceil(math.log2(workers))) if workers > 1 else x
    cap = max(0, cap)
    copy_cost = (1 << cut.n_a) + (1 << cut.n_b)
    for x_b in range(cap + 1):
        branches = space_size(schmidt_decompose(g).rank for g in cross[x - x_b :])
        d_b = circuit.n_cycles - (cross[x - x_b].cycle if x_b > 0 else circuit.n_cycles)
        if branches * max(1, d_b) * copy_cost >= 32 * copy_cost:
            return x_b
    return cap


def make_plan(
    circuit: Circuit,
    fidelity: float = 1.0,
    x_p: int | None = None,
    x_b: int | None = None,
    seed: int = 0,
    cut: Cut | None = None,
    workers: int = 1,
) -> SimPlan:
    """Build the plan (reference ``make_plan``, ``pathsum.py:294-329``)."""
    if not 0 < fidelity <= 1:
        raise CircuitError(f"fidelity must be in (0, 1], got {fidelity}")
    if cut is None:
        cut = choose_cut(circuit)
    cross = cross_gates(circuit, cut)
    radices = tuple(schmidt_decompose(g).rank for g in cross)
    x = len(radices)
    if x_p is None and x_b is None:
        x_b = _auto_branch_digits(circuit, cut, cross, workers)
        x_p = x - x_b
    elif x_p is None:
        x_p = x - x_b
    elif x_b is None:
        x_b = x - x_p
    if x_p < 0 or x_b < 0 or x_p + x_b != x:
        raise CircuitError(f"split x_p={x_p}, x_b={x_b} incompatible with {x} cross gates")
    d_p = cross[x_p].cycle if x_b > 0 else circuit.n_cycles
    d_b = circuit.n_cycles - d_p
    retained = retained_prefixes(space_size(radices[:x_p]), fidelity, seed)
    return SimPlan(cut, fidelity, radices, x_p, x_b, d_p, d_b, seed, retained)

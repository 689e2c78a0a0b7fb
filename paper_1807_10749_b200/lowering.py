"""Lowering of a circuit under a cut into the flat op stream the C ABI takes.

Mirrors ``_lower_uncached`` / ``_one_qubit_op`` (reference
``pathsum.py:157-195``) op for op:

* gates are visited in circuit order (stable cycle order);
* a gate inside one block becomes ``diag1``/``mat1`` (one qubit; ``diag1``
  when both off-diagonals are exactly zero), ``diag2`` (CZ) or ``mat2``
  (any other two-qubit gate, ``|first second>`` order);
* a gate across the cut becomes ``("cross", k)`` and its Schmidt terms are
  split into a block-A and a block-B one-qubit op, swapping the term sides
  when the gate's first qubit lies in block B;
* the local qubit of a global qubit is its index in the sorted block tuple.

Coefficients are kept in complex128; the engine rounds them to complex64 in
``c64`` mode exactly as the reference's ``astype(DTYPE)`` does.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .circuit import Circuit, Cut, gate_block, gate_matrix, kind_name
from .plan import schmidt_decompose

OP_DIAG1, OP_MAT1, OP_DIAG2, OP_MAT2, OP_CROSS = 0, 1, 2, 3, 4
OP_NAMES = ("diag1", "mat1", "diag2", "mat2", "cross")


@dataclass
class LoweredProgram:
    n_a: int
    n_b: int
    op_kind: np.ndarray
    op_blk: np.ndarray
    op_q0: np.ndarray
    op_q1: np.ndarray
    op_cycle: np.ndarray
    op_coef: np.ndarray
    cross_rank: np.ndarray
    cross_cycle: np.ndarray
    cross_qa: np.ndarray
    cross_qb: np.ndarray
    term_kind_a: np.ndarray
    term_coef_a: np.ndarray
    term_kind_b: np.ndarray
    term_coef_b: np.ndarray
    coef: np.ndarray  # complex128 pool

    @property
    def n_ops(self) -> int:
        return len(self.op_kind)

    @property
    def n_cross(self) -> int:
        return len(self.cross_rank)

    @property
    def radices(self) -> tuple:
        return tuple(int(r) for r in self.cross_rank)


class _Pool:
    def __init__(self):
        self.chunks = []
        self.size = 0

    def add(self, values) -> int:
        arr = np.asarray(values, dtype=np.complex128).ravel()
        at = self.size
        self.chunks.append(arr)
        self.size += arr.size
        return at

    def array(self) -> np.ndarray:
        if not self.chunks:
            return np.zeros(0, dtype=np.complex128)
        return np.concatenate(self.chunks)


def _single(u: np.ndarray, pool: _Pool) -> tuple:
    """(kind, coef offset) of a one-qubit operator, diag1 iff off-diagonals are 0."""
    if abs(u[0, 1]) == 0 and abs(u[1, 0]) == 0:
        return OP_DIAG1, pool.add(np.diag(u))
    return OP_MAT1, pool.add(u)


def lower_circuit(circuit: Circuit, cut: Cut) -> LoweredProgram:
    """Lower any circuit record (ours or ``gridsim``'s: gates with ``cycle``,
    ``kind.value``, ``qubits``, ``matrix``) under any cut record."""
    where_a = {q: j for j, q in enumerate(cut.block_a)}
    where_b = {q: j for j, q in enumerate(cut.block_b)}
    pool = _Pool()
    ops = []  # (kind, blk, q0, q1, cycle, coef)
    xr, xc, xqa, xqb = [], [], [], []
    tka, tca, tkb, tcb = [], [], [], []
    for g in circuit.gates:
        side = gate_block(g, cut)
        if side == "cross":
            k = len(xr)
            first, second = g.qubits
            a_first = first in where_a
            qa = where_a[first] if a_first else where_a[second]
            qb = where_b[second] if a_first else where_b[first]
            dec = schmidt_decompose(g)
            for left, right in dec.terms:
                on_a, on_b = (left, right) if a_first else (right, left)
                ka, ca = _single(on_a, pool)
                kb, cb = _single(on_b, pool)
                tka.append(ka)
                tca.append(ca)
                tkb.append(kb)
                tcb.append(cb)
            xr.append(dec.rank)
            xc.append(g.cycle)
            xqa.append(qa)
            xqb.append(qb)
            ops.append((OP_CROSS, -1, k, -1, g.cycle, 0))
            continue
        blk = 0 if side == "a" else 1
        where = where_a if blk == 0 else where_b
        u = gate_matrix(g)
        if len(g.qubits) == 1:
            kind, at = _single(u, pool)
            ops.append((kind, blk, where[g.qubits[0]], -1, g.cycle, at))
        elif kind_name(g.kind) == "cz":
            ops.append(
                (OP_DIAG2, blk, where[g.qubits[0]], where[g.qubits[1]], g.cycle, pool.add(np.diag(u)))
            )
        else:
            ops.append((OP_MAT2, blk, where[g.qubits[0]], where[g.qubits[1]], g.cycle, pool.add(u)))
    cols = list(zip(*ops)) if ops else [[]] * 6
    i32 = lambda v: np.asarray(v, dtype=np.int32)
    i64 = lambda v: np.asarray(v, dtype=np.int64)
    return LoweredProgram(
        n_a=cut.n_a,
        n_b=cut.n_b,
        op_kind=i32(cols[0]),
        op_blk=i32(cols[1]),
        op_q0=i32(cols[2]),
        op_q1=i32(cols[3]),
        op_cycle=i32(cols[4]),
        op_coef=i64(cols[5]),
        cross_rank=i32(xr),
        cross_cycle=i32(xc),
        cross_qa=i32(xqa),
        cross_qb=i32(xqb),
        term_kind_a=i32(tka),
        term_coef_a=i64(tca),
        term_kind_b=i32(tkb),
        term_coef_b=i64(tcb),
        coef=pool.array(),
    )


def lowered(circuit: Circuit, cut: Cut) -> LoweredProgram:
    """Cached :func:`lower_circuit`, kept on the circuit like ``_lower`` (``pathsum.py:145-155``)."""
    cache = circuit.__dict__.setdefault("_b200_lowered", {})
    prog = cache.get(cut)
    if prog is None:
        prog = cache[cut] = lower_circuit(circuit, cut)
    return prog

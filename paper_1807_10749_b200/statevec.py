"""Full state-vector engine on the B200.

Mirrors the reference's dense engine surface (``gridsim/statevec.py``):

* ``StateBlock`` (``statevec.py:40-60``): ``2**n_qubits`` complex64
  amplitudes, qubit 0 in the most significant bit;
* ``run_full(circuit, slice_bytes, mem_limit)`` (``statevec.py:410-446``):
  evolve ``|0...0>`` through the whole circuit; ``MemoryBudgetError`` when the
  state does not fit ``mem_limit`` (``:420-425``);
* ``fetch_amplitudes(state, indices)`` (``statevec.py:471-476``):
  ``IndexError`` outside the state.

``run_full`` lowers the circuit *uncut* (every gate on one block holding the
whole register) and runs it through the same pass scheduler and generated
sm_100a pass kernels as the path sum (``gs_run_full`` in the C ABI); the
reference's L2 slicing has no counterpart here -- a pass already streams
tiles of 2^13 amplitudes through registers and shared memory -- so
``slice_bytes`` is accepted and ignored (the reference's result does not
depend on it either, ``:416-418``).  There is no CPU fallback.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .amplitudes import ACC_DTYPE, AmplitudeBatch
from .circuit import Circuit, Cut
from .lowering import lowered

DTYPE = np.complex64
DEFAULT_SLICE_BYTES = 262144


class MemoryBudgetError(MemoryError):
    pass


@dataclass
class StateBlock:
    """2**n_qubits amplitudes (complex64; complex128 from a c128 run), qubit 0 the MSB."""

    n_qubits: int
    amps: np.ndarray

    @classmethod
    def zero_state(cls, n_qubits: int) -> "StateBlock":
        amps = np.zeros(2**n_qubits, dtype=DTYPE)
        amps[0] = 1.0
        return cls(n_qubits, amps)

    def copy(self) -> "StateBlock":
        return StateBlock(self.n_qubits, self.amps.copy())

    def norm_squared(self) -> float:
        return float(np.einsum("i,i->", self.amps, self.amps.conj(), dtype=ACC_DTYPE).real)


def full_cut(circuit: Circuit) -> Cut:
    """The trivial cut: block A is the whole register, block B is empty."""
    return Cut("full", -1, tuple(range(circuit.n_qubits)), ())


def run_full(
    circuit: Circuit,
    slice_bytes: int = DEFAULT_SLICE_BYTES,
    mem_limit: int | None = None,
    device: int = 0,
    dtype="c64",
) -> StateBlock:
    """Simulate the full circuit from |0...0> on the GPU (reference ``run_full``)."""
    from .engine import ENGINES, precision_code, run_with_memory_retry

    n = circuit.n_qubits
    precision_code(dtype)  # ValueError for an unknown dtype, before any work
    required = (2**n) * np.dtype(DTYPE).itemsize
    if mem_limit is not None and required > mem_limit:
        raise MemoryBudgetError(f"state of {n} qubits requires {required} bytes, budget is {mem_limit}")
    if n > 31:
        raise MemoryBudgetError(f"state of {n} qubits exceeds the 2^31-amplitude block limit")
    del slice_bytes
    eng = ENGINES.get(device, dtype)
    with eng.lock:
        eng.load_program(lowered(circuit, full_cut(circuit)))
        return StateBlock(n, run_with_memory_retry(eng, eng.run_full).amps)


def fetch_amplitudes(state: StateBlock, indices) -> AmplitudeBatch:
    """Read amplitudes at the requested indices, in request order."""
    idx = np.asarray(indices, dtype=np.int64)
    if len(idx) and (idx.min() < 0 or idx.max() >= len(state.amps)):
        raise IndexError("amplitude index outside the state")
    return AmplitudeBatch(idx, state.amps[idx].astype(ACC_DTYPE))

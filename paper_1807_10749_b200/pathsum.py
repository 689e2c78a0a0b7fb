"""Drop-in hybrid path-sum entry points, executed on a B200.

Same names, arguments, result type and exceptions as the reference engine
(``gridsim/pathsum.py``):

* ``run_approx(circuit, plan, requests, skip_zeros=True, engine=...)``
  (``pathsum.py:419-443``) -- sum over every retained prefix and branch;
* ``run_batched(circuit, plan, requests, prefixes=None, row_cap=None)``
  (``pathsum.py:574-640``) -- any subset of prefixes (the shard hook);
* ``run_prefix_tree(circuit, plan, prefix, requests, skip_zeros=True)``
  (``pathsum.py:377-416``) -- one prefix, all its branches;
* ``run_path(circuit, plan, path, requests, skip_zeros=True)``
  (``pathsum.py:347-362``) -- a single path.

All four lower the circuit (cached on the circuit object, like ``_lower``),
split the requests into block-local indices and call the C ABI; the result is
an :class:`AmplitudeBatch` in request order.  ``engine`` accepts the
reference's ``"batched"`` and ``"perjob"`` names (both run here on the GPU --
there is no CPU path) and ``"b200"``; anything else is a ``ValueError``.
``skip_zeros`` and ``row_cap`` are accepted for signature compatibility; the
results never depended on them in the reference either (``test_pathsum.py:197-202``).
Extra keywords: ``device`` (CUDA ordinal) and ``dtype`` (``"c64"`` -- the
reference's complex64 states -- or ``"c128"``).
"""
from __future__ import annotations

import numpy as np

from .amplitudes import AmplitudeBatch
from .circuit import Circuit
from .engine import ENGINES, run_with_memory_retry
from .lowering import lowered
from .plan import SimPlan, path_digits

ENGINE_NAMES = ("b200", "batched", "perjob")


def _engine_for(circuit: Circuit, plan: SimPlan, requests, device: int, dtype):
    """Engine with ``circuit`` loaded and ``requests`` set; the caller must hold
    ``eng.lock`` (acquired here, re-entrant) until its runs are done."""
    prog = lowered(circuit, plan.cut)
    if prog.radices != tuple(int(r) for r in plan.radices):
        raise ValueError("plan radices do not match the circuit's cross gates under plan.cut")
    idx = np.asarray(requests, dtype=np.int64).ravel()
    eng = ENGINES.get(device, dtype)
    with eng.lock:
        eng.load_program(prog)
        # split_requests (pathsum.py:122-140) runs on the device; IndexError as in the reference
        eng.set_requests_global(idx, circuit.n_qubits, plan.cut.block_a, plan.cut.block_b)
    return eng, idx


def _run(circuit, plan, requests, prefixes, branch_lo, branch_hi, device, dtype):
    prog = lowered(circuit, plan.cut)
    if prog.radices != tuple(int(r) for r in plan.radices):
        raise ValueError("plan radices do not match the circuit's cross gates under plan.cut")
    idx = np.asarray(requests, dtype=np.int64).ravel()
    eng = ENGINES.get(device, dtype)
    with eng.lock:  # one load -> split -> run sequence at a time per context
        eng.load_program(prog)
        # split_requests (pathsum.py:122-140) runs on the device, overlapped with the
        # first gate passes; IndexError as in the reference
        res = run_with_memory_retry(eng, lambda: eng.run_batched(
            idx, circuit.n_qubits, plan.cut.block_a, plan.cut.block_b, plan.x_p, prefixes, branch_lo,
            branch_hi))
    return AmplitudeBatch(idx, res.amps)


def run_approx(
    circuit: Circuit,
    plan: SimPlan,
    requests,
    skip_zeros: bool = True,
    engine: str = "b200",
    device: int = 0,
    dtype="c64",
) -> AmplitudeBatch:
    """Sum of all retained prefixes x all branches at the requested indices."""
    if engine not in ENGINE_NAMES:
        raise ValueError(f"unknown engine {engine!r}")
    return _run(circuit, plan, requests, plan.retained, 0, plan.branch_space, device, dtype)


def run_batched(
    circuit: Circuit,
    plan: SimPlan,
    requests,
    prefixes=None,
    row_cap: int | None = None,
    device: int = 0,
    dtype="c64",
) -> AmplitudeBatch:
    """Sum over ``prefixes`` (default ``plan.retained``) x all branches."""
    pre = plan.retained if prefixes is None else np.asarray(prefixes, dtype=np.int64)
    return _run(circuit, plan, requests, pre, 0, plan.branch_space, device, dtype)


def run_prefix_tree(
    circuit: Circuit,
    plan: SimPlan,
    prefix: int,
    requests,
    skip_zeros: bool = True,
    device: int = 0,
    dtype="c64",
) -> AmplitudeBatch:
    """Contribution of one prefix job: every branch completion of ``prefix``."""
    path_digits(int(prefix), plan.radices[: plan.x_p])  # ValueError outside the prefix space
    return _run(circuit, plan, requests, [int(prefix)], 0, plan.branch_space, device, dtype)


def run_path(
    circuit: Circuit,
    plan: SimPlan,
    path: int,
    requests,
    skip_zeros: bool = True,
    device: int = 0,
    dtype="c64",
) -> AmplitudeBatch:
    """Contribution of the single path ``path`` (prefix * branch_space + branch)."""
    path = int(path)
    path_digits(path, plan.radices)  # ValueError outside the path space
    prefix, branch = divmod(path, plan.branch_space)
    return _run(circuit, plan, requests, [prefix], branch, branch + 1, device, dtype)

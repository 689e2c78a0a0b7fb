"""B200-native Schroedinger-Feynman path-sum engine (arXiv 1807.10749).

Drop-in for the hot path of the reference ``gridsim`` package: the circuit IR
and planner keep the reference semantics on the host; ``run_approx`` and its
siblings execute the path sum in hand-written sm_100a CUDA kernels through
the C ABI declared in ``include/gridsim_b200.h``.

The engine symbols (``run_approx`` ...) import the CUDA library lazily so the
host-side modules stay importable on machines without the built ``.so``.
"""
from .amplitudes import AmplitudeBatch, estimate_fidelity, read_amplitudes, write_amplitudes
from .circuit import (
    Circuit,
    CircuitError,
    Cut,
    Gate,
    GateKind,
    ParseError,
    all_cuts,
    choose_cut,
    circuit_hash,
    gate_block,
    gate_matrix,
    parse_circuit,
    serialize_circuit,
)
from .plan import (
    SimPlan,
    TermDecomposition,
    make_plan,
    path_digits,
    path_id,
    retained_prefixes,
    schmidt_decompose,
    split_requests,
)
from .requests import challenge_indices

__version__ = "0.1.0"

_ENGINE_NAMES = ("run_approx", "run_batched", "run_prefix_tree", "run_path")


def __getattr__(name):
    if name in _ENGINE_NAMES:
        from . import pathsum

        return getattr(pathsum, name)
    raise AttributeError(name)


__all__ = [
    "AmplitudeBatch",
    "Circuit",
    "CircuitError",
    "Cut",
    "Gate",
    "GateKind",
    "ParseError",
    "SimPlan",
    "TermDecomposition",
    "all_cuts",
    "challenge_indices",
    "choose_cut",
    "circuit_hash",
    "estimate_fidelity",
    "gate_block",
    "gate_matrix",
    "make_plan",
    "parse_circuit",
    "path_digits",
    "path_id",
    "read_amplitudes",
    "retained_prefixes",
    "run_approx",
    "run_batched",
    "run_path",
    "run_prefix_tree",
    "schmidt_decompose",
    "serialize_circuit",
    "split_requests",
    "write_amplitudes",
    "__version__",
]

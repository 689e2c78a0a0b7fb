"""``engine="b200"`` for the reference package ``gridsim`` -- the drop-in boundary.

The reference's only extension point on the hot path is the ``engine=`` string
of ``gridsim.pathsum.run_approx`` (``pathsum.py:419-443``, dispatch at
``:433-436``), plus the ``prefixes=`` subset hook of ``run_batched``
(``:574-579``) that campaign workers and shards use.  :func:`install` plugs
this package in there:

* ``gridsim.pathsum.run_approx(..., engine="b200")`` runs the path sum through
  the C ABI (``include/gridsim_b200.h``) on a B200 and returns
  ``gridsim.statevec.AmplitudeBatch`` in request order;
* with ``default=True`` the reference's own default engine (``"batched"``) and
  ``run_batched`` / ``run_prefix_tree`` / ``run_path`` / ``run_full`` are routed
  to the device as well -- in ``gridsim.pathsum`` and in every ``gridsim``
  module that bound those names at import (``validate``, ``cli``,
  ``orchestrator``, ``statevec``), so unmodified callers (the CLI ``pathsim``
  command, verifier rounds, campaign workers) run on the B200;
* :func:`uninstall` restores the reference functions.

Inputs are the reference's own objects: ``gridsim.Circuit`` / ``Gate`` /
``GateKind`` / ``Cut`` / ``SimPlan`` are consumed as they are (the lowering
keys gates by ``kind.value`` and ``matrix``, never by enum identity), and the
plan is used as given -- its retained prefixes are never recomputed.

``gridsim`` itself is located by :func:`load_gridsim`: an importable
``gridsim``, else the offline install under ``<repo>/baseline/_ref``
(``pip install --no-index --target baseline/_ref``), else ``ImportError``.
The product engine never imports ``gridsim``; only this adapter (and the
modules that are thin layers over the reference, ``validate`` and ``shards``)
do.
"""
from __future__ import annotations

import contextlib
import importlib
import os
import sys
import threading

import numpy as np

ENGINE = "b200"
_REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_REF_DIRS = (os.path.join(_REPO, "baseline", "_ref"),)
_LOCK = threading.RLock()
_SAVED: dict = {}  # (module name, attribute) -> reference object
_ROUTED = ("run_approx", "run_batched", "run_prefix_tree", "run_path", "run_full")
_BINDERS = ("gridsim.pathsum", "gridsim.validate", "gridsim.cli", "gridsim.orchestrator",
            "gridsim.statevec")


def load_gridsim(submodule: str | None = None):
    """Import ``gridsim`` (or ``gridsim.<submodule>``); see the module docstring."""
    name = "gridsim" + (f".{submodule}" if submodule else "")
    try:
        return importlib.import_module(name)
    except ImportError:
        pass
    for d in _REF_DIRS:
        if os.path.isdir(os.path.join(d, "gridsim")) and d not in sys.path:
            sys.path.append(d)
    try:
        return importlib.import_module(name)
    except ImportError as exc:
        raise ImportError(
            "the reference package gridsim is not installed; install it offline with "
            "`python -m pip install --no-index --no-build-isolation --no-deps "
            "--target baseline/_ref <gridsim source>`"
        ) from exc


def gridsim_available() -> bool:
    try:
        load_gridsim()
        return True
    except ImportError:
        return False


def _batch(ref_batch_type, res):
    return ref_batch_type(np.asarray(res.indices, dtype=np.int64), np.asarray(res.amps))


def _device_functions(sv):
    """B200 versions of the routed functions, returning the reference's types."""
    from . import pathsum as ours
    from . import statevec as ours_sv

    Batch = sv.AmplitudeBatch

    def run_approx(circuit, plan, requests, skip_zeros=True, engine=ENGINE, **kw):
        return _batch(Batch, ours.run_approx(circuit, plan, requests, skip_zeros, ENGINE, **kw))

    def run_batched(circuit, plan, requests, prefixes=None, row_cap=None, **kw):
        return _batch(Batch, ours.run_batched(circuit, plan, requests, prefixes, row_cap, **kw))

    def run_prefix_tree(circuit, plan, prefix, requests, skip_zeros=True, _split=None, _out=None,
                        **kw):
        res = ours.run_prefix_tree(circuit, plan, prefix, requests, skip_zeros, **kw)
        if _out is not None:  # the reference's in-place accumulate form (pathsum.py:377-416)
            _out.amps += res.amps
            return _out
        return _batch(Batch, res)

    def run_path(circuit, plan, path, requests, skip_zeros=True, **kw):
        return _batch(Batch, ours.run_path(circuit, plan, path, requests, skip_zeros, **kw))

    def run_full(circuit, slice_bytes=None, mem_limit=None, **kw):
        args = {} if mem_limit is None else {"mem_limit": mem_limit}
        st = ours_sv.run_full(circuit, **args, **kw)
        return sv.StateBlock(st.n_qubits, st.amps)

    return {"run_approx": run_approx, "run_batched": run_batched,
            "run_prefix_tree": run_prefix_tree, "run_path": run_path, "run_full": run_full}


def run_approx_b200(circuit, plan, requests, skip_zeros: bool = True, **kw):
    """``run_approx`` on the B200 for ``gridsim`` objects, returning
    ``gridsim.statevec.AmplitudeBatch`` (the function the reference's
    ``engine="b200"`` branch calls)."""
    return _device_functions(load_gridsim("statevec"))["run_approx"](circuit, plan, requests, skip_zeros, **kw)


def install(default: bool = False) -> None:
    """Register ``engine="b200"`` in ``gridsim`` (see the module docstring).

    Idempotent; a second call may switch ``default`` on or off.
    """
    with _LOCK:
        uninstall()
        ps = load_gridsim("pathsum")
        sv = load_gridsim("statevec")
        dev = _device_functions(sv)
        ref_approx = ps.run_approx

        def run_approx(circuit, plan, requests, skip_zeros=True, engine="batched"):
            if engine == ENGINE or (default and engine == "batched"):
                return dev["run_approx"](circuit, plan, requests, skip_zeros)
            return ref_approx(circuit, plan, requests, skip_zeros, engine)

        run_approx.__doc__ = ref_approx.__doc__
        run_approx.__wrapped__ = ref_approx
        replace = {"run_approx": run_approx}
        refs = {name: getattr(sv if name == "run_full" else ps, name) for name in _ROUTED}
        if default:
            for name in _ROUTED[1:]:
                replace[name] = dev[name]
        for modname in _BINDERS:
            try:
                mod = load_gridsim(modname.split(".", 1)[1])
            except ImportError:
                continue
            for name, fn in replace.items():
                if getattr(mod, name, None) is refs[name]:
                    _SAVED[(modname, name)] = refs[name]
                    setattr(mod, name, fn)


def uninstall() -> None:
    """Put the reference functions back wherever :func:`install` replaced them."""
    with _LOCK:
        for (modname, name), fn in _SAVED.items():
            setattr(sys.modules[modname], name, fn)
        _SAVED.clear()


def installed() -> bool:
    return bool(_SAVED)


@contextlib.contextmanager
def routed_to_device(default: bool = True):
    """``install(default)`` for the duration of a block, then restore the previous state.

    Not re-entrant across threads: the routing is process-global, like the
    reference's own module-level functions.
    """
    with _LOCK:
        before = dict(_SAVED)
        was_default = before and any(k[1] != "run_approx" for k in before)
        install(default=default)
        try:
            yield
        finally:
            uninstall()
            if before:
                install(default=bool(was_default))


def to_gridsim(circuit):
    """The same circuit as a ``gridsim.Circuit`` (through the shared text format;
    identity when it already is one)."""
    gc = load_gridsim("circuit")
    if isinstance(circuit, gc.Circuit):
        return circuit
    from .circuit import serialize_circuit

    return gc.parse_circuit(serialize_circuit(circuit), circuit.rows, circuit.cols)


def to_gridsim_cut(cut):
    gc = load_gridsim("circuit")
    if cut is None or isinstance(cut, gc.Cut):
        return cut
    return gc.Cut(cut.orientation, cut.position, tuple(cut.block_a), tuple(cut.block_b))

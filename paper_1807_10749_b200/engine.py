"""ctypes binding of ``libgridsim_b200.so`` (C ABI: ``include/gridsim_b200.h``).

There is no CPU fallback: if the shared library is missing the import of
this module raises, and a context on a machine without a CUDA device fails at
creation.  Host-only contexts (``device=-1``) exist for planning/dry runs and
compute nothing.
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass

import numpy as np

from .circuit import CircuitError
from .lowering import LoweredProgram

LIB_NAME = "libgridsim_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

GS_OK, GS_ERR_ARG, GS_ERR_PLAN, GS_ERR_INDEX, GS_ERR_CUDA, GS_ERR_NOMEM, GS_ERR_STATE = (
    0, -1, -2, -3, -4, -5, -6,
)
GS_C64, GS_C128 = 0, 1

# every symbol include/gridsim_b200.h declares
EXPORTED_SYMBOLS = (
    "gs_sampler_last_error",
    "gs_committed_indices",
    "gs_sample",
    "gs_tail_mass",
    "gs_fidelity",
    "gs_probabilities",
    "gs_abi_version",
    "gs_device_count",
    "gs_create",
    "gs_destroy",
    "gs_last_error",
    "gs_set_stream",
    "gs_set_option",
    "gs_load_program",
    "gs_set_requests",
    "gs_run",
    "gs_describe",
    "gs_set_requests_global",
    "gs_run_batched",
    "gs_run_full",
    "gs_host_alloc",
    "gs_host_free",
)


class GsStats(ctypes.Structure):
    _fields_ = [
        ("n_paths", ctypes.c_int64),
        ("n_nodes", ctypes.c_int64),
        ("n_levels", ctypes.c_int64),
        ("n_pass_launches", ctypes.c_int64),
        ("n_gather_launches", ctypes.c_int64),
        ("n_launches", ctypes.c_int64),
        ("pass_bytes", ctypes.c_double),
        ("gather_bytes", ctypes.c_double),
        ("ms_pass", ctypes.c_double),
        ("ms_gather", ctypes.c_double),
        ("ms_total", ctypes.c_double),
        ("pass_amp_updates", ctypes.c_double),
        ("pass_bytes_min", ctypes.c_double),
        ("h2d_bytes", ctypes.c_double),
        ("d2h_bytes", ctypes.c_double),
        ("host_ms_enqueue", ctypes.c_double),
        ("host_ms_max_gap", ctypes.c_double),
        ("ms_leaf", ctypes.c_double),
        ("upper_bytes_alg", ctypes.c_double),
        ("leaf_bytes_alg", ctypes.c_double),
        ("n_leaf_launches", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


_P = ctypes.c_void_p
_I32P = ctypes.POINTER(ctypes.c_int32)
_I64P = ctypes.POINTER(ctypes.c_int64)
_F64P = ctypes.POINTER(ctypes.c_double)


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    lib = ctypes.CDLL(LIB_PATH)
    lib.gs_abi_version.restype = ctypes.c_int
    lib.gs_device_count.argtypes = [ctypes.POINTER(ctypes.c_int)]
    lib.gs_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]
    lib.gs_destroy.argtypes = [_P]
    lib.gs_destroy.restype = None
    lib.gs_last_error.argtypes = [_P]
    lib.gs_last_error.restype = ctypes.c_char_p
    lib.gs_set_stream.argtypes = [_P, _P]
    lib.gs_set_option.argtypes = [_P, ctypes.c_char_p, ctypes.c_int64]
    lib.gs_load_program.argtypes = [
        _P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
        _I32P, _I32P, _I32P, _I32P, _I32P, _I64P,
        ctypes.c_int32, _I32P, _I32P, _I32P, _I32P,
        _I32P, _I64P, _I32P, _I64P,
        ctypes.c_int64, _F64P,
    ]
    lib.gs_set_requests.argtypes = [_P, ctypes.c_int64, _I64P, _I64P]
    lib.gs_set_requests_global.argtypes = [_P, ctypes.c_int64, _I64P, ctypes.c_int32, _I32P, _I32P]
    lib.gs_describe.argtypes = [_P, ctypes.c_char_p, ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]
    lib.gs_run_batched.argtypes = [
        _P, ctypes.c_int64, _I64P, ctypes.c_int32, _I32P, _I32P, ctypes.c_int32, ctypes.c_int64, _I64P,
        ctypes.c_int64, ctypes.c_int64, _F64P, _P, ctypes.c_int32, ctypes.POINTER(GsStats),
    ]
    lib.gs_run.argtypes = [
        _P, ctypes.c_int32, ctypes.c_int64, _I64P, ctypes.c_int64, ctypes.c_int64,
        _F64P, _P, ctypes.c_int32, ctypes.POINTER(GsStats),
    ]
    lib.gs_run_full.argtypes = [_P, _P, _P, ctypes.POINTER(GsStats)]
    lib.gs_host_alloc.argtypes = [ctypes.c_int64, ctypes.POINTER(_P)]
    lib.gs_host_free.argtypes = [_P]
    lib.gs_host_free.restype = None
    if lib.gs_abi_version() != 2:
        raise ImportError("libgridsim_b200.so ABI version mismatch")
    return lib


LIB = _load()


def _ptr(arr: np.ndarray, ctype):
    return arr.ctypes.data_as(ctypes.POINTER(ctype))


def device_count() -> int:
    n = ctypes.c_int(0)
    LIB.gs_device_count(ctypes.byref(n))
    return n.value


class _PinnedBlock:
    """Owner of one page-locked host block; numpy views keep it alive through
    ``__array_interface__``, and its release returns the block to the pool."""

    def __init__(self, pool, ptr: int, nbytes: int, count: int, dtype=np.complex128):
        self._pool, self.ptr, self.nbytes = pool, ptr, nbytes
        self.__array_interface__ = {
            "shape": (count,), "typestr": np.dtype(dtype).str, "data": (ptr, False), "version": 3,
        }

    def __del__(self):
        pool = self._pool
        if pool is not None:
            try:
                pool._give_back(self.ptr, self.nbytes)
            except Exception:  # interpreter shutdown
                pass


class _PinnedPool:
    """Reusable page-locked result buffers (gs_host_alloc): run_batched returns
    its complex128 amplitudes in them, so the result download is one full-speed
    DMA; a buffer is reused once every array on it has been released."""

    def __init__(self, keep_bytes: int = 1 << 30):
        self.free = {}  # nbytes -> [ptr]
        self.kept = 0
        self.keep_bytes = keep_bytes
        self.pid = os.getpid()

    def array(self, count: int, dtype=np.complex128) -> np.ndarray | None:
        if os.getpid() != self.pid:  # pinned memory belongs to the parent's CUDA context
            self.__init__(self.keep_bytes)
        nbytes = max(16, np.dtype(dtype).itemsize * count)
        lst = self.free.get(nbytes)
        if lst:
            ptr = lst.pop()
            self.kept -= nbytes
        else:
            p = _P()
            if LIB.gs_host_alloc(nbytes, ctypes.byref(p)) != GS_OK or not p.value:
                return None
            ptr = p.value
        return np.asarray(_PinnedBlock(self, ptr, nbytes, count, dtype))

    def _give_back(self, ptr: int, nbytes: int):
        if os.getpid() != self.pid:
            return
        if self.kept + nbytes <= self.keep_bytes:
            self.free.setdefault(nbytes, []).append(ptr)
            self.kept += nbytes
        else:
            LIB.gs_host_free(_P(ptr))


_PINNED = _PinnedPool()


class EngineError(RuntimeError):
    pass


def _raise(code: int, msg: str):
    if code == GS_ERR_ARG:
        raise ValueError(msg)
    if code == GS_ERR_PLAN:
        raise CircuitError(msg)
    if code == GS_ERR_INDEX:
        raise IndexError(msg)
    if code == GS_ERR_NOMEM:
        raise MemoryError(msg)
    raise EngineError(msg)


def precision_code(dtype) -> int:
    if dtype in ("c64", np.complex64) or dtype == np.dtype(np.complex64):
        return GS_C64
    if dtype in ("c128", np.complex128) or dtype == np.dtype(np.complex128):
        return GS_C128
    raise ValueError(f"unsupported dtype {dtype!r}; use 'c64' or 'c128'")


@dataclass
class RunResult:
    amps: np.ndarray | None
    stats: dict


class Engine:
    """One device context: a loaded program, a request set and runs over leaves.

    A context holds mutable state (the loaded program, the request set, the
    run's buffers), so a load -> set requests -> run sequence must not
    interleave with another thread's.  The library releases the GIL during
    its calls; callers hold ``engine.lock`` across the whole sequence (the
    package's entry points do).  The lock is re-entrant.
    """

    def __init__(self, device: int = 0, dtype="c64"):
        self.lock = threading.RLock()
        self.device = int(device)
        self.precision = precision_code(dtype)
        h = _P()
        code = LIB.gs_create(self.device, self.precision, ctypes.byref(h))
        if code != GS_OK:
            raise EngineError(
                f"gs_create(device={device}) failed with code {code}: no usable CUDA device"
            )
        self._h = h
        self._program = None
        self._requests = None
        self.n_req = -1

    def close(self):
        if getattr(self, "_h", None):
            LIB.gs_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, code: int):
        if code != GS_OK:
            if not getattr(self, "_h", None):
                raise EngineError("engine context was released (ENGINES.release_others); get a fresh one")
            _raise(code, LIB.gs_last_error(self._h).decode())

    def set_option(self, key: str, value: int):
        self._check(LIB.gs_set_option(self._h, key.encode(), int(value)))

    def set_stream(self, stream_handle: int | None):
        self._check(LIB.gs_set_stream(self._h, _P(stream_handle or 0)))

    def load_program(self, prog: LoweredProgram):
        if self._program is prog:
            return
        coef = np.ascontiguousarray(
            np.stack([prog.coef.real, prog.coef.imag], axis=-1).ravel(), dtype=np.float64
        )
        if coef.size == 0:
            coef = np.zeros(2, dtype=np.float64)
        arrs = {
            name: np.ascontiguousarray(getattr(prog, name))
            for name in (
                "op_kind", "op_blk", "op_q0", "op_q1", "op_cycle", "op_coef",
                "cross_rank", "cross_cycle", "cross_qa", "cross_qb",
                "term_kind_a", "term_coef_a", "term_kind_b", "term_coef_b",
            )
        }
        for name, a in arrs.items():
            if a.size == 0:
                arrs[name] = np.zeros(1, dtype=a.dtype)
        i32, i64 = ctypes.c_int32, ctypes.c_int64
        code = LIB.gs_load_program(
            self._h, prog.n_a, prog.n_b, prog.n_ops,
            _ptr(arrs["op_kind"], i32), _ptr(arrs["op_blk"], i32), _ptr(arrs["op_q0"], i32),
            _ptr(arrs["op_q1"], i32), _ptr(arrs["op_cycle"], i32), _ptr(arrs["op_coef"], i64),
            prog.n_cross, _ptr(arrs["cross_rank"], i32), _ptr(arrs["cross_cycle"], i32),
            _ptr(arrs["cross_qa"], i32), _ptr(arrs["cross_qb"], i32),
            _ptr(arrs["term_kind_a"], i32), _ptr(arrs["term_coef_a"], i64),
            _ptr(arrs["term_kind_b"], i32), _ptr(arrs["term_coef_b"], i64),
            int(prog.coef.size), _ptr(coef, ctypes.c_double),
        )
        self._check(code)
        self._program = prog
        self._requests = None
        self.n_req = -1

    def describe(self) -> dict:
        import json

        need = ctypes.c_int64(0)
        self._check(LIB.gs_describe(self._h, None, 0, ctypes.byref(need)))
        buf = ctypes.create_string_buffer(int(need.value))
        self._check(LIB.gs_describe(self._h, buf, need.value, ctypes.byref(need)))
        return json.loads(buf.value.decode())

    def set_requests_global(self, indices, n_qubits: int, block_a, block_b):
        """Upload global indices; the device splits them for the loaded cut."""
        idx = np.ascontiguousarray(indices, dtype=np.int64).ravel()
        pidx = idx if idx.size else np.zeros(1, dtype=np.int64)
        ba = np.ascontiguousarray(block_a, dtype=np.int32)
        bb = np.ascontiguousarray(block_b, dtype=np.int32)
        self._check(LIB.gs_set_requests_global(
            self._h, idx.size, _ptr(pidx, ctypes.c_int64), int(n_qubits),
            _ptr(ba, ctypes.c_int32), _ptr(bb, ctypes.c_int32)))
        self._requests = None
        self.n_req = int(idx.size)

    def set_requests(self, idx_a: np.ndarray, idx_b: np.ndarray, key=None):
        if key is not None and self._requests is not None and self._requests == key:
            return
        a = np.ascontiguousarray(idx_a, dtype=np.int64)
        b = np.ascontiguousarray(idx_b, dtype=np.int64)
        if a.shape != b.shape:
            raise ValueError("idx_a and idx_b differ in length")
        pa = a if a.size else np.zeros(1, dtype=np.int64)
        pb = b if b.size else np.zeros(1, dtype=np.int64)
        self._check(
            LIB.gs_set_requests(self._h, a.size, _ptr(pa, ctypes.c_int64), _ptr(pb, ctypes.c_int64))
        )
        self._requests = key
        self.n_req = int(a.size)

    def run_batched(self, indices, n_qubits: int, block_a, block_b, x_p: int, prefixes, branch_lo: int,
                    branch_hi: int, out: np.ndarray | None = None) -> RunResult:
        """gs_run_batched: load `indices` (global basis indices) and sum the leaves
        in one call; the request upload overlaps the first gate passes."""
        idx = np.ascontiguousarray(indices, dtype=np.int64).ravel()
        pidx = idx if idx.size else np.zeros(1, dtype=np.int64)
        ba = np.ascontiguousarray(block_a, dtype=np.int32)
        bb = np.ascontiguousarray(block_b, dtype=np.int32)
        pre = np.ascontiguousarray(prefixes, dtype=np.int64).ravel()
        ppre = pre if pre.size else np.zeros(1, dtype=np.int64)
        # every entry is overwritten: no need to zero-fill; page-locked when possible
        host = out
        if host is None and self.device >= 0 and idx.size:
            host = _PINNED.array(idx.size)
        if host is None:
            host = np.empty(idx.size, dtype=np.complex128)
        if host.dtype != np.complex128 or not host.flags.c_contiguous or host.size != idx.size:
            raise ValueError("output must be a contiguous complex128 array with one entry per request")
        hp = host.view(np.float64) if host.size else None
        st = GsStats()
        self.n_req = -1
        self._requests = None
        self._check(LIB.gs_run_batched(
            self._h, idx.size, _ptr(pidx, ctypes.c_int64), int(n_qubits), _ptr(ba, ctypes.c_int32),
            _ptr(bb, ctypes.c_int32), int(x_p), pre.size, _ptr(ppre, ctypes.c_int64), int(branch_lo),
            int(branch_hi), _ptr(hp, ctypes.c_double) if hp is not None else None, None, 0, ctypes.byref(st)))
        self.n_req = int(idx.size)
        return RunResult(host, st.as_dict())

    def run_full(self, out: np.ndarray | None = None) -> RunResult:
        """gs_run_full: the loaded (uncut) program's full state, complex64 (c64
        engine) or complex128 (c128), qubit 0 in the most significant bit."""
        prog = self._program
        if prog is None:
            raise RuntimeError("no program loaded")
        dt = np.complex64 if self.precision == 0 else np.complex128
        n = 1 << int(prog.n_a)
        host = out if out is not None else (_PINNED.array(n, dt) if self.device >= 0 else None)
        if host is None:
            host = np.empty(n, dtype=dt)
        if host.dtype != dt or not host.flags.c_contiguous or host.size != n:
            raise ValueError(f"output must be a contiguous {np.dtype(dt).name} array of 2^{prog.n_a} entries")
        st = GsStats()
        self._check(LIB.gs_run_full(self._h, host.ctypes.data_as(_P), None, ctypes.byref(st)))
        return RunResult(host, st.as_dict())

    def run(
        self,
        x_p: int,
        prefixes,
        branch_lo: int,
        branch_hi: int,
        out: np.ndarray | None = None,
        out_device_ptr: int | None = None,
        accumulate: bool = False,
        want_host: bool = True,
    ) -> RunResult:
        pre = np.ascontiguousarray(prefixes, dtype=np.int64).ravel()
        ppre = pre if pre.size else np.zeros(1, dtype=np.int64)
        host = None
        if want_host:
            host = out if out is not None else np.zeros(max(self.n_req, 0), dtype=np.complex128)
            if host.dtype != np.complex128 or not host.flags.c_contiguous:
                raise ValueError("output must be a contiguous complex128 array")
        st = GsStats()
        hp = host.view(np.float64) if host is not None and host.size else None
        code = LIB.gs_run(
            self._h, int(x_p), pre.size, _ptr(ppre, ctypes.c_int64), int(branch_lo), int(branch_hi),
            _ptr(hp, ctypes.c_double) if hp is not None else None,
            _P(out_device_ptr or 0), 1 if accumulate else 0, ctypes.byref(st),
        )
        self._check(code)
        return RunResult(host, st.as_dict())


class _EngineCache:
    """Per-process engines, created lazily (never before a fork)."""

    def __init__(self):
        self.pid = None
        self.engines = {}
        self._lock = threading.Lock()

    def get(self, device: int, dtype) -> Engine:
        """The process's engine for (device, dtype); hold ``engine.lock`` while using it."""
        key = (int(device), precision_code(dtype))
        with self._lock:
            if self.pid != os.getpid():
                self.pid = os.getpid()
                self.engines = {}
            eng = self.engines.get(key)
            if eng is None:
                eng = self.engines[key] = Engine(device, dtype)
            return eng

    def release_others(self, keep: Engine) -> bool:
        """Destroy this process's other idle engines on ``keep``'s device (each
        sizes its path-tree buffers from the free HBM it saw, so a second
        context can find too little).  True when any memory was released."""
        freed = False
        with self._lock:
            for key, eng in list(self.engines.items()):
                if eng is keep or eng.device != keep.device or not eng.lock.acquire(blocking=False):
                    continue
                try:
                    eng.close()
                    del self.engines[key]
                    freed = True
                finally:
                    eng.lock.release()
        return freed


def run_with_memory_retry(eng: Engine, fn):
    """``fn()``; on a device-memory shortfall, release the process's other idle
    engines and try once more."""
    try:
        return fn()
    except MemoryError:
        if not ENGINES.release_others(eng):
            raise
        return fn()


ENGINES = _EngineCache()

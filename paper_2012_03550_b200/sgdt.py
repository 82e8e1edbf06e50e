"""Python front end of the C-ABI (include/sgdt.h) -- plumbing for tests and bench.

The product is libsgdt.so (CUDA kernels for sm_100a + the C-ABI).  This module
only marshals numpy buffers through ctypes; it never computes anything on the
host and there is no fallback: if the library or a GPU is missing it raises.

Names and error behaviour mirror the reference API (proj/include/sptucker):
ConfigError / DataError / NumericError / DomainError (common.hpp:13-43) are
raised for the matching C-ABI codes.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _build

MAX_ORDER = 8


class SptuckerError(RuntimeError):
    code = 1


class InternalError(SptuckerError):
    code = 1


class ConfigError(SptuckerError):
    code = 2


class DataError(SptuckerError):
    code = 3


class NumericError(SptuckerError):
    code = 4


class DomainError(SptuckerError):
    code = 5


_ERRORS = {1: InternalError, 2: ConfigError, 3: DataError, 4: NumericError, 5: DomainError}


class _TensorDesc(C.Structure):
    _fields_ = [("order", C.c_int), ("dims", C.POINTER(C.c_uint32)), ("nnz", C.c_uint64),
                ("coords", C.POINTER(C.c_uint32)), ("values", C.POINTER(C.c_double)),
                ("mode_perm", C.POINTER(C.POINTER(C.c_uint32)))]


class CoreHyper(C.Structure):
    """CoreHyper (core_optimizer.hpp:13-19)."""
    _fields_ = [("lr", C.c_double), ("reg", C.c_double), ("batch_m", C.c_uint64),
                ("resample_per_mode", C.c_int), ("incremental_residual", C.c_int)]


class FactorHyper(C.Structure):
    """FactorHyper (factor_optimizer.hpp:14-18)."""
    _fields_ = [("lr", C.c_double), ("reg", C.c_double), ("row_fraction", C.c_double)]


class _CoreStats(C.Structure):
    _fields_ = [("batch_size", C.c_uint64), ("effective_workers", C.c_uint64)]


class _FactorStats(C.Structure):
    _fields_ = [("rows_updated", C.c_uint64), ("rows_skipped", C.c_uint64),
                ("max_imbalance", C.c_double)]


class Timing(C.Structure):
    _fields_ = [("sample_ms", C.c_float), ("core_ms", C.c_float), ("factor_ms", C.c_float),
                ("factor_mode_ms", C.c_float * MAX_ORDER), ("epochs", C.c_uint32)]


_lib = None


def lib_path() -> str:
    """libsgdt.so in-tree; SGDT_LIB overrides it (A/B builds of the same ABI)."""
    return os.environ.get("SGDT_LIB") or _build.LIB


def load(build_if_missing: bool = True):
    """Load libsgdt.so (building it in-tree first if it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not os.path.exists(path):
        if not build_if_missing or path != _build.LIB:
            raise ImportError(f"{path} is missing; run __graft_entry__.build()")
        _build.build()
    L = C.CDLL(path)
    vp = C.c_void_p
    u32p = C.POINTER(C.c_uint32)
    u64p = C.POINTER(C.c_uint64)
    dpp = C.POINTER(C.c_void_p)
    L.sgdt_last_error.restype = C.c_char_p
    L.sgdt_version.restype = C.c_char_p
    L.sgdt_session_create.argtypes = [C.POINTER(_TensorDesc), C.POINTER(_TensorDesc), u32p,
                                      C.c_uint32, C.c_int, C.POINTER(vp)]
    L.sgdt_session_destroy.argtypes = [vp]
    L.sgdt_session_stream.argtypes = [vp]
    L.sgdt_session_stream.restype = vp
    L.sgdt_set_model.argtypes = [vp, dpp, dpp]
    L.sgdt_get_model.argtypes = [vp, dpp, dpp]
    L.sgdt_set_rng.argtypes = [vp, u64p, C.c_uint32]
    L.sgdt_get_rng.argtypes = [vp, u64p, u32p]
    L.sgdt_reset_pool.argtypes = [vp]
    L.sgdt_sample_batch.argtypes = [vp, C.c_uint64, u32p]
    L.sgdt_last_batch.argtypes = [vp, u32p, u64p]
    L.sgdt_core_epoch.argtypes = [vp, C.POINTER(CoreHyper), C.POINTER(_CoreStats)]
    L.sgdt_factor_epoch.argtypes = [vp, C.POINTER(FactorHyper), C.POINTER(_FactorStats)]
    L.sgdt_run_epochs.argtypes = [vp, C.POINTER(CoreHyper), C.POINTER(FactorHyper), C.c_uint64]
    L.sgdt_run_epochs_host.argtypes = [vp, C.POINTER(CoreHyper), C.POINTER(FactorHyper), C.c_uint64, dpp, dpp, dpp, dpp]
    L.sgdt_eval.argtypes = [vp, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double)]
    L.sgdt_train.argtypes = [vp, C.POINTER(CoreHyper), C.POINTER(FactorHyper), C.c_uint64,
                             C.POINTER(C.c_double)]
    L.sgdt_last_timing.argtypes = [vp, C.POINTER(Timing)]
    L.sgdt_launch_count.argtypes = [vp]
    L.sgdt_launch_count.restype = C.c_uint64
    L.sgdt_rng_next_below.argtypes = [u64p, C.c_uint32, u64p, C.c_uint64, u64p, u64p, u32p]
    L.sgdt_partition_even.argtypes = [C.c_uint64, C.c_uint64, u64p, u64p]
    L.sgdt_split_ids.argtypes = [C.c_uint64, C.c_double, C.c_uint64, C.c_int, u32p, u32p]
    L.sgdt_synth.argtypes = [C.POINTER(SynthSpec), C.c_int, u32p, C.POINTER(C.c_double)]
    _lib = L
    return L


def _ck(rc: int) -> None:
    if rc != 0:
        msg = _lib.sgdt_last_error().decode(errors="replace")
        raise _ERRORS.get(rc, InternalError)(msg)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


def mt19937_64_state(seed: int) -> tuple[np.ndarray, int]:
    """State of a freshly seeded std::mt19937_64 (what Rng(seed) holds, rng.hpp:15)."""
    x = [0] * 312
    x[0] = seed & 0xFFFFFFFFFFFFFFFF
    for i in range(1, 312):
        x[i] = (6364136223846793005 * (x[i - 1] ^ (x[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
    return np.array(x, np.uint64), 312


def partition_even(count: int, workers: int):
    """partition_even (scheduler.cpp:34-46) through the C-ABI."""
    load()
    b = np.empty(workers, np.uint64)
    e = np.empty(workers, np.uint64)
    _lib.sgdt_partition_even(count, workers, _p(b, C.c_uint64), _p(e, C.c_uint64))
    return list(zip(b.tolist(), e.tolist()))


def split_ids(nnz: int, test_fraction: float, seed: int, device: int = -1):
    """train_test_split's id halves (sptensor.cpp:217-254) on the device:
    returns (test_ids, train_ids), each sorted ascending."""
    load()
    ntest = int(round(test_fraction * nnz)) if 0.0 < test_fraction < 1.0 else 0
    te = np.empty(max(ntest, 1), np.uint32)
    tr = np.empty(max(nnz - ntest, 1), np.uint32)
    _ck(_lib.sgdt_split_ids(nnz, test_fraction, seed, device, _p(te, C.c_uint32), _p(tr, C.c_uint32)))
    return te[:ntest], tr[: nnz - ntest]


class SynthSpec(C.Structure):
    _fields_ = [("order", C.c_int), ("dims", C.POINTER(C.c_uint32)), ("zipf", C.POINTER(C.c_double)),
                ("nnz", C.c_uint64), ("teacher_j", C.c_uint32), ("teacher_r", C.c_uint32),
                ("ratings", C.c_int), ("noise", C.c_double), ("seed", C.c_uint64)]


def synth(dims, zipf, nnz: int, teacher_j: int, teacher_r: int, ratings: bool, noise: float, seed: int,
          device: int = -1):
    """sgdt_synth: the config 2-5 tensor generated on the device; returns host
    (coords uint32 [nnz, N] 1-based, values f64 [nnz]) in linear-position order."""
    load()
    d = np.ascontiguousarray(dims, np.uint32)
    z = np.ascontiguousarray(zipf, np.float64)
    spec = SynthSpec(len(d), _p(d, C.c_uint32), _p(z, C.c_double), nnz, teacher_j, teacher_r,
                     1 if ratings else 0, noise, seed)
    coords = np.empty((nnz, len(d)), np.uint32)
    values = np.empty(nnz, np.float64)
    _ck(_lib.sgdt_synth(C.byref(spec), device, _p(coords, C.c_uint32), _p(values, C.c_double)))
    return coords, values


def rng_next_below(state: np.ndarray, pos: int, bounds: np.ndarray):
    """Device Rng::next_below over an explicit state; returns (values, state, pos)."""
    load()
    state = np.ascontiguousarray(state, np.uint64)
    bounds = np.ascontiguousarray(bounds, np.uint64)
    out = np.empty(len(bounds), np.uint64)
    st2 = np.empty(312, np.uint64)
    p2 = C.c_uint32()
    _ck(_lib.sgdt_rng_next_below(_p(state, C.c_uint64), pos, _p(bounds, C.c_uint64), len(bounds),
                                 _p(out, C.c_uint64), _p(st2, C.c_uint64), C.byref(p2)))
    return out, st2, p2.value


class _Tensor:
    """Host buffers of one CooTensor kept alive for the C-ABI call."""

    def __init__(self, dims, coords, values, perms=None):
        self.dims = np.ascontiguousarray(dims, np.uint32)
        self.order = len(self.dims)
        self.coords = np.ascontiguousarray(coords, np.uint32).reshape(-1)
        self.values = np.ascontiguousarray(values, np.float64)
        self.perms = None
        if perms is not None:
            self.perms = [np.ascontiguousarray(p, np.uint32) for p in perms]
            self._pp = (C.POINTER(C.c_uint32) * MAX_ORDER)(*[_p(p, C.c_uint32) for p in self.perms])
        self.desc = _TensorDesc(self.order, _p(self.dims, C.c_uint32), len(self.values),
                                _p(self.coords, C.c_uint32), _p(self.values, C.c_double),
                                C.cast(self._pp, C.POINTER(C.POINTER(C.c_uint32))) if perms is not None else None)


class Session:
    """A device-resident training session (one GPU).

    train/test: (dims, coords[nnz, N] 1-based, values[nnz] fp64[, perms]).
    """

    def __init__(self, dims, coords, values, J, R, test=None, perms=None, device=-1):
        load()
        self._tr = _Tensor(dims, coords, values, perms)
        self._te = _Tensor(dims, *test) if test is not None else None
        self.order = self._tr.order
        self.dims = [int(d) for d in self._tr.dims]
        self.J = np.ascontiguousarray(J, np.uint32)
        self.R = int(R)
        self.nnz = len(self._tr.values)
        h = C.c_void_p()
        _ck(_lib.sgdt_session_create(C.byref(self._tr.desc),
                                     C.byref(self._te.desc) if self._te else None,
                                     _p(self.J, C.c_uint32), self.R, device, C.byref(h)))
        self.h = h
        # drop host copies of the big arrays once uploaded
        self._tr = None
        self._te = None

    def close(self):
        if getattr(self, "h", None):
            _lib.sgdt_session_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return _lib.sgdt_session_stream(self.h)

    # ---- model / rng -----------------------------------------------------
    def set_model(self, A, B) -> None:
        A = [np.ascontiguousarray(a, np.float64) for a in A]
        B = [np.ascontiguousarray(b, np.float64) for b in B]
        pa = (C.c_void_p * MAX_ORDER)(*[a.ctypes.data for a in A])
        pb = (C.c_void_p * MAX_ORDER)(*[b.ctypes.data for b in B])
        _ck(_lib.sgdt_set_model(self.h, pa, pb))

    def get_model(self, out=None):
        if out is None:
            A = [np.empty((self.dims[n], int(self.J[n]))) for n in range(self.order)]
            B = [np.empty((int(self.J[n]), self.R)) for n in range(self.order)]
        else:
            A, B = out
        pa = (C.c_void_p * MAX_ORDER)(*[a.ctypes.data for a in A])
        pb = (C.c_void_p * MAX_ORDER)(*[b.ctypes.data for b in B])
        _ck(_lib.sgdt_get_model(self.h, pa, pb))
        return A, B

    def q_rows(self, n: int, lo: int = 0, hi: int | None = None) -> np.ndarray:
        """Rows [lo, hi) of the device's Kruskal rows Q^(n) = A^(n) B^(n) (fp32)."""
        hi = self.dims[n] if hi is None else hi
        out = np.empty((hi - lo, self.R), np.float32)
        _lib.sgdt_q_rows.argtypes = [C.c_void_p, C.c_int, C.c_uint32, C.c_uint32, C.c_void_p]
        _ck(_lib.sgdt_q_rows(self.h, n, lo, hi, out.ctypes.data_as(C.c_void_p)))
        return out

    def set_rng(self, state: np.ndarray, pos: int) -> None:
        state = np.ascontiguousarray(state, np.uint64)
        _ck(_lib.sgdt_set_rng(self.h, _p(state, C.c_uint64), pos))

    def seed(self, seed: int) -> None:
        self.set_rng(*mt19937_64_state(seed))

    def get_rng(self):
        st = np.empty(312, np.uint64)
        pos = C.c_uint32()
        _ck(_lib.sgdt_get_rng(self.h, _p(st, C.c_uint64), C.byref(pos)))
        return st, pos.value

    def reset_pool(self) -> None:
        _ck(_lib.sgdt_reset_pool(self.h))

    # ---- hot path ----------------------------------------------------------
    def sample_batch(self, m: int) -> np.ndarray:
        out = np.empty(m, np.uint32)
        _ck(_lib.sgdt_sample_batch(self.h, m, _p(out, C.c_uint32)))
        return out

    def last_batch(self) -> np.ndarray:
        n = C.c_uint64()
        _ck(_lib.sgdt_last_batch(self.h, None, C.byref(n)))
        out = np.empty(n.value, np.uint32)
        _ck(_lib.sgdt_last_batch(self.h, _p(out, C.c_uint32), C.byref(n)))
        return out

    def core_epoch(self, lr, reg, batch_m, resample=False, incremental=False):
        st = _CoreStats()
        _ck(_lib.sgdt_core_epoch(self.h, C.byref(CoreHyper(lr, reg, batch_m, int(resample),
                                                           int(incremental))), C.byref(st)))
        return st.batch_size, st.effective_workers

    def factor_epoch(self, lr, reg, row_fraction=1.0):
        st = _FactorStats()
        _ck(_lib.sgdt_factor_epoch(self.h, C.byref(FactorHyper(lr, reg, row_fraction)), C.byref(st)))
        return st.rows_updated, st.rows_skipped

    def run_epochs(self, core: CoreHyper, factor: FactorHyper, epochs: int = 1) -> None:
        _ck(_lib.sgdt_run_epochs(self.h, C.byref(core), C.byref(factor), epochs))

    def run_epochs_host(self, core: CoreHyper, factor: FactorHyper, epochs: int, model_in, model_out=None):
        """sgdt_run_epochs_host: host fp64 model in, `epochs` epochs, host fp64
        model out (model_out may be model_in; pinned buffers copy fastest)."""
        A, B = model_in
        for x in list(A) + list(B):
            if x.dtype != np.float64 or not x.flags.c_contiguous:
                raise DataError("run_epochs_host: model arrays must be C-contiguous float64")
        if model_out is None:
            model_out = ([np.empty_like(a) for a in A], [np.empty_like(b) for b in B])
        oA, oB = model_out
        ptrs = lambda xs: (C.c_void_p * MAX_ORDER)(*[x.ctypes.data for x in xs])
        _ck(_lib.sgdt_run_epochs_host(self.h, C.byref(core), C.byref(factor), epochs, ptrs(A), ptrs(B), ptrs(oA),
                                      ptrs(oB)))
        return oA, oB

    def eval(self, which: int = 0):
        a, b = C.c_double(), C.c_double()
        _ck(_lib.sgdt_eval(self.h, which, C.byref(a), C.byref(b)))
        return a.value, b.value

    def train(self, core: CoreHyper, factor: FactorHyper, epochs: int) -> np.ndarray:
        out = np.zeros(epochs * 6)
        _ck(_lib.sgdt_train(self.h, C.byref(core), C.byref(factor), epochs, _p(out, C.c_double)))
        return out.reshape(epochs, 6)

    def launch_count(self) -> int:
        return int(_lib.sgdt_launch_count(self.h))

    def last_timing(self) -> Timing:
        t = Timing()
        _ck(_lib.sgdt_last_timing(self.h, C.byref(t)))
        return t

"""ctypes front end for the TEST-ONLY oracle libraries.

* ``Oracle``  -> oracle/_build/libsgdt_oracle.so: the plain-C restatement of the
  reference algorithm (oracle/sgdt_oracle.c).
* ``RefLib``  -> oracle/_ref/libsptucker_ref.so: the unmodified reference
  sources from /root/reference/proj compiled with our POD bridge
  (oracle/ref_bridge.cpp).  Only present where it was built.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this module.  It is the checker, never the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libsgdt_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsptucker_ref.so")
REF_SRC = "/root/reference/proj"

MAX_ORDER = 8
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build_oracle(ref: bool | None = None) -> None:
    """Compile the C restatement (and the reference bridge when the reference
    sources are present, or when ref=True)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref is None:
        ref = os.path.isdir(REF_SRC)
    if ref:
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)
        if os.path.exists(os.path.join(HERE, "..", "paper_2012_03550_b200", "lib", "libsptucker_b200.so")):
            subprocess.run(["make", "-s", "-C", HERE, "acceptance"], check=True)


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: code {code}")
        self.code = code


def _ck(rc: int, what: str) -> None:
    if rc != 0:
        raise OracleError(rc, what)


# --------------------------------------------------------------------------
# plain-C oracle
# --------------------------------------------------------------------------
class _Rng(C.Structure):
    _fields_ = [("mt", C.c_uint64 * 312), ("idx", C.c_uint32), ("has_spare", C.c_int),
                ("spare", C.c_double)]


class _Tensor(C.Structure):
    _fields_ = [("order", C.c_int), ("dims", C.c_uint32 * MAX_ORDER), ("nnz", C.c_size_t),
                ("coords", C.POINTER(C.c_uint32)), ("values", C.POINTER(C.c_double)),
                ("perm", C.POINTER(C.c_uint32) * MAX_ORDER),
                ("offsets", C.POINTER(C.c_uint64) * MAX_ORDER)]


class _Model(C.Structure):
    _fields_ = [("order", C.c_int), ("dims", C.c_uint32 * MAX_ORDER),
                ("J", C.c_uint32 * MAX_ORDER), ("R", C.c_uint32),
                ("A", C.POINTER(C.c_double) * MAX_ORDER), ("B", C.POINTER(C.c_double) * MAX_ORDER),
                ("core_elems", C.c_uint64), ("core", C.POINTER(C.c_double)),
                ("unfold", C.POINTER(C.c_double) * MAX_ORDER)]


class _CoreHyper(C.Structure):
    _fields_ = [("lr", C.c_double), ("reg", C.c_double), ("batch_m", C.c_size_t),
                ("resample_per_mode", C.c_int), ("incremental_residual", C.c_int)]


class _FactorHyper(C.Structure):
    _fields_ = [("lr", C.c_double), ("reg", C.c_double), ("row_fraction", C.c_double)]


class _CoreWs(C.Structure):
    _fields_ = [("pool", C.POINTER(C.c_uint32)), ("pool_valid", C.c_int),
                ("batch", C.POINTER(C.c_uint32)), ("batch_len", C.c_size_t)]


class _Hyper(C.Structure):
    _fields_ = [("lr_a", C.c_double), ("lr_b", C.c_double), ("reg_a", C.c_double),
                ("reg_b", C.c_double), ("batch_m", C.c_size_t), ("row_fraction", C.c_double),
                ("epochs", C.c_size_t), ("seed", C.c_uint64), ("init_mean", C.c_double),
                ("init_stddev", C.c_double), ("resample_core_batch", C.c_int),
                ("incremental_residual", C.c_int)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build_oracle(ref=False)
        L = C.CDLL(ORACLE_SO)
        L.or_rng_seed.argtypes = [C.POINTER(_Rng), C.c_uint64]
        L.or_rng_next.argtypes = [C.POINTER(_Rng)]
        L.or_rng_next.restype = C.c_uint64
        L.or_next_below.argtypes = [C.POINTER(_Rng), C.c_uint64]
        L.or_next_below.restype = C.c_uint64
        L.or_next_gaussian.argtypes = [C.POINTER(_Rng), C.c_double, C.c_double]
        L.or_next_gaussian.restype = C.c_double
        L.or_mt_outputs.argtypes = [C.c_uint64, C.c_size_t, u64p]
        L.or_tensor_init.argtypes = [C.POINTER(_Tensor), C.c_int, u32p, C.c_size_t, u32p, f64p]
        L.or_tensor_free.argtypes = [C.POINTER(_Tensor)]
        L.or_model_init.argtypes = [C.POINTER(_Model), C.c_int, u32p, u32p, C.c_uint32]
        L.or_model_free.argtypes = [C.POINTER(_Model)]
        L.or_model_init_gaussian.argtypes = [C.POINTER(_Model), C.c_double, C.c_double,
                                             C.c_uint64]
        L.or_model_refresh_core.argtypes = [C.POINTER(_Model)]
        L.or_model_predict.argtypes = [C.POINTER(_Model), u32p]
        L.or_model_predict.restype = C.c_double
        L.or_sample_batch.argtypes = [C.c_size_t, C.c_size_t, C.POINTER(_Rng),
                                      C.POINTER(C.c_uint32), C.POINTER(C.c_int), u32p]
        L.or_core_ws_init.argtypes = [C.POINTER(_CoreWs), C.c_size_t]
        L.or_core_ws_free.argtypes = [C.POINTER(_CoreWs)]
        L.or_update_core_epoch.argtypes = [C.POINTER(_Model), C.POINTER(_Tensor),
                                           C.POINTER(_CoreHyper), C.POINTER(_Rng),
                                           C.POINTER(_CoreWs)]
        L.or_update_factor_epoch.argtypes = [C.POINTER(_Model), C.POINTER(_Tensor),
                                             C.POINTER(_FactorHyper), C.POINTER(_Rng),
                                             C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]
        L.or_rmse_mae.argtypes = [C.POINTER(_Model), C.POINTER(_Tensor), C.POINTER(C.c_double),
                                  C.POINTER(C.c_double)]
        L.or_train.argtypes = [C.POINTER(_Model), C.POINTER(_Tensor), C.POINTER(_Tensor),
                               C.POINTER(_Hyper), f64p]
        L.or_synth_planted.argtypes = [C.c_int, u32p, u32p, C.c_uint32, C.c_size_t, C.c_double,
                                       C.c_double, C.c_double, C.c_uint64, u32p, f64p]
        L.or_train_test_split_ids.argtypes = [C.c_size_t, C.c_double, C.c_uint64, u32p,
                                              C.POINTER(C.c_size_t)]
        _lib = L
    return _lib


class Rng:
    """std::mt19937_64-backed Rng (rng.hpp:13-49), C restatement."""

    def __init__(self, seed: int):
        self.s = _Rng()
        lib().or_rng_seed(C.byref(self.s), C.c_uint64(seed))

    def next_u64(self) -> int:
        return lib().or_rng_next(C.byref(self.s))

    def next_below(self, bound: int) -> int:
        return lib().or_next_below(C.byref(self.s), C.c_uint64(bound))

    def next_gaussian(self, mean: float, sd: float) -> float:
        return lib().or_next_gaussian(C.byref(self.s), mean, sd)

    def state(self) -> tuple[np.ndarray, int]:
        """(312-word MT state, index) -- the state the device sampler imports."""
        return np.array(self.s.mt[:], dtype=np.uint64), int(self.s.idx)


def mt_outputs(seed: int, n: int) -> np.ndarray:
    out = np.empty(n, np.uint64)
    lib().or_mt_outputs(seed, n, out)
    return out


class Tensor:
    """CooTensor (sptensor.hpp:66-107): 1-based coords, fp64 values, per-mode perms."""

    def __init__(self, dims, coords: np.ndarray, values: np.ndarray):
        self.dims = np.ascontiguousarray(dims, np.uint32)
        self.order = len(self.dims)
        self.coords = np.ascontiguousarray(coords, np.uint32).reshape(-1, self.order)
        self.values = np.ascontiguousarray(values, np.float64)
        self.t = _Tensor()
        _ck(lib().or_tensor_init(C.byref(self.t), self.order, self.dims, len(self.values),
                                 self.coords.reshape(-1), self.values), "or_tensor_init")

    @property
    def nnz(self) -> int:
        return len(self.values)

    def perm(self, n: int) -> np.ndarray:
        return np.ctypeslib.as_array(self.t.perm[n], (self.nnz,)).copy()

    def offsets(self, n: int) -> np.ndarray:
        return np.ctypeslib.as_array(self.t.offsets[n], (int(self.dims[n]) + 1,)).copy()

    def __del__(self):
        if getattr(self, "t", None) is not None and _lib is not None:
            _lib.or_tensor_free(C.byref(self.t))
            self.t = None


class Model:
    """TuckerModel (model.hpp:40-91), fp64, with dense core cache."""

    def __init__(self, dims, J, R: int):
        self.dims = np.ascontiguousarray(dims, np.uint32)
        self.J = np.ascontiguousarray(J, np.uint32)
        self.R = int(R)
        self.order = len(self.dims)
        self.m = _Model()
        _ck(lib().or_model_init(C.byref(self.m), self.order, self.dims, self.J, self.R),
            "or_model_init")

    def A(self, n: int) -> np.ndarray:
        """Live view of A^(n) (I_n x J_n)."""
        return np.ctypeslib.as_array(self.m.A[n], (int(self.dims[n]), int(self.J[n])))

    def B(self, n: int) -> np.ndarray:
        """Live view of B^(n) (J_n x R)."""
        return np.ctypeslib.as_array(self.m.B[n], (int(self.J[n]), self.R))

    def init_gaussian(self, mean: float, sd: float, seed: int) -> "Model":
        _ck(lib().or_model_init_gaussian(C.byref(self.m), mean, sd, seed), "init_gaussian")
        return self

    def set_params(self, A, B) -> None:
        for n in range(self.order):
            self.A(n)[...] = A[n]
            self.B(n)[...] = B[n]
        lib().or_model_refresh_core(C.byref(self.m))

    def params(self):
        return ([self.A(n).copy() for n in range(self.order)],
                [self.B(n).copy() for n in range(self.order)])

    def copy(self) -> "Model":
        out = Model(self.dims, self.J, self.R)
        out.set_params(*self.params())
        return out

    def predict(self, coord) -> float:
        return lib().or_model_predict(C.byref(self.m), np.ascontiguousarray(coord, np.uint32))

    def __del__(self):
        if getattr(self, "m", None) is not None and _lib is not None:
            _lib.or_model_free(C.byref(self.m))
            self.m = None


class CoreWorkspace:
    def __init__(self, nnz: int):
        self.ws = _CoreWs()
        _ck(lib().or_core_ws_init(C.byref(self.ws), nnz), "core_ws_init")

    def batch(self) -> np.ndarray:
        return np.ctypeslib.as_array(self.ws.batch, (self.ws.batch_len,)).copy()

    def __del__(self):
        if getattr(self, "ws", None) is not None and _lib is not None:
            _lib.or_core_ws_free(C.byref(self.ws))
            self.ws = None


def sample_batch(nnz: int, m: int, rng: Rng, ws: CoreWorkspace) -> np.ndarray:
    out = np.empty(m, np.uint32)
    valid = C.c_int(ws.ws.pool_valid)
    _ck(lib().or_sample_batch(nnz, m, C.byref(rng.s), ws.ws.pool, C.byref(valid), out),
        "sample_batch")
    ws.ws.pool_valid = valid.value
    return out


def update_core_epoch(model: Model, t: Tensor, lr, reg, batch_m, rng: Rng, ws: CoreWorkspace,
                      resample=False, incremental=False) -> None:
    h = _CoreHyper(lr, reg, batch_m, int(resample), int(incremental))
    _ck(lib().or_update_core_epoch(C.byref(model.m), C.byref(t.t), C.byref(h), C.byref(rng.s),
                                   C.byref(ws.ws)), "update_core_epoch")


def update_factor_epoch(model: Model, t: Tensor, lr, reg, rng: Rng, row_fraction=1.0):
    h = _FactorHyper(lr, reg, row_fraction)
    up, sk = C.c_size_t(), C.c_size_t()
    _ck(lib().or_update_factor_epoch(C.byref(model.m), C.byref(t.t), C.byref(h),
                                     C.byref(rng.s), C.byref(up), C.byref(sk)),
        "update_factor_epoch")
    return up.value, sk.value


def rmse_mae(model: Model, t: Tensor):
    a, b = C.c_double(), C.c_double()
    _ck(lib().or_rmse_mae(C.byref(model.m), C.byref(t.t), C.byref(a), C.byref(b)), "rmse_mae")
    return a.value, b.value


def train(model: Model, tr: Tensor, te: Tensor | None, *, lr_a, lr_b, reg_a, reg_b, batch_m,
          epochs, seed, row_fraction=1.0, resample=False, incremental=False) -> np.ndarray:
    h = _Hyper(lr_a, lr_b, reg_a, reg_b, batch_m, row_fraction, epochs, seed, 0.5, 0.1,
               int(resample), int(incremental))
    out = np.zeros(epochs * 4, np.float64)
    _ck(lib().or_train(C.byref(model.m), C.byref(tr.t), C.byref(te.t) if te else None,
                       C.byref(h), out), "train")
    return out.reshape(epochs, 4)


def synth_planted(dims, tJ, tR, nnz, noise, tmean=0.5, tsd=0.1, seed=1):
    dims = np.ascontiguousarray(dims, np.uint32)
    order = len(dims)
    coords = np.empty(nnz * order, np.uint32)
    values = np.empty(nnz, np.float64)
    _ck(lib().or_synth_planted(order, dims, np.ascontiguousarray(tJ, np.uint32), tR, nnz, noise,
                               tmean, tsd, seed, coords, values), "synth_planted")
    return coords.reshape(nnz, order), values


def train_test_split(dims, coords, values, frac, seed):
    """(train_coords, train_values, test_coords, test_values), sptensor.cpp:217-254."""
    nnz = len(values)
    ids = np.empty(nnz, np.uint32)
    nt = C.c_size_t()
    _ck(lib().or_train_test_split_ids(nnz, frac, seed, ids, C.byref(nt)), "train_test_split")
    te, tr = ids[: nt.value], ids[nt.value:]
    return coords[tr], values[tr], coords[te], values[te]


# --------------------------------------------------------------------------
# the reference itself, compiled from source (optional)
# --------------------------------------------------------------------------
_ref = None


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            raise FileNotFoundError(REF_SO)
        L = C.CDLL(REF_SO)
        vp, ip = C.c_void_p, C.POINTER(C.c_int)
        L.ref_mt_outputs.argtypes = [C.c_uint64, C.c_size_t, u64p]
        L.ref_next_below_seq.argtypes = [C.c_uint64, C.c_size_t, u64p, u64p]
        L.ref_gaussian_seq.argtypes = [C.c_uint64, C.c_size_t, C.c_double, C.c_double, f64p]
        L.ref_synth_planted.argtypes = [C.c_int, u32p, u32p, C.c_uint32, C.c_size_t, C.c_double,
                                        C.c_double, C.c_double, C.c_uint64, u32p, f64p]
        L.ref_tensor_new.argtypes = [C.c_int, u32p, C.c_size_t, u32p, f64p, ip]
        L.ref_tensor_new.restype = vp
        L.ref_tensor_free.argtypes = [vp]
        L.ref_tensor_perm.argtypes = [vp, C.c_int, u32p, u64p]
        L.ref_train_test_split.argtypes = [vp, C.c_double, C.c_uint64, u32p, f64p, u32p, f64p]
        L.ref_model_new.argtypes = [C.c_int, u32p, u32p, C.c_uint32, ip]
        L.ref_model_new.restype = vp
        L.ref_model_free.argtypes = [vp]
        L.ref_model_init_gaussian.argtypes = [vp, C.c_double, C.c_double, C.c_uint64]
        L.ref_model_params.argtypes = [vp, C.c_int, C.POINTER(C.c_void_p), C.POINTER(C.c_void_p)]
        L.ref_model_predict.argtypes = [vp, u32p]
        L.ref_model_predict.restype = C.c_double
        L.ref_rng_new.argtypes = [C.c_uint64]
        L.ref_rng_new.restype = vp
        L.ref_rng_free.argtypes = [vp]
        L.ref_sample_batch.argtypes = [vp, vp, C.c_size_t, u32p]
        L.ref_core_epoch.argtypes = [vp, vp, vp, C.c_double, C.c_double, C.c_size_t, C.c_int,
                                     C.c_int, C.c_int, C.c_size_t, C.c_void_p]
        L.ref_factor_epoch.argtypes = [vp, vp, vp, C.c_double, C.c_double, C.c_double, C.c_int,
                                       C.c_size_t, C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]
        L.ref_rmse_mae.argtypes = [vp, vp, C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_train_from_scratch.argtypes = [vp, vp, u32p, C.c_uint32, C.c_double, C.c_double,
                                             C.c_double, C.c_double, C.c_size_t, C.c_double,
                                             C.c_size_t, C.c_uint64, C.c_double, C.c_double,
                                             C.c_int, C.c_size_t, vp, f64p]
        L.ref_bench_epoch_seconds.argtypes = [vp, u32p, C.c_uint32, C.c_double, C.c_double,
                                              C.c_double, C.c_size_t, C.c_int, C.c_size_t,
                                              C.c_size_t, C.c_size_t, C.c_uint64,
                                              C.POINTER(C.c_double)]
        L.ref_time_epochs.argtypes = [vp, u32p, C.c_uint32, C.c_double, C.c_double, C.c_double, C.c_size_t,
                                      C.c_int, C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint64, C.c_double,
                                      C.c_double, C.POINTER(C.c_double)]
        L.ref_time_epochs_budget.argtypes = [vp, u32p, C.c_uint32, C.c_double, C.c_double, C.c_double,
                                             C.c_size_t, C.c_int, C.c_size_t, C.c_size_t, C.c_size_t, C.c_uint64,
                                             C.c_double, C.c_double, C.c_double, f64p, C.POINTER(C.c_size_t),
                                             C.POINTER(C.c_size_t)]
        _ref = L
    return _ref


STRATEGY = {"serial": 0, "naive": 1, "improved": 2}


class RefTensor:
    def __init__(self, dims, coords, values):
        self.dims = np.ascontiguousarray(dims, np.uint32)
        self.order = len(self.dims)
        self.coords = np.ascontiguousarray(coords, np.uint32).reshape(-1)
        self.values = np.ascontiguousarray(values, np.float64)
        rc = C.c_int()
        self.h = ref().ref_tensor_new(self.order, self.dims, len(self.values), self.coords,
                                      self.values, C.byref(rc))
        _ck(rc.value, "ref_tensor_new")

    @property
    def nnz(self):
        return len(self.values)

    def perm(self, n):
        p = np.empty(self.nnz, np.uint32)
        o = np.empty(int(self.dims[n]) + 1, np.uint64)
        _ck(ref().ref_tensor_perm(self.h, n, p, o), "ref_tensor_perm")
        return p, o

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_tensor_free(self.h)
            self.h = None


class RefModel:
    def __init__(self, dims, J, R):
        self.dims = np.ascontiguousarray(dims, np.uint32)
        self.J = np.ascontiguousarray(J, np.uint32)
        self.R = int(R)
        self.order = len(self.dims)
        rc = C.c_int()
        self.h = ref().ref_model_new(self.order, self.dims, self.J, self.R, C.byref(rc))
        _ck(rc.value, "ref_model_new")

    def init_gaussian(self, mean, sd, seed):
        _ck(ref().ref_model_init_gaussian(self.h, mean, sd, seed), "init_gaussian")
        return self

    def _ptrs(self, arrs):
        return (C.c_void_p * MAX_ORDER)(*[a.ctypes.data for a in arrs])

    def set_params(self, A, B):
        A = [np.ascontiguousarray(a, np.float64) for a in A]
        B = [np.ascontiguousarray(b, np.float64) for b in B]
        _ck(ref().ref_model_params(self.h, 0, self._ptrs(A), self._ptrs(B)), "params")

    def params(self):
        A = [np.empty((int(self.dims[n]), int(self.J[n]))) for n in range(self.order)]
        B = [np.empty((int(self.J[n]), self.R)) for n in range(self.order)]
        _ck(ref().ref_model_params(self.h, 1, self._ptrs(A), self._ptrs(B)), "params")
        return A, B

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_model_free(self.h)
            self.h = None


class RefRng:
    def __init__(self, seed):
        self.h = ref().ref_rng_new(seed)

    def __del__(self):
        if getattr(self, "h", None) and _ref is not None:
            _ref.ref_rng_free(self.h)
            self.h = None


def ref_rmse_mae(model: RefModel, t: RefTensor):
    a, b = C.c_double(), C.c_double()
    _ck(ref().ref_rmse_mae(model.h, t.h, C.byref(a), C.byref(b)), "ref_rmse_mae")
    return a.value, b.value

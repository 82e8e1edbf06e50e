"""TEST INFRASTRUCTURE ONLY: numpy restatement of the device generator
sgdt_synth (paper_2012_03550_b200/csrc/sgdt_synth.cu) for the BASELINE config
2-5 tensors.  The reference has no such generator (synth.cpp:16-103 draws
uniform positions with a Gaussian teacher); SURVEY.md 8(d) specifies this one:
Zipf indices by inverse CDF, first draw wins, ascending linear position
(synth.cpp:40), unit-variance Kruskal teacher, ratings or Gaussian noise.

Only tests/ use it, as the checker of sgdt_synth at small sizes: indices and
their order bit-exact, values to fp64 rounding (device pow/log/cos and FMA
contraction differ from libm/numpy in the last bits).
"""
from __future__ import annotations

import math

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = 0x9E3779B9, 0xBB67AE85
TAG_DRAW, TAG_TEACHER, TAG_NOISE = 0x5A1F0000, 0x7EAC0000, 0x00150000
CDF_BLOCK = 1024
SUM_CHUNK = 4096
MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32_10(c0, c1, c2, c3, k0: int, k1: int):
    """Philox4x32-10 (Salmon et al., SC'11) over uint32 arrays."""
    c = [np.asarray(x, np.uint64) & MASK32 for x in (c0, c1, c2, c3)]
    c = [np.broadcast_to(x, np.broadcast(*c).shape).copy() for x in c]
    k0 &= 0xFFFFFFFF
    k1 &= 0xFFFFFFFF
    for i in range(10):
        if i:
            k0 = (k0 + W0) & 0xFFFFFFFF
            k1 = (k1 + W1) & 0xFFFFFFFF
        p0 = M0 * c[0]
        p1 = M1 * c[2]
        c = [(p1 >> np.uint64(32)) ^ c[1] ^ np.uint64(k0), p1 & MASK32,
             (p0 >> np.uint64(32)) ^ c[3] ^ np.uint64(k1), p0 & MASK32]
    return c


def unit53(hi, lo):
    return ((hi << np.uint64(32)) | lo) >> np.uint64(11)


def _u53(hi, lo):
    return unit53(hi, lo).astype(np.float64) * 2.0 ** -53


def zipf_cdf(I: int, s: float) -> np.ndarray:
    w = np.power(np.arange(1, I + 1, dtype=np.float64), -s)
    nb = (I + CDF_BLOCK - 1) // CDF_BLOCK
    pad = np.zeros(nb * CDF_BLOCK)
    pad[:I] = w
    within = np.cumsum(pad.reshape(nb, CDF_BLOCK), axis=1)  # sequential per block
    tot = within[:, -1].copy()
    off = np.zeros(nb)
    acc = 0.0
    for b in range(nb):  # sequential exclusive scan of the block totals
        off[b] = acc
        acc += tot[b]
    cdf = (off[:, None] + within).reshape(-1)[:I]
    return cdf / acc


def draw_indices(dims, zipf, d: np.ndarray, seed: int, cdfs):
    out = []
    for k, (I, s) in enumerate(zip(dims, zipf)):
        r = philox4x32_10(d & 0xFFFFFFFF, d >> 32, k, TAG_DRAW, seed, seed >> 32)
        u = _u53(r[0], r[1])
        if s == 0.0:
            v = np.minimum((u * I).astype(np.uint64), I - 1)
        else:
            v = np.minimum(np.searchsorted(cdfs[k], u, side="right"), I - 1)
        out.append(v.astype(np.int64))
    return out


def normal_at(e: np.ndarray, stream: int, tag: int, seed: int) -> np.ndarray:
    r = philox4x32_10(e & 0xFFFFFFFF, e >> 32, stream, tag, seed, seed >> 32)
    u1, u2 = _u53(r[0], r[1]), _u53(r[2], r[3])
    return np.sqrt(-2.0 * np.log(1.0 - u1)) * np.cos(6.283185307179586 * u2)


def synth(dims, zipf, nnz: int, J: int, R: int, ratings: bool, noise: float, seed: int):
    """(coords uint32 [nnz, N] 1-based, values f64 [nnz]) exactly as sgdt_synth."""
    N = len(dims)
    cdfs = [zipf_cdf(I, s) if s != 0.0 else None for I, s in zip(dims, zipf)]
    keys: dict[int, int] = {}
    order: list[int] = []
    d0, batch = 0, max(4 * nnz, 1024)
    while len(order) < nnz:  # first draw wins
        d = np.arange(d0, d0 + batch, dtype=np.uint64)
        idx = draw_indices(dims, zipf, d, seed, cdfs)
        for q in range(batch):
            key, stride = 0, 1
            for k in range(N):
                key += int(idx[k][q]) * stride
                stride *= dims[k]
            if key not in keys:
                keys[key] = d0 + q
                order.append(key)
                if len(order) == nnz:
                    break
        d0 += batch
    kept = sorted(order)
    coords = np.empty((nnz, N), np.uint32)
    for e, key in enumerate(kept):
        for k in range(N):
            coords[e, k] = key % dims[k] + 1
            key //= dims[k]
    sigma = (J * R ** (1.0 / N)) ** -0.25
    Q = []
    for k in range(N):
        A = sigma * normal_at(np.arange(dims[k] * J, dtype=np.uint64), 16 + 2 * k, TAG_TEACHER, seed)
        B = sigma * normal_at(np.arange(J * R, dtype=np.uint64), 17 + 2 * k, TAG_TEACHER, seed)
        A = A.reshape(dims[k], J)
        B = B.reshape(J, R)
        q = np.zeros((dims[k], R))
        for j in range(J):  # j ascending, as the device
            q += A[:, j:j + 1] * B[j:j + 1, :]
        Q.append(q)
    x = np.zeros(nnz)
    for r in range(R):
        c = np.ones(nnz)
        for k in range(N):
            c = c * Q[k][coords[:, k].astype(np.int64) - 1, r]
        x = x + c
    if ratings:
        def chunked(v):
            acc = 0.0
            for c0 in range(0, len(v), SUM_CHUNK):
                acc += float(np.cumsum(v[c0:c0 + SUM_CHUNK])[-1])
            return acc
        mean = chunked(x) / nnz
        sd = math.sqrt(chunked((x - mean) ** 2) / (nnz - 1))
        v = np.clip(np.rint(3.0 + (x - mean) / sd), 1.0, 5.0)
    elif noise > 0.0:
        v = x + noise * normal_at(np.arange(nnz, dtype=np.uint64), 99, TAG_NOISE, seed)
    else:
        v = x
    return coords, v


# ---------------------------------------------------------------- host C++
# oracle/synth_host.cpp: the same generator on all host threads, for sizes the
# numpy restatement cannot reach (bench.py's reference arm builds the full
# config tensor with it, without loading any product library).
_host = None


def _host_lib():
    global _host
    if _host is None:
        import ctypes as C
        import os
        so = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_build", "libsynth_host.so")
        L = C.CDLL(so)
        u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
        f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        L.sh_synth.argtypes = [C.c_int, u32p, f64p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_int, C.c_double,
                               C.c_uint64, C.c_int, u32p, f64p]
        L.sh_synth.restype = C.c_int
        _host = L
    return _host


def synth_host(dims, zipf, nnz: int, J: int, R: int, ratings: bool, noise: float, seed: int, threads: int = 0):
    """Same result as synth() (and sgdt_synth), computed by synth_host.cpp."""
    d = np.ascontiguousarray(dims, np.uint32)
    z = np.ascontiguousarray(zipf, np.float64)
    coords = np.empty((nnz, len(dims)), np.uint32)
    values = np.empty(nnz, np.float64)
    rc = _host_lib().sh_synth(len(dims), d, z, nnz, J, R, int(ratings), noise, seed, threads, coords, values)
    if rc != 0:
        raise ValueError(f"sh_synth failed with code {rc}")
    return coords, values


def split_ids_host(nnz: int, test_fraction: float, seed: int):
    """(test_ids, train_ids) of train_test_split, by synth_host.cpp's
    sh_split_ids (the reference's Fisher-Yates with Rng(seed), both halves
    ascending)."""
    import ctypes as C
    L = _host_lib()
    u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
    L.sh_split_ids.argtypes = [C.c_uint64, C.c_double, C.c_uint64, u32p, u32p]
    L.sh_split_ids.restype = C.c_uint64
    ntest = int(round(test_fraction * nnz))
    te = np.empty(max(ntest, 1), np.uint32)
    tr = np.empty(max(nnz - ntest, 1), np.uint32)
    got = L.sh_split_ids(nnz, test_fraction, seed, te, tr)
    if got == 0:
        raise ValueError("degenerate split")
    return te[:got], tr[:nnz - got]

"""Synthetic stand-ins for the BASELINE configs that the reference generator
cannot produce ("C2-C5 need a new generator").

Input preparation only (never inside a timed region): torch is used as plumbing
to draw and sort on the device.  The reference's own generator (synth_planted,
synth.cpp:16-67: uniform distinct positions sorted by linear position, planted
Tucker teacher) is what config 1 uses; configs 2-5 need Zipf indices and a
unit-variance teacher, built here with the same conventions:
  * indices: bounded-support Zipf(s) by inverse CDF on 1..I_n (rank 1 hottest)
    or uniform, per mode;
  * duplicates dropped keeping the first draw, until exactly `nnz` distinct;
  * entries sorted by linear position (mode 1 fastest), as draw_positions does
    (synth.cpp:40);
  * teacher A^(n), B^(n) i.i.d. N(0, sigma^2), sigma = (J R^(1/N))^(-1/4), so
    that xhat has unit variance (Var = R (J sigma^4)^N);
  * config 2 values: xhat affinely mapped to mean 3 / std 1, rounded to an
    integer and clipped to [1, 5] (ratings);  configs 3-5: xhat + N(0, noise^2).
The 90/10 split is the reference's train_test_split (Fisher-Yates with
Rng(seed + 7), both halves in entry order), computed on the device by
sgdt_split_ids.
No dataset is fetched or reproduced: Netflix/MovieLens/Yahoo are not here.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch


@dataclasses.dataclass
class SynthSpec:
    dims: tuple
    zipf: tuple            # per mode: exponent s, or 0.0 for uniform
    nnz: int
    teacher_j: int
    teacher_r: int
    values: str = "gauss"  # "ratings" (C2) or "gauss"
    noise: float = 0.01
    seed: int = 1
    test_fraction: float = 0.1

    @property
    def order_count(self) -> int:
        return len(self.dims)

    @property
    def unit_sigma(self) -> float:
        """Teacher / init scale giving xhat unit variance: (J R^(1/N))^(-1/4)."""
        return (self.teacher_j * self.teacher_r ** (1.0 / len(self.dims))) ** -0.25


CONFIGS = {
    2: SynthSpec(dims=(480000, 17800, 2200), zipf=(1.1, 1.1, 0.0), nnz=100_000_000, teacher_j=10,
                 teacher_r=10, values="ratings"),
    3: SynthSpec(dims=(1_000_000, 1_000_000, 100_000, 50), zipf=(1.05, 1.05, 1.05, 0.0),
                 nnz=500_000_000, teacher_j=8, teacher_r=8, noise=0.05),
    4: SynthSpec(dims=(100_000, 100_000, 100_000, 100_000, 1000), zipf=(0.0,) * 5,
                 nnz=50_000_000, teacher_j=16, teacher_r=16, noise=0.01),
    5: SynthSpec(dims=(10_000_000, 10_000_000, 1000), zipf=(1.1, 1.1, 0.0), nnz=250_000_000,
                 teacher_j=32, teacher_r=32, noise=0.01),
}


def _draw_mode(I: int, s: float, count: int, gen: torch.Generator, device) -> torch.Tensor:
    """0-based indices in [0, I): Zipf(s) by inverse CDF (rank 1 hottest) or uniform."""
    if s == 0.0:
        return torch.randint(0, I, (count,), generator=gen, device=device, dtype=torch.int64)
    w = torch.arange(1, I + 1, device=device, dtype=torch.float64).pow_(-s)
    cdf = torch.cumsum(w, 0)
    cdf /= cdf[-1].clone()
    u = torch.rand(count, generator=gen, device=device, dtype=torch.float64)
    return torch.searchsorted(cdf, u).clamp_(max=I - 1)


def _linear_key(idx, dims):
    key = torch.zeros_like(idx[0])
    stride = 1
    for k, d in enumerate(dims):
        key += idx[k] * stride
        stride *= d
    return key


def _unkey(key, dims):
    out = []
    for d in dims:
        out.append(key % d)
        key = key // d
    return out


def _draw_tuples_wide(spec: SynthSpec, device):
    """Index spaces beyond 2^63 cells (config 4): dedupe whole coordinate
    tuples; rows come back sorted lexicographically from the last mode, i.e.
    by linear position with mode 1 fastest."""
    gen = torch.Generator(device=device)
    gen.manual_seed(spec.seed)
    cols = None
    while True:
        batch = max(1 << 20, spec.nnz - (0 if cols is None else cols.shape[0]) + spec.nnz // 64)
        idx = torch.stack([_draw_mode(d, s, batch, gen, device) for d, s in zip(spec.dims, spec.zipf)], 1)
        cols = idx if cols is None else torch.cat([cols, idx])
        rev = cols.flip(1)
        uniq, inv = torch.unique(rev, dim=0, return_inverse=True)
        first = torch.full((uniq.shape[0],), cols.shape[0], dtype=torch.int64, device=device)
        first.scatter_reduce_(0, inv, torch.arange(cols.shape[0], device=device), reduce="amin")
        if uniq.shape[0] >= spec.nnz:
            keep = torch.sort(first).values[: spec.nnz]  # first occurrences in draw order
            sel = cols[keep].flip(1)
            order = torch.unique(sel, dim=0)  # lexicographic = linear position order
            return [order[:, spec.order_count - 1 - k] for k in range(spec.order_count)]


def draw_positions(spec: SynthSpec, device) -> torch.Tensor:
    """Exactly spec.nnz distinct linear keys, first-drawn wins, sorted."""
    gen = torch.Generator(device=device)
    gen.manual_seed(spec.seed)
    total = math.prod(spec.dims)
    assert total < 2**63
    keys = torch.empty(0, dtype=torch.int64, device=device)
    batch = max(1 << 20, spec.nnz // 2)
    while True:
        idx = [_draw_mode(d, s, batch, gen, device) for d, s in zip(spec.dims, spec.zipf)]
        keys = torch.cat([keys, _linear_key(idx, spec.dims)])
        del idx
        sk, perm = torch.sort(keys, stable=True)
        first = torch.ones_like(sk, dtype=torch.bool)
        first[1:] = sk[1:] != sk[:-1]
        if int(first.sum()) >= spec.nnz:
            pos = torch.sort(perm[first]).values[: spec.nnz]  # first occurrences, draw order
            out = torch.sort(keys[pos]).values
            del sk, perm, first, keys
            return out
        del sk, perm, first


def teacher(spec: SynthSpec, device):
    gen = torch.Generator(device=device)
    gen.manual_seed(spec.seed + 1000003)
    N = len(spec.dims)
    J, R = spec.teacher_j, spec.teacher_r
    sigma = (J * R ** (1.0 / N)) ** -0.25
    A = [torch.randn(d, J, generator=gen, device=device, dtype=torch.float64) * sigma for d in spec.dims]
    B = [torch.randn(J, R, generator=gen, device=device, dtype=torch.float64) * sigma for _ in spec.dims]
    return A, B


def generate(spec: SynthSpec, device="cuda", with_perms: bool = False):
    """Returns (train, test), each (coords u32 [nnz,N] 1-based, values f64) as
    torch tensors on `device`, plus (with_perms) the mode-sorted permutations
    of train (the session builds its own mode orders on the device, so
    callers normally leave them out)."""
    device = torch.device(device)
    if math.prod(spec.dims) >= 2**62:
        idx = _draw_tuples_wide(dataclasses.replace(spec), device)
    else:
        keys = draw_positions(spec, device)
        idx = _unkey(keys, spec.dims)
        del keys
    A, B = teacher(spec, device)
    Q = [a @ b for a, b in zip(A, B)]
    nnz = spec.nnz
    xhat = torch.empty(nnz, dtype=torch.float64, device=device)
    step = 1 << 24
    for s0 in range(0, nnz, step):
        prod = None
        for k in range(len(spec.dims)):
            rows = Q[k][idx[k][s0:s0 + step]]
            prod = rows if prod is None else prod * rows
        xhat[s0:s0 + step] = prod.sum(1)
    gen = torch.Generator(device=device)
    gen.manual_seed(spec.seed + 7)
    if spec.values == "ratings":
        v = 3.0 + (xhat - xhat.mean()) / xhat.std()
        v = torch.round(v).clamp_(1.0, 5.0)
    else:
        v = xhat + spec.noise * torch.randn(nnz, generator=gen, device=device, dtype=torch.float64)
    del xhat, Q
    coords = torch.stack([i.to(torch.int32) + 1 for i in idx], 1)
    del idx
    # the reference's split (sptensor.cpp:217-254: Fisher-Yates with
    # Rng(seed), both halves sorted), run on the device by sgdt_split_ids
    from . import sgdt
    te_ids, tr_ids = sgdt.split_ids(nnz, spec.test_fraction, spec.seed + 7,
                                    device.index if device.type == "cuda" and device.index is not None else -1)
    te = torch.from_numpy(te_ids.astype(np.int64)).to(device)
    tr = torch.from_numpy(tr_ids.astype(np.int64)).to(device)
    del te_ids, tr_ids
    train = (coords[tr], v[tr])
    test = (coords[te], v[te])
    del coords, v
    perms = None
    if with_perms:
        perms = [torch.sort(train[0][:, n], stable=True).indices.to(torch.int32) for n in range(len(spec.dims))]
    return train, test, perms


def scaled(spec: SynthSpec, factor: float, nnz: int) -> SynthSpec:
    """Same distributions on a smaller index space (parity-scale instances)."""
    dims = tuple(max(2, int(round(d * factor))) for d in spec.dims)
    return dataclasses.replace(spec, dims=dims, nnz=nnz)

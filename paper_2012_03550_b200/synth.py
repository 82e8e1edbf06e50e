"""Synthetic stand-ins for the BASELINE configs that the reference generator
cannot produce ("C2-C5 need a new generator").

Input preparation only (never inside a timed region).  The reference's own
generator (synth_planted, synth.cpp:16-67: uniform distinct positions sorted
by linear position, planted Tucker teacher) is what config 1 uses; configs
2-5 need Zipf indices and a unit-variance teacher, drawn on the device by
sgdt_synth (csrc/sgdt_synth.cu, checked against oracle/synth_oracle.py):
  * indices: bounded-support Zipf(s) by inverse CDF on 1..I_n (rank 1
    hottest) or uniform, per mode, from Philox4x32-10 streams;
  * duplicates dropped keeping the first draw, exactly `nnz` distinct;
  * entries sorted by linear position (mode 1 fastest), as draw_positions does
    (synth.cpp:40);
  * teacher A^(n), B^(n) i.i.d. N(0, sigma^2), sigma = (J R^(1/N))^(-1/4), so
    that xhat has unit variance (Var = R (J sigma^4)^N);
  * config 2 values: xhat standardised to mean 3 / std 1, rounded to an
    integer and clipped to [1, 5] (ratings);  configs 3-5: xhat + N(0, noise^2).
The 90/10 split is the reference's train_test_split (Fisher-Yates with
Rng(seed + 7), both halves in entry order), computed on the device by
sgdt_split_ids.
No dataset is fetched or reproduced: Netflix/MovieLens/Yahoo are not here.
"""
from __future__ import annotations

import dataclasses

import numpy as np


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


def generate(spec: SynthSpec, device="cuda", with_perms: bool = False):
    """Returns (train, test), each (coords uint32 [nnz, N] 1-based, values f64)
    as host arrays, plus (with_perms) the mode-sorted permutations of train
    (the session builds its own mode orders on the device, so callers
    normally leave them out).  The tensor is drawn by sgdt_synth on the
    device (csrc/sgdt_synth.cu); the 90/10 split is the reference's
    train_test_split (sptensor.cpp:217-254: Fisher-Yates with Rng(seed + 7),
    both halves in entry order), also on the device (sgdt_split_ids)."""
    import torch

    from . import sgdt
    dev = torch.device(device) if not isinstance(device, int) else torch.device("cuda", device)
    index = -1 if dev.type != "cuda" else (dev.index if dev.index is not None else torch.cuda.current_device())
    coords, v = sgdt.synth(spec.dims, spec.zipf, spec.nnz, spec.teacher_j, spec.teacher_r,
                           spec.values == "ratings", spec.noise, spec.seed, device=index)
    te_ids, tr_ids = sgdt.split_ids(spec.nnz, spec.test_fraction, spec.seed + 7, index)
    train = (coords[tr_ids], v[tr_ids])
    test = (coords[te_ids], v[te_ids])
    del coords, v
    perms = None
    if with_perms:
        perms = [np.argsort(train[0][:, n], kind="stable").astype(np.uint32) for n in range(len(spec.dims))]
    return train, test, perms


def scaled(spec: SynthSpec, factor: float, nnz: int) -> SynthSpec:
    """Same distributions on a smaller index space (parity-scale instances)."""
    dims = tuple(max(2, int(round(d * factor))) for d in spec.dims)
    return dataclasses.replace(spec, dims=dims, nnz=nnz)

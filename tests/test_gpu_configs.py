"""Value parity at the BASELINE configurations (SURVEY.md
8(c): "parity is shown on scaled-down instances with identical N, J, R and
distributions").

* Scaled instances of configs 2-5, drawn by the device generator sgdt_synth
  with each config's order, Zipf exponents, teacher ranks and value model
  (config 2: integer ratings; 3-5: Gaussian teacher + noise), 20k-300k
  nonzeros, M scaled with nnz.  Two teacher-forced epochs against the pinned
  C oracle: Psi bit-exact, B^(n) after the core phase and A^(n) after the
  factor phase within rel_err 1e-4 (|g - ref| / max(1, |ref|),
  oracle.cpp:409-411).  Config 4 keeps N = 5 with J = R = 10 (16^5 exceeds
  the dense-core cap of the oracle and the reference, model.hpp:25).
* The full-size config 2 tensor (90M training nonzeros, Zipf head rows of
  millions of entries) against the reference itself (oracle/_ref, the
  unmodified sources, Strategy::Improved on every host thread): one
  teacher-forced epoch (Psi bit-exact, B and A within 1e-4), then two
  free-run epochs from the same start on both sides, test RMSE within 1e-3
  (test_trainer.cpp:175-222 is the reference's own fast-vs-literal check).
"""
import os

import numpy as np
import pytest

from oracle import oracle_py as O

pytestmark = pytest.mark.gpu

TOL = 1e-4
LR = REG = 0.01


def sg():
    from paper_2012_03550_b200 import sgdt
    return sgdt


def rel_err(g, ref):
    g = np.asarray(g, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(g - ref) / np.maximum(1.0, np.abs(ref)))) if g.size else 0.0


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def scaled_spec(cfg, nnz, J=None, dims=None):
    """The config's distributions on a smaller index space: every dim scaled
    by (nnz / nnz_config)^(1/N) (same density), or explicit dims."""
    import dataclasses
    from paper_2012_03550_b200 import synth
    spec = synth.CONFIGS[cfg]
    factor = (nnz / spec.nnz) ** (1.0 / len(spec.dims))
    sp = synth.scaled(spec, factor, nnz)
    if dims is not None:
        sp = dataclasses.replace(sp, dims=tuple(dims))
    if J is not None:
        sp = dataclasses.replace(sp, teacher_j=J, teacher_r=J)
    return sp


def init_moments(cfg, sp):
    # the bench's initialisation (bench.py init_stats)
    return (0.3, 0.1) if cfg == 2 else (0.0, sp.unit_sigma)


def fp32_model(dims, J, R, mean, sd, seed):
    m = O.Model(dims, J, R).init_gaussian(mean, sd, seed)
    A, B = m.params()
    m.set_params([f32(a) for a in A], [f32(b) for b in B])
    return m


# config, nnz, J (None: the config's), M, dims (None: density-preserving).
# Config 4 keeps its ~450 entries per row in modes 1-4 (and 45,000 in mode 5)
# instead of its density: at 20k entries the density-preserving shape
# (20913^4 x 209) leaves one entry per row, where lr 0.01 diverges in the
# reference itself (NumericError from the oracle's first factor epoch).
# The "rows" instances keep the config's mean entries per row instead of its
# density (dims = I_n x nnz / nnz_config): on the density-preserving config 3
# shape (~1.4 entries per row) free-run SGD at lr 0.01 diverges in the
# reference too (oracle: NumericError in epoch 2), so the free runs use these.
SCALED = [
    (2, 300_000, None, 2048, None),
    (3, 200_000, None, 1024, None),
    (3, 200_000, None, 1024, (444, 444, 44, 2)),
    (4, 20_000, 10, 256, (44, 44, 44, 44, 2)),
    (5, 60_000, None, 512, None),
    (5, 60_000, None, 512, (2667, 2667, 2)),
]
IDS = ["config2", "config3", "config3_rows", "config4_rows", "config5", "config5_rows"]


@pytest.mark.parametrize("cfg,nnz,J,M,dims", SCALED, ids=IDS)
def test_scaled_config_teacher_forced_parity(cfg, nnz, J, M, dims):
    from paper_2012_03550_b200 import synth
    sp = scaled_spec(cfg, nnz, J, dims)
    (trc, trv), (tec, tev), _ = synth.generate(sp, 0)
    dims, order = sp.dims, len(sp.dims)
    Jv, R = (sp.teacher_j,) * order, sp.teacher_r
    # every instance has a row longer than one 2048-entry chunk (the
    # split-row path): a Zipf head row, or config 4's mode-5 rows
    counts = [np.bincount(trc[:, n], minlength=dims[n] + 1) for n in range(order)]
    assert max(int(c.max()) for c in counts) > 2048
    t = O.Tensor(dims, trc, trv)
    s = sg().Session(dims, trc, trv, Jv, R, test=(tec, tev))
    m = fp32_model(dims, Jv, R, *init_moments(cfg, sp), 23)
    rng = O.Rng(2)
    ws = O.CoreWorkspace(len(trv))
    s.set_rng(*rng.state())
    for epoch in range(2):
        s.set_model(*m.params())
        s.core_epoch(LR, REG, M)
        O.update_core_epoch(m, t, LR, REG, M, rng, ws)
        assert np.array_equal(s.last_batch(), ws.batch()), f"Psi epoch {epoch}"
        A, B = s.get_model()
        RA, RB = m.params()
        for n in range(order):
            assert rel_err(B[n], RB[n]) <= TOL, f"config {cfg} core B^({n}) epoch {epoch}: {rel_err(B[n], RB[n])}"
        m.set_params([f32(a) for a in RA], [f32(b) for b in RB])
        s.set_model(*m.params())
        up, sk = s.factor_epoch(LR, REG)
        assert (up, sk) == O.update_factor_epoch(m, t, LR, REG, rng)
        A, B = s.get_model()
        RA, RB = m.params()
        for n in range(order):
            assert rel_err(A[n], RA[n]) <= TOL, f"config {cfg} factor A^({n}) epoch {epoch}: {rel_err(A[n], RA[n])}"
        m.set_params([f32(a) for a in RA], [f32(b) for b in RB])
        st, pos = s.get_rng()
        rst, rpos = rng.state()
        assert pos == rpos and np.array_equal(st, rst)
    # RMSE of the same (fp32-representable) model on the test split
    s.set_model(*m.params())
    got = s.eval(1)
    ref = O.rmse_mae(m, O.Tensor(dims, tec, tev))
    assert abs(got[0] - ref[0]) <= 1e-5 * max(1.0, ref[0]) and abs(got[1] - ref[1]) <= 1e-5 * max(1.0, ref[1])


FREE = [0, 2, 3, 5]


@pytest.mark.parametrize("cfg,nnz,J,M,dims", [SCALED[i] for i in FREE], ids=[IDS[i] for i in FREE])
def test_scaled_config_free_run_rmse(cfg, nnz, J, M, dims):
    """Three free-run epochs (the device's fp32 trajectory against the
    oracle's fp64 one from the same start): test RMSE within 1e-3 each epoch."""
    from paper_2012_03550_b200 import synth
    sp = scaled_spec(cfg, nnz, J, dims)
    (trc, trv), (tec, tev), _ = synth.generate(sp, 0)
    dims, order = sp.dims, len(sp.dims)
    Jv, R = (sp.teacher_j,) * order, sp.teacher_r
    m = fp32_model(dims, Jv, R, *init_moments(cfg, sp), 29)
    s = sg().Session(dims, trc, trv, Jv, R, test=(tec, tev))
    s.set_model(*m.params())
    s.seed(2)
    met = s.train(sg().CoreHyper(LR, REG, M, 0, 0), sg().FactorHyper(LR, REG, 1.0), 3)
    rng = O.Rng(2)
    ws = O.CoreWorkspace(len(trv))
    t, te = O.Tensor(dims, trc, trv), O.Tensor(dims, tec, tev)
    for e in range(3):
        O.update_core_epoch(m, t, LR, REG, M, rng, ws)
        O.update_factor_epoch(m, t, LR, REG, rng)
        assert abs(met[e, 4] - O.rmse_mae(m, te)[0]) <= 1e-3


@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref (the compiled reference) is not built")
def test_full_size_config2_against_reference():
    from paper_2012_03550_b200 import synth
    import ctypes as C
    sp = synth.CONFIGS[2]
    (trc, trv), (tec, tev), _ = synth.generate(sp, 0)
    dims, order, J, R, M = sp.dims, 3, (10, 10, 10), 10, 65536
    threads = os.cpu_count() or 1
    s = sg().Session(dims, trc, trv, J, R, test=(tec, tev))
    rt, rte = O.RefTensor(dims, trc, trv), O.RefTensor(dims, tec, tev)
    m0 = fp32_model(dims, J, R, 0.3, 0.1, 1)  # C oracle used only to draw the start
    A0, B0 = m0.params()
    rm = O.RefModel(dims, J, R)
    rm.set_params(A0, B0)
    rr = O.RefRng(2)
    s.seed(2)
    L = O.ref()
    # teacher-forced epoch: core phase
    s.set_model(A0, B0)
    s.core_epoch(LR, REG, M)
    psi = np.empty(M, np.uint32)
    assert L.ref_core_epoch(rm.h, rt.h, rr.h, LR, REG, M, 0, 0, O.STRATEGY["improved"], threads,
                            psi.ctypes.data_as(C.c_void_p)) == 0
    assert np.array_equal(s.last_batch(), psi)
    A, B = s.get_model()
    RA, RB = rm.params()
    for n in range(order):
        assert rel_err(B[n], RB[n]) <= TOL, f"core B^({n}): {rel_err(B[n], RB[n])}"
    # factor phase from the reference's state
    RA, RB = [f32(a) for a in RA], [f32(b) for b in RB]
    rm.set_params(RA, RB)
    s.set_model(RA, RB)
    s.factor_epoch(LR, REG)
    up, sk = C.c_size_t(), C.c_size_t()
    assert L.ref_factor_epoch(rm.h, rt.h, rr.h, LR, REG, 1.0, O.STRATEGY["improved"], threads,
                              C.byref(up), C.byref(sk)) == 0
    A, B = s.get_model()
    RA, RB = rm.params()
    for n in range(order):
        assert rel_err(A[n], RA[n]) <= TOL, f"factor A^({n}): {rel_err(A[n], RA[n])}"
    # free run: two more epochs on both sides from the same start
    RA, RB = [f32(a) for a in RA], [f32(b) for b in RB]
    rm.set_params(RA, RB)
    s.set_model(RA, RB)
    met = s.train(sg().CoreHyper(LR, REG, M, 0, 0), sg().FactorHyper(LR, REG, 1.0), 2)
    for e in range(2):
        assert L.ref_core_epoch(rm.h, rt.h, rr.h, LR, REG, M, 0, 0, O.STRATEGY["improved"], threads, None) == 0
        assert L.ref_factor_epoch(rm.h, rt.h, rr.h, LR, REG, 1.0, O.STRATEGY["improved"], threads,
                                  C.byref(up), C.byref(sk)) == 0
        ref_rmse = O.ref_rmse_mae(rm, rte)[0]
        assert abs(met[e, 4] - ref_rmse) <= 1e-3, (e, met[e, 4], ref_rmse)

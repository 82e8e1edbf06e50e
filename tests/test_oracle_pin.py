"""Pin the C oracle restatement against the reference itself (CPU only).

The reference (/root/reference/proj) is compiled from its own sources into
oracle/_ref/libsptucker_ref.so; every oracle routine must reproduce it
bit-for-bit (same fp64 operation order).  Where the reference build is absent
(the GPU box) these tests fall back to the committed golden fixtures, which were
produced by the reference (tests/golden/make_golden.py).
"""
import json
import os

import numpy as np
import pytest

from oracle import oracle_py as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built here")


def test_mt19937_64_known_answer():
    # [rand.predef]: the 10000th output of a default-constructed mt19937_64.
    out = O.mt_outputs(5489, 10000)
    assert int(out[-1]) == 9981545732273789042


@needs_ref
@pytest.mark.parametrize("seed", [0, 1, 2, 12345, 2**64 - 1])
def test_engine_matches_reference(seed):
    ref = np.empty(2000, np.uint64)
    O.ref().ref_mt_outputs(seed, 2000, ref)
    assert np.array_equal(O.mt_outputs(seed, 2000), ref)


@needs_ref
def test_next_below_and_gaussian_match_reference():
    rs = np.random.default_rng(3)
    bounds = np.concatenate([rs.integers(1, 2**32, 500, dtype=np.uint64),
                             np.array([1, 2, 3, 2**63 + 5, 2**64 - 1, 2**63], np.uint64)])
    ref = np.empty(len(bounds), np.uint64)
    O.ref().ref_next_below_seq(77, len(bounds), bounds, ref)
    r = O.Rng(77)
    mine = np.array([r.next_below(int(b)) for b in bounds], np.uint64)
    assert np.array_equal(mine, ref)
    g_ref = np.empty(501)
    O.ref().ref_gaussian_seq(9, 501, 0.5, 0.1, g_ref)
    r = O.Rng(9)
    g = np.array([r.next_gaussian(0.5, 0.1) for _ in range(501)])
    assert np.array_equal(g, g_ref)


SYNTH_CASES = [
    ((12, 10, 8), (2, 2, 2), 2, 180, 0.02, 0.5, 0.1, 54),
    ((30, 25), (3, 3), 3, 220, 0.01, 0.5, 0.1, 61),
    ((5, 4, 3, 3), (2, 2, 2, 2), 2, 100, 0.05, 0.0, 1.0, 7),
    ((1000, 800, 600), (5, 5, 5), 5, 3000, 0.01, 0.0, 1.0, 1),  # rejection branch
]


@needs_ref
@pytest.mark.parametrize("case", SYNTH_CASES)
def test_synth_planted_matches_reference(case):
    dims, tJ, tR, nnz, noise, tm, ts, seed = case
    c, v = O.synth_planted(dims, tJ, tR, nnz, noise, tm, ts, seed)
    rc = np.empty(nnz * len(dims), np.uint32)
    rv = np.empty(nnz)
    assert O.ref().ref_synth_planted(len(dims), np.array(dims, np.uint32),
                                     np.array(tJ, np.uint32), tR, nnz, noise, tm, ts, seed,
                                     rc, rv) == 0
    assert np.array_equal(c.reshape(-1), rc)
    assert np.array_equal(v, rv)


@needs_ref
def test_split_and_perms_match_reference():
    dims = (40, 30, 20)
    c, v = O.synth_planted(dims, (3, 3, 3), 3, 2000, 0.1, 0.5, 0.1, 5)
    rt = O.RefTensor(dims, c, v)
    ntest = int(round(0.1 * 2000))
    trc = np.empty((2000 - ntest) * 3, np.uint32)
    trv = np.empty(2000 - ntest)
    tec = np.empty(ntest * 3, np.uint32)
    tev = np.empty(ntest)
    assert O.ref().ref_train_test_split(rt.h, 0.1, 1, trc, trv, tec, tev) == 0
    a, b, cc, d = O.train_test_split(dims, c, v, 0.1, 1)
    assert np.array_equal(a.reshape(-1), trc) and np.array_equal(b, trv)
    assert np.array_equal(cc.reshape(-1), tec) and np.array_equal(d, tev)
    t = O.Tensor(dims, c, v)
    for n in range(3):
        p, o = rt.perm(n)
        assert np.array_equal(t.perm(n), p)
        assert np.array_equal(t.offsets(n), o)


@needs_ref
@pytest.mark.parametrize("m", [1, 7, 100, 500])
def test_sample_batch_matches_reference_with_persistent_pool(m):
    dims = (20, 20, 10)
    c, v = O.synth_planted(dims, (2, 2, 2), 2, 500, 0.0, 0.5, 0.1, 3)
    rt = O.RefTensor(dims, c, v)
    rr = O.RefRng(11)
    r = O.Rng(11)
    ws = O.CoreWorkspace(500)
    for _ in range(25):
        ref = np.empty(m, np.uint32)
        assert O.ref().ref_sample_batch(rr.h, rt.h, m, ref) == 0
        assert np.array_equal(O.sample_batch(500, m, r, ws), ref)


def _epoch_case(order_dims, J, R, nnz, batch_m, seed, resample=False, incremental=False,
                row_fraction=1.0, epochs=3):
    c, v = O.synth_planted(order_dims, J, R, nnz, 0.05, 0.5, 0.1, seed)
    t = O.Tensor(order_dims, c, v)
    rt = O.RefTensor(order_dims, c, v)
    m = O.Model(order_dims, J, R).init_gaussian(0.5, 0.2, seed + 100)
    rm = O.RefModel(order_dims, J, R)
    rm.set_params(*m.params())
    r, rr = O.Rng(seed + 1), O.RefRng(seed + 1)
    ws = O.CoreWorkspace(nnz)
    for _ in range(epochs):
        O.update_core_epoch(m, t, 0.02, 0.01, batch_m, r, ws, resample, incremental)
        assert O.ref().ref_core_epoch(rm.h, rt.h, rr.h, 0.02, 0.01, batch_m, int(resample),
                                      int(incremental), 0, 1, None) == 0
        A, B = m.params()
        RA, RB = rm.params()
        for n in range(len(order_dims)):
            assert np.array_equal(B[n], RB[n]) and np.array_equal(A[n], RA[n])
        O.update_factor_epoch(m, t, 0.02, 0.01, r, row_fraction)
        assert O.ref().ref_factor_epoch(rm.h, rt.h, rr.h, 0.02, 0.01, row_fraction, 0, 1,
                                        None, None) == 0
        A, B = m.params()
        RA, RB = rm.params()
        for n in range(len(order_dims)):
            assert np.array_equal(B[n], RB[n]) and np.array_equal(A[n], RA[n])
    assert O.rmse_mae(m, t) == O.ref_rmse_mae(rm, rt)


@needs_ref
@pytest.mark.parametrize("case", [
    dict(order_dims=(12, 10, 8), J=(3, 3, 3), R=2, nnz=300, batch_m=16, seed=1),
    dict(order_dims=(12, 10, 8), J=(3, 4, 3), R=3, nnz=300, batch_m=0, seed=2),
    dict(order_dims=(9, 7, 6, 5), J=(2, 3, 2, 2), R=2, nnz=400, batch_m=50, seed=3,
         resample=True),
    dict(order_dims=(30, 25), J=(3, 3), R=3, nnz=220, batch_m=20, seed=4, incremental=True),
    dict(order_dims=(15, 12, 10), J=(3, 3, 3), R=3, nnz=600, batch_m=32, seed=5,
         row_fraction=0.5),
])
def test_epochs_bit_identical_to_reference(case):
    _epoch_case(**case)


@needs_ref
def test_train_bit_identical_to_reference():
    dims = (40, 30, 20)
    c, v = O.synth_planted(dims, (3, 3, 3), 3, 3000, 0.01, 0.0, 1.0, 1)
    trc, trv, tec, tev = O.train_test_split(dims, c, v, 0.1, 1)
    tr, te = O.Tensor(dims, trc, trv), O.Tensor(dims, tec, tev)
    m = O.Model(dims, (3, 3, 3), 3).init_gaussian(0.5, 0.1, 1)
    mine = O.train(m, tr, te, lr_a=0.01, lr_b=0.01, reg_a=0.01, reg_b=0.01, batch_m=64,
                   epochs=4, seed=1)
    rtr, rte = O.RefTensor(dims, trc, trv), O.RefTensor(dims, tec, tev)
    rm = O.RefModel(dims, (3, 3, 3), 3)
    met = np.zeros(4 * 6)
    assert O.ref().ref_train_from_scratch(rtr.h, rte.h, np.array([3, 3, 3], np.uint32), 3, 0.01,
                                          0.01, 0.01, 0.01, 64, 1.0, 4, 1, 0.5, 0.1, 0, 1,
                                          rm.h, met) == 0
    met = met.reshape(4, 6)
    assert np.array_equal(mine, met[:, 2:])
    A, B = m.params()
    RA, RB = rm.params()
    for n in range(3):
        assert np.array_equal(A[n], RA[n]) and np.array_equal(B[n], RB[n])


def test_oracle_matches_committed_golden_vectors():
    """Golden vectors were produced by the reference itself (make_golden.py)."""
    path = os.path.join(GOLDEN, "config1.json")
    g = json.load(open(path))
    spec = g["spec"]
    c, v = O.synth_planted(spec["dims"], spec["tJ"], spec["tR"], spec["nnz"], spec["noise"],
                           spec["tmean"], spec["tsd"], spec["seed"])
    assert np.array_equal(c.reshape(-1)[:64], np.array(g["coords_head"], np.uint32))
    assert np.array_equal(v[:32], np.array(g["values_head"]))
    trc, trv, tec, tev = O.train_test_split(spec["dims"], c, v, 0.1, 1)
    tr, te = O.Tensor(spec["dims"], trc, trv), O.Tensor(spec["dims"], tec, tev)
    h = g["hyper"]
    ws = O.CoreWorkspace(tr.nnz)
    r = O.Rng(h["seed"] + 1)
    m = O.Model(spec["dims"], h["J"], h["R"]).init_gaussian(0.5, 0.1, h["seed"])
    for ep, psi_head in enumerate(g["psi_head"]):
        O.update_core_epoch(m, tr, h["lr_b"], h["reg_b"], h["batch_m"], r, ws)
        assert ws.batch()[: len(psi_head)].tolist() == psi_head
        O.update_factor_epoch(m, tr, h["lr_a"], h["reg_a"], r)
        rm_tr = O.rmse_mae(m, tr)
        rm_te = O.rmse_mae(m, te)
        assert rm_tr == (g["train_rmse"][ep], g["train_mae"][ep])
        assert rm_te == (g["test_rmse"][ep], g["test_mae"][ep])
    A, B = m.params()
    for n in range(3):
        assert float(A[n].sum()) == g["final_A_sum"][n]
        assert B[n].tolist() == g["final_B"][n]

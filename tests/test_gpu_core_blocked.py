"""The blocked core phase (sgdt_core_blocked.cu) and the sharded core phase
built on it, against the oracle's serial update_core_epoch.

Blocked: columns of B^(n) in blocks of T; one reduction of V0 and of the
in-block Gram terms per block, then T exact Gauss-Seidel column steps
(sgdt.h "sharded core phase").  T = 1 is the column algorithm, T = R one
reduction per mode.  Single GPU: SGDT_CORE=blocked (session-level switch),
SGDT_CORE_T picks T.  Sharded: ranks as threads on one GPU (each a sharded
session; the exchange slots are written with peer stores by the producing
kernel and ordered by host barriers -- no kernel waits on another), Psi
sliced by partition_even(M, P), slots summed in rank order.

Bars: Psi bit-exact, B^(n) within rel_err 1e-4 of the oracle (teacher
forced), every rank's B bit-identical, run-to-run bit-identical."""
import threading

import numpy as np
import pytest

from oracle import oracle_py as O

pytestmark = pytest.mark.gpu

TOL = 1e-4

CASES = [
    dict(dims=(12, 10, 8), J=(3, 3, 3), R=2, nnz=300, batch_m=16),
    dict(dims=(40, 30, 20), J=(5, 5, 5), R=5, nnz=5000, batch_m=256),
    dict(dims=(12, 10, 8), J=(3, 4, 3), R=3, nnz=300, batch_m=0),
    dict(dims=(9, 7, 6, 5), J=(2, 3, 2, 2), R=2, nnz=400, batch_m=50, resample=True),
    dict(dims=(8, 7, 6, 5, 4), J=(3, 3, 3, 3, 3), R=3, nnz=1500, batch_m=100),
    dict(dims=(50, 40, 30), J=(10, 10, 10), R=10, nnz=8000, batch_m=1024),
    dict(dims=(60, 50, 40), J=(8, 8, 8, 8)[:3], R=8, nnz=12000, batch_m=5000),
    dict(dims=(20, 20, 20), J=(16, 12, 16), R=12, nnz=3000, batch_m=300),
    dict(dims=(20, 20, 20), J=(32, 32, 32), R=32, nnz=3000, batch_m=300),
    dict(dims=(9, 8, 7, 6, 5), J=(10, 10, 10, 10, 10), R=10, nnz=3000, batch_m=256),
    dict(dims=(40, 30, 20), J=(64, 40, 37), R=32, nnz=6000, batch_m=700),
]


def cid(c):
    return "x".join(map(str, c["dims"])) + f"_R{c['R']}"


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def rel_err(g, ref):
    g, ref = np.asarray(g, np.float64), np.asarray(ref, np.float64)
    return float(np.max(np.abs(g - ref) / np.maximum(1.0, np.abs(ref)))) if g.size else 0.0


def unit_sigma(dims, J, R):
    return (min(J) * R ** (1.0 / len(dims))) ** -0.25


def setup(case, seed=17):
    dims, J, R, nnz = case["dims"], case["J"], case["R"], case["nnz"]
    sig = unit_sigma(dims, J, R)
    c, v = O.synth_planted(dims, J, min(J), nnz, 0.05, 0.0, sig, seed)
    m = O.Model(dims, J, R).init_gaussian(0.0, sig, 23)
    A, B = m.params()
    m.set_params([f32(a) for a in A], [f32(b) for b in B])
    return (c, v), m


def oracle_core(case, tr, m, rng, ws):
    t = O.Tensor(case["dims"], *tr)
    O.update_core_epoch(m, t, 0.01, 0.01, case["batch_m"], rng, ws, case.get("resample", False), False)
    return m.params()[1]


@pytest.mark.parametrize("T", ["1", "2", "5", "32"])
@pytest.mark.parametrize("case", CASES, ids=cid)
def test_blocked_core_teacher_forced(monkeypatch, case, T):
    from paper_2012_03550_b200 import sgdt
    monkeypatch.setenv("SGDT_CORE", "blocked")
    monkeypatch.setenv("SGDT_CORE_T", T)
    tr, m = setup(case)
    dims, J, R, bm = case["dims"], case["J"], case["R"], case["batch_m"]
    s = sgdt.Session(dims, tr[0], tr[1], J, R)
    rng = O.Rng(5)
    ws = O.CoreWorkspace(len(tr[1]))
    s.set_rng(*rng.state())
    for epoch in range(2):
        s.set_model(*m.params())
        s.core_epoch(0.01, 0.01, bm, case.get("resample", False), False)
        RB = oracle_core(case, tr, m, rng, ws)
        if bm:
            assert np.array_equal(s.last_batch(), ws.batch())
        _, B = s.get_model()
        for n in range(len(dims)):
            assert rel_err(B[n], RB[n]) <= TOL, f"B^({n}) epoch {epoch} T={T}"
        RA, RB = m.params()
        m.set_params([f32(a) for a in RA], [f32(b) for b in RB])
        st, pos = s.get_rng()
        rst, rpos = rng.state()
        assert pos == rpos and np.array_equal(st, rst)


def test_blocked_core_q_refresh_and_rerun_identical(monkeypatch):
    """The final step's Q^(k) = A^(k) B^(k) feeds the factor phase: a blocked
    epoch followed by a factor epoch matches the oracle, and reruns are
    bit-identical."""
    from paper_2012_03550_b200 import sgdt
    monkeypatch.setenv("SGDT_CORE", "blocked")
    case = CASES[5]
    tr, m = setup(case)
    dims, J, R, bm = case["dims"], case["J"], case["R"], case["batch_m"]
    t = O.Tensor(dims, *tr)
    start = m.params()
    outs = []
    for _ in range(2):
        s = sgdt.Session(dims, tr[0], tr[1], J, R)
        s.set_model(*start)
        s.seed(9)
        s.core_epoch(0.01, 0.01, bm)
        s.factor_epoch(0.01, 0.01)
        outs.append(s.get_model())
    for n in range(3):
        assert np.array_equal(outs[0][0][n], outs[1][0][n]) and np.array_equal(outs[0][1][n], outs[1][1][n])
    mo = O.Model(dims, J, R)
    mo.set_params(*start)
    rng = O.Rng(9)
    O.update_core_epoch(mo, t, 0.01, 0.01, bm, rng, O.CoreWorkspace(len(tr[1])))
    O.update_factor_epoch(mo, t, 0.01, 0.01, rng)
    RA, RB = mo.params()
    for n in range(3):
        assert rel_err(outs[0][1][n], RB[n]) <= TOL
        assert rel_err(outs[0][0][n], RA[n]) <= 5 * TOL  # one free-run epoch: core error feeds the factor pass


def run_sharded_core(case, world, block, tr, start, seed=5):
    from paper_2012_03550_b200 import distributed as D
    from paper_2012_03550_b200 import sgdt
    dims, J, R = case["dims"], case["J"], case["R"]
    groups = D.ThreadGroup.make(world)
    sess = [D.ShardedSession(dims, tr[0], tr[1], J, R, r, world) for r in range(world)]
    ch = sgdt.CoreHyper(0.01, 0.01, case["batch_m"], 1 if case.get("resample") else 0, 0)
    Ts, errs = [None] * world, []

    def body(r):
        try:
            sess[r].set_model(*start)
            sess[r].seed(seed)
            D.connect_peers(sess[r], groups[r])
            groups[r].barrier()
            Ts[r] = D.core_epoch_sharded(sess[r], groups[r], ch, block)
            sess[r].synchronize()
            sess[r].check()
        except Exception as e:  # surfaced below
            errs.append(e)
            raise

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    return [s.get_model()[1] for s in sess], Ts[0], sess


@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("block", [1, 3, 0])
@pytest.mark.parametrize("case", [CASES[1], CASES[3], CASES[5], CASES[8]], ids=cid)
def test_sharded_core_matches_oracle(case, world, block):
    tr, m = setup(case)
    start = m.params()
    Bs, T, _ = run_sharded_core(case, world, block, tr, start)
    for r in range(1, world):
        for n in range(len(case["dims"])):
            assert np.array_equal(Bs[r][n], Bs[0][n]), f"rank {r} B^({n}) differs"
    rng = O.Rng(5)
    RB = oracle_core(case, tr, m, rng, O.CoreWorkspace(len(tr[1])))
    for n in range(len(case["dims"])):
        assert rel_err(Bs[0][n], RB[n]) <= TOL, f"B^({n}) world={world} T={T}"


def test_sharded_epochs_p2p_with_sharded_core_match_oracle():
    """Whole epochs through run_epochs_p2p(core='sharded') on 2 thread ranks:
    B and A within the bars of one free-run epoch from the same start."""
    from paper_2012_03550_b200 import distributed as D
    from paper_2012_03550_b200 import sgdt
    case = CASES[5]
    tr, m = setup(case)
    dims, J, R, bm = case["dims"], case["J"], case["R"], case["batch_m"]
    start = m.params()
    world = 2
    groups = D.ThreadGroup.make(world)
    sess = [D.ShardedSession(dims, tr[0], tr[1], J, R, r, world) for r in range(world)]
    ch = sgdt.CoreHyper(0.01, 0.01, bm, 0, 0)
    fh = sgdt.FactorHyper(0.01, 0.01, 1.0)
    errs = []

    def body(r):
        try:
            sess[r].set_model(*start)
            sess[r].seed(9)
            D.connect_peers(sess[r], groups[r])
            groups[r].barrier()
            D.run_epochs_p2p(sess[r], groups[r], ch, fh, 1, core="sharded")
            sess[r].synchronize()
        except Exception as e:
            errs.append(e)
            raise

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    t = O.Tensor(dims, *tr)
    mo = O.Model(dims, J, R)
    mo.set_params(*start)
    rng = O.Rng(9)
    O.update_core_epoch(mo, t, 0.01, 0.01, bm, rng, O.CoreWorkspace(len(tr[1])))
    O.update_factor_epoch(mo, t, 0.01, 0.01, rng)
    RA, RB = mo.params()
    models = [s.get_model() for s in sess]
    for n in range(3):
        assert np.array_equal(models[0][1][n], models[1][1][n])
        assert np.max(np.abs(models[0][0][n] - models[1][0][n])) == 0.0
        assert rel_err(models[0][1][n], RB[n]) <= TOL
        assert rel_err(models[0][0][n], RA[n]) <= 5 * TOL

"""Size-independent properties at BASELINE config 2's full size (480,000 x
17,800 x 2,200, 90M training nonzeros, J = R = 10, M = 65,536), where the
oracle cannot run:
  * the persistent sample pool stays a permutation of 0..nnz-1 and every Psi
    is a set of distinct entry ids (sptensor.cpp:256-270);
  * the first Psi equals the first m draws of the reference's partial
    Fisher-Yates recomputed on the host for the drawn positions only;
  * epochs are run-to-run bit-identical (no atomics on parameters);
  * lr = 0 freezes both phases bit-exactly and consumes no RNG;
  * training reduces the train RMSE, and the test RMSE stays finite.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c2():
    from paper_2012_03550_b200 import synth
    train, test, perms = synth.generate(synth.CONFIGS[2], "cuda", with_perms=True)
    return dict(dims=synth.CONFIGS[2].dims, train=train, test=test, perms=perms)


def session(c2):
    from paper_2012_03550_b200 import sgdt
    s = sgdt.Session(c2["dims"], *c2["train"], [10, 10, 10], 10, test=c2["test"], perms=c2["perms"], device=0)
    rs = np.random.default_rng(1)
    B = [rs.normal(0.3, 0.1, (10, 10)) for _ in c2["dims"]]  # bench.init_stats(2)
    A = [rs.normal(0.3, 0.1, (d, 10)) for d in c2["dims"]]
    s.set_model(A, B)
    s.seed(2)
    return s


def test_pool_stays_a_permutation_and_batches_are_distinct(c2):
    from paper_2012_03550_b200 import sgdt
    s = session(c2)
    nnz = len(c2["train"][1])
    seen = []
    for _ in range(3):
        s.run_epochs(sgdt.CoreHyper(0.01, 0.01, 65536, 0, 0), sgdt.FactorHyper(0.01, 0.01, 1.0), 1)
        b = s.last_batch()
        assert len(b) == 65536 and len(np.unique(b)) == 65536 and b.max() < nnz
        seen.append(b)
    import ctypes as C
    pool = np.empty(nnz, np.uint32)
    sgdt._ck(sgdt.load().sgdt_get_pool(s.h, pool.ctypes.data_as(C.POINTER(C.c_uint32))))
    assert np.array_equal(np.sort(pool), np.arange(nnz, dtype=np.uint32))
    assert np.array_equal(pool[:65536], seen[-1])


def test_first_batch_matches_host_fisher_yates(c2):
    """Draws j_i = i + next_below(nnz - i) from Rng(2); the host replays the
    swaps lazily (a dict of touched positions) for the first 65,536 steps."""
    from oracle import oracle_py as O
    s = session(c2)
    nnz = len(c2["train"][1])
    got = s.sample_batch(65536)
    r = O.Rng(2)
    moved = {}
    want = np.empty(65536, np.uint32)
    for i in range(65536):
        j = i + r.next_below(nnz - i)
        vi, vj = moved.get(i, i), moved.get(j, j)
        moved[i], moved[j] = vj, vi
        want[i] = vj
    assert np.array_equal(got, want)
    st, pos = s.get_rng()
    rst, rpos = r.state()
    assert pos == rpos and np.array_equal(st, rst)


def test_epochs_are_run_to_run_bit_identical(c2):
    from paper_2012_03550_b200 import sgdt
    outs = []
    for _ in range(2):
        s = session(c2)
        s.run_epochs(sgdt.CoreHyper(0.01, 0.01, 65536, 0, 0), sgdt.FactorHyper(0.01, 0.01, 1.0), 2)
        outs.append(s.get_model())
        s.close()
    for n in range(3):
        assert np.array_equal(outs[0][0][n], outs[1][0][n]) and np.array_equal(outs[0][1][n], outs[1][1][n])


def test_lr_zero_is_a_bit_exact_freeze(c2):
    from paper_2012_03550_b200 import sgdt
    s = session(c2)
    A0, B0 = s.get_model()
    st0, p0 = s.get_rng()
    s.run_epochs(sgdt.CoreHyper(0.0, 0.01, 65536, 0, 0), sgdt.FactorHyper(0.0, 0.01, 1.0), 2)
    A1, B1 = s.get_model()
    st1, p1 = s.get_rng()
    assert p0 == p1 and np.array_equal(st0, st1)
    for n in range(3):
        assert np.array_equal(A0[n], A1[n]) and np.array_equal(B0[n], B1[n])


def test_training_reduces_rmse(c2):
    from paper_2012_03550_b200 import sgdt
    s = session(c2)
    r0 = s.eval(0)[0]
    met = s.train(sgdt.CoreHyper(0.01, 0.01, 65536, 0, 0), sgdt.FactorHyper(0.01, 0.01, 1.0), 3)
    assert met[-1, 2] < r0 and met[-1, 2] <= met[0, 2] + 1e-9
    assert np.all(np.isfinite(met[:, 4]))


def test_generated_config2_tensor_properties(c2):
    """sgdt_synth at full size (the oracle restatement is checked at small
    sizes in test_synth.py): distinct positions, ratings 1..5, the Zipf modes
    hottest at index 1, and the 90/10 split sizes of train_test_split."""
    dims = np.array(c2["dims"], np.int64)
    trc, trv = c2["train"]
    tec, tev = c2["test"]
    assert len(trv) == 90_000_000 and len(tev) == 10_000_000
    allc = np.concatenate([trc, tec]).astype(np.int64)
    assert allc.min() >= 1 and np.all(allc.max(0) <= dims)
    key = (allc[:, 0] - 1) + dims[0] * ((allc[:, 1] - 1) + dims[1] * (allc[:, 2] - 1))
    assert len(np.unique(key)) == len(key)
    assert set(np.unique(np.concatenate([trv, tev]))) <= {1.0, 2.0, 3.0, 4.0, 5.0}
    for n in (0, 1):  # Zipf(1.1) modes: index 1 holds the most entries
        counts = np.bincount(allc[:, n])
        assert counts[1] == counts.max()

"""The config 2-5 generator: sgdt_synth on the device
against its numpy restatement oracle/synth_oracle.py, plus the Philox4x32-10
known-answer vectors of Salmon et al. (Random123 kat_vectors) on the oracle."""
import numpy as np
import pytest

from oracle import synth_oracle as S


def test_philox_known_answers():
    kats = [((0, 0, 0, 0), (0, 0), (0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8)),
            ((0xffffffff,) * 4, (0xffffffff,) * 2, (0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd)),
            ((0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344), (0xa4093822, 0x299f31d0),
             (0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1))]
    for c, k, want in kats:
        got = S.philox4x32_10(*[np.uint64(x) for x in c], *k)
        assert tuple(int(x) for x in got) == want


def test_oracle_shape_and_distribution():
    dims = (400, 300, 20)
    c, v = S.synth(dims, (1.1, 1.1, 0.0), 5000, 10, 10, True, 0.0, 1)
    assert c.shape == (5000, 3) and c.min() >= 1 and (c.max(0) <= dims).all()
    key = (c[:, 0] - 1) + dims[0] * ((c[:, 1] - 1) + dims[1] * (c[:, 2] - 1).astype(np.int64))
    assert np.all(np.diff(key) > 0)  # distinct, ascending linear position
    assert set(np.unique(v)) <= {1.0, 2.0, 3.0, 4.0, 5.0}
    # Zipf: row 1 of mode 1 is the hottest
    assert np.bincount(c[:, 0])[1] == np.bincount(c[:, 0]).max()


SPECS = [
    dict(dims=(300, 200, 50), zipf=(1.1, 1.1, 0.0), nnz=20000, J=10, R=10, ratings=True, noise=0.0, seed=1),
    dict(dims=(500, 400, 60, 7), zipf=(1.05, 1.05, 1.05, 0.0), nnz=15000, J=8, R=8, ratings=False, noise=0.05,
         seed=3),
    dict(dims=(2000,) * 4 + (30,), zipf=(0.0,) * 5, nnz=8000, J=4, R=4, ratings=False, noise=0.01, seed=5),
    dict(dims=(10 ** 7, 10 ** 7, 1000), zipf=(1.1, 1.1, 0.0), nnz=6000, J=6, R=6, ratings=False, noise=0.01,
         seed=2),
    # index space beyond 2^64 (two-word keys), as BASELINE config 4
    dict(dims=(100000,) * 4 + (1000,), zipf=(0.0,) * 5, nnz=5000, J=3, R=3, ratings=False, noise=0.01, seed=9),
]


@pytest.mark.gpu
@pytest.mark.parametrize("spec", SPECS, ids=[str(i) for i in range(len(SPECS))])
def test_device_generator_matches_oracle(spec):
    from paper_2012_03550_b200 import sgdt
    args = (spec["dims"], spec["zipf"], spec["nnz"], spec["J"], spec["R"], spec["ratings"], spec["noise"],
            spec["seed"])
    c, v = sgdt.synth(*args, device=0)
    rc, rv = S.synth(*args)
    assert np.array_equal(c, rc)  # indices, dedup and order: bit-exact
    # values: device pow/log/cos and FMA contraction round differently
    assert np.allclose(v, rv, rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
def test_device_generator_errors():
    from paper_2012_03550_b200 import sgdt
    with pytest.raises(Exception):
        sgdt.synth((10, 10), (0.0, 0.0), 60, 2, 2, False, 0.0, 1)  # more than half the index space
    with pytest.raises(Exception):
        sgdt.synth((10,), (0.0,), 3, 2, 2, False, 0.0, 1)  # order 1


_NUMPY_CACHE = {}


def _numpy_synth(args):
    if args not in _NUMPY_CACHE:
        _NUMPY_CACHE[args] = S.synth(*args)
    return _NUMPY_CACHE[args]


@pytest.mark.parametrize("spec", SPECS, ids=[str(i) for i in range(len(SPECS))])
@pytest.mark.parametrize("threads", [1, 5])
def test_host_generator_matches_oracle(spec, threads):
    """oracle/synth_host.cpp (the bench reference arm's input generator) against
    the numpy restatement: indices bit-exact, values to fp64 rounding."""
    args = (spec["dims"], spec["zipf"], spec["nnz"], spec["J"], spec["R"], spec["ratings"], spec["noise"],
            spec["seed"])
    c, v = S.synth_host(*args, threads=threads)
    rc, rv = _numpy_synth(args)
    assert np.array_equal(c, rc)
    assert np.allclose(v, rv, rtol=1e-12, atol=1e-12)


def test_host_generator_errors():
    with pytest.raises(ValueError):
        S.synth_host((10, 10), (0.0, 0.0), 60, 2, 2, False, 0.0, 1)
    with pytest.raises(ValueError):
        S.synth_host((10, 10), (-1.0, 0.0), 5, 2, 2, False, 0.0, 1)


@pytest.mark.gpu
def test_host_generator_matches_device_at_scale():
    """A config-2-shaped tensor of 3M entries: host and device generators give
    the same positions in the same order (the reference arm trains on the
    host one, the GPU arm on the device one)."""
    from paper_2012_03550_b200 import sgdt
    args = ((48000, 1780, 2200), (1.1, 1.1, 0.0), 3_000_000, 10, 10, True, 0.0, 1)
    c, v = sgdt.synth(*args, device=0)
    hc, hv = S.synth_host(*args)
    assert np.array_equal(c, hc)
    assert np.mean(v != hv) < 1e-4  # ratings: a rounding tie may flip in a rare entry


@pytest.mark.parametrize("nnz,frac,seed", [(10, 0.1, 1), (1000, 0.25, 7), (200_003, 0.1, 8)])
def test_host_split_matches_oracle(nnz, frac, seed):
    from oracle import oracle_py as O
    import ctypes as C
    ids = np.empty(nnz, np.uint32)
    nt = C.c_size_t()
    assert O.lib().or_train_test_split_ids(nnz, frac, seed, ids, C.byref(nt)) == 0
    te, tr = S.split_ids_host(nnz, frac, seed)
    assert np.array_equal(te, ids[:nt.value]) and np.array_equal(tr, ids[nt.value:])

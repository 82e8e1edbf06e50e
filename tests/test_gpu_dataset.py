"""Device dataset build: the C-ABI session rejects
duplicate coordinates exactly as the reference CooTensor constructor does
(sptensor.cpp:90-100: DataError "entry <e>: duplicate coordinate" at the first
entry whose position was seen before), now checked on the device by a radix
sort of packed coordinate keys (sgdt_session.cu: check_duplicates)."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden", "io")


def sg():
    from paper_2012_03550_b200 import sgdt
    return sgdt


def first_duplicate(coords, dims):
    """The reference's answer: smallest entry id whose coordinates occur at a
    smaller id (the hash-set insert order of sptensor.cpp:90-100)."""
    _, first = np.unique(coords, axis=0, return_index=True)
    mask = np.ones(len(coords), bool)
    mask[first] = False
    dup = np.flatnonzero(mask)
    return int(dup[0]) if len(dup) else None


def load_tns(path):
    rows = [list(map(float, ln.split())) for ln in open(path) if ln.strip()]
    a = np.array(rows)
    return a[:, :-1].astype(np.uint32), a[:, -1]


@pytest.mark.parametrize("name,want", [("duplicate.tns", 2), ("duplicate_late.tns", 3)])
def test_reference_fixture_duplicates(name, want):
    c, v = load_tns(os.path.join(GOLD, name))
    dims = tuple(int(x) for x in c.max(0))
    with pytest.raises(sg().DataError, match=f"entry {want}: duplicate coordinate"):
        sg().Session(dims, c, v, (1,) * len(dims), 1)


@pytest.mark.parametrize("dims,nnz,seed", [
    ((300, 200, 100), 1_000_000, 1),                      # 23-bit keys, many collisions
    ((1000, 1000, 1000), 2_000_000, 2),                   # one 30-bit word
    ((100000, 100000, 100000, 100000, 1000), 300_000, 3),  # 78 bits: two sort passes (config 4's space)
    ((2 ** 32 - 1,) * 3, 200_000, 4),                     # 96 bits, full 32-bit fields
])
def test_first_duplicate_matches_reference_rule(dims, nnz, seed):
    rs = np.random.default_rng(seed)
    c = np.stack([rs.integers(1, min(d, 50) + 1 if nnz > 1_500_000 else d + 1, nnz, dtype=np.uint64)
                  for d in dims], 1).astype(np.uint32)
    if first_duplicate(c, dims) is None:  # plant two late repeats
        c[nnz - 5] = c[nnz // 3]
        c[nnz - 2] = c[7]
    want = first_duplicate(c, dims)
    with pytest.raises(sg().DataError, match=f"train: entry {want}: duplicate coordinate"):
        sg().Session(dims, c, np.ones(nnz), (2,) * len(dims), 2)


def test_distinct_tensor_accepted_and_test_tensor_checked():
    dims = (50, 40, 30)
    rs = np.random.default_rng(9)
    lin = rs.choice(50 * 40 * 30, 20000, replace=False)
    c = np.stack([lin % 50 + 1, lin // 50 % 40 + 1, lin // 2000 + 1], 1).astype(np.uint32)
    s = sg().Session(dims, c, np.ones(len(c)), (3, 3, 3), 3)  # no error
    del s
    te = c[:100].copy()
    te[60] = te[10]
    with pytest.raises(sg().DataError, match="test: entry 60: duplicate coordinate"):
        sg().Session(dims, c, np.ones(len(c)), (3, 3, 3), 3, test=(te, np.ones(100)))

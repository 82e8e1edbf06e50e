"""CPU checks of the C-ABI library: it loads, exports exactly the entry points
include/sgdt.h declares, and its pure-host helpers agree with the oracle.
No kernel is launched here (there is no GPU in the build container)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import oracle_py as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "sgdt.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sgdt_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2012_03550_b200 import sgdt
    return sgdt.load()


def test_library_exports_every_declared_symbol(lib):
    from paper_2012_03550_b200 import _build
    syms = declared_symbols()
    assert len(syms) >= 20
    for name in syms:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _build.LIB], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (sgdt_[a-z0-9_]+)$", out, flags=re.M))
    assert set(syms) <= exported


def test_library_is_sm100a_only():
    from paper_2012_03550_b200 import _build
    out = subprocess.run(["cuobjdump", "--list-elf", _build.LIB], capture_output=True,
                         text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_version_and_error_strings(lib):
    lib.sgdt_version.restype = C.c_char_p
    assert b"sm_100a" in lib.sgdt_version()


@pytest.mark.parametrize("count,workers", [(0, 1), (10, 3), (7, 16), (1024, 148), (5, 5)])
def test_partition_even_matches_reference(count, workers):
    from paper_2012_03550_b200 import sgdt
    got = sgdt.partition_even(count, workers)
    b = (C.c_size_t * workers)()
    e = (C.c_size_t * workers)()
    O.lib().or_partition_even.argtypes = [C.c_size_t, C.c_size_t, C.c_void_p, C.c_void_p]
    O.lib().or_partition_even(count, workers, b, e)
    assert got == list(zip(list(b), list(e)))


def test_mt_seed_state_matches_oracle():
    from paper_2012_03550_b200 import sgdt
    for seed in (0, 1, 2, 5489, 2**64 - 1):
        st, pos = sgdt.mt19937_64_state(seed)
        rst, rpos = O.Rng(seed).state()
        assert pos == rpos and np.array_equal(st, rst)


def test_session_without_gpu_fails_loudly(lib):
    """No silent CPU fallback: without a device the session call errors."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2012_03550_b200 import sgdt
    coords = np.array([[1, 1], [2, 1]], np.uint32)
    with pytest.raises(sgdt.SptuckerError):
        sgdt.Session((2, 1), coords, np.array([1.0, 2.0]), (1, 1), 1)

"""The I/O golden fixtures (tests/golden/io) are the reference's own output:
regenerate them through oracle/_ref (the unmodified reference sources, built
where /root/reference exists) and compare byte for byte.  The replay against
the C++ host API is tests/test_cpp_api.py (test_sptucker --golden)."""
import filecmp
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from oracle import oracle_py as O  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden", "io")


@pytest.mark.skipif(not O.ref_available(), reason="reference bridge not built (no /root/reference here)")
def test_io_fixtures_are_reference_output(tmp_path):
    import make_io_golden
    out = str(tmp_path / "io")
    make_io_golden.generate(out)
    names = sorted(os.listdir(GOLDEN))
    assert names == sorted(os.listdir(out))
    match, mismatch, errors = filecmp.cmpfiles(GOLDEN, out, names, shallow=False)
    assert not mismatch and not errors, (mismatch, errors)

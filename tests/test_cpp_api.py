"""The C++ host API (namespace sptucker over include/sgdt.h): build, exported
surface, and the C++ parity suite tests/cpp/test_sptucker.cpp (GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def built():
    from paper_2012_03550_b200 import _build_cpp
    lib = _build_cpp.build()
    return lib, _build_cpp.TEST_BIN


# The reference entry points a C++ caller of the hot path links against
# (proj/include/sptucker/*.hpp); all must be defined by libsptucker_b200.so.
API = [
    "sptucker::update_core_epoch(", "sptucker::update_factor_epoch(", "sptucker::rmse_mae(",
    "sptucker::train(", "sptucker::train_from_scratch(", "sptucker::sample_batch(",
    "sptucker::train_test_split(", "sptucker::partition_even(", "sptucker::reduce_in_order(",
    "sptucker::sgd_step(", "sptucker::compute_w_row(", "sptucker::grad_b(", "sptucker::core_residual(",
    "sptucker::grad_a_row(", "sptucker::grad_a_row_gram(", "sptucker::row_batch(",
    "sptucker::comm_cost_report(", "sptucker::CooTensor::CooTensor(", "sptucker::Shape::Shape(",
    "sptucker::TuckerModel::init_gaussian(", "sptucker::TuckerModel::predict(",
    "sptucker::HyperParams::validate(",
    # host I/O and generators
    "sptucker::CooTensor::load_delimited(", "sptucker::CooTensor::save_delimited(",
    "sptucker::TuckerModel::save(", "sptucker::TuckerModel::load(", "sptucker::write_metrics_csv(",
    "sptucker::parse_metrics_csv(", "sptucker::synth_planted(", "sptucker::synth_ratings(",
    "sptucker::unfold_col_index(", "sptucker::vec_index(", "sptucker::invert_vec_index(",
    # the reference's epoch benches (eval.hpp:53-95)
    "sptucker::bench_rank_scaling(", "sptucker::bench_speedup(", "sptucker::fit_linear(",
]
GOLDEN_IO = os.path.join(ROOT, "tests", "golden", "io")


def test_cpp_api_exports(built):
    lib, _ = built
    out = subprocess.run(["nm", "-DC", "--defined-only", lib], capture_output=True, text=True).stdout
    for sym in API:
        assert sym in out, sym
    # and it is a client of the C-ABI, not a CPU implementation of the hot path
    deps = subprocess.run(["ldd", lib], capture_output=True, text=True).stdout
    assert "libsgdt.so" in deps


def test_cpp_suite_cpu_part(built):
    _, exe = built
    r = subprocess.run([exe, "--cpu-only", "--golden", GOLDEN_IO], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
def test_cpp_suite_on_gpu(built):
    _, exe = built
    r = subprocess.run([exe, "--golden", GOLDEN_IO], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert re.search(r"\d+ checks, 0 failures", r.stdout)

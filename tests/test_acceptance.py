"""The reference's own acceptance suite, UNMODIFIED, run against the drop-in.

oracle/_ref/acceptance_b200 is /root/reference/proj/tests/acceptance/acceptance_main.cpp
plus proj/tests/oracle/oracle.cpp compiled against the drop-in headers
(paper_2012_03550_b200/cpp/include) and linked to libsptucker_b200.so
(`make -C oracle acceptance`, run by build() where the reference is present;
the binary travels to the GPU box with the snapshot).

Criteria (acceptance_main.cpp:636-647):
  C1 gradient fidelity   (FD vs grad_b / grad_a_row; sample_batch on the device)  gpu
  C2 model identities    (predict, reconstruct_core, compute_w_row, e_column)     host
  C3 index algebra       (unfold_col_index / vec_index)                          host
  C4 convergence         (train_from_scratch on the device)                      gpu
  C5 MovieLens surrogate (synth_ratings, train, RMSE bound)                      gpu
  C8 comm-cost model     (dense vs Kruskal parameter counts)                     host
  C9 determinism         (model files / metrics byte-identical across reruns)    gpu
  C10 strategy equivalence (serial / naive / improved within 1e-3)               gpu
C6 (rank scaling: s/epoch linear in J on CPU threads) and C7 (speedup of 4 CPU
threads over 1) measure the reference's CPU WorkerPool, which the drop-in
replaces with the device; they are not run.
"""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_b200")

needs_bin = pytest.mark.skipif(not os.path.exists(BIN),
                               reason="oracle/_ref/acceptance_b200 not built (needs /root/reference at build time)")


def run_criterion(n: int, timeout: float = 600.0) -> str:
    p = subprocess.run([BIN, "--only", str(n)], capture_output=True, text=True, timeout=timeout)
    out = p.stdout.strip()
    assert p.returncode == 0 and out.startswith("[PASS]"), f"C{n}: rc={p.returncode}\n{out}\n{p.stderr[-2000:]}"
    return out


@needs_bin
@pytest.mark.parametrize("n", [2, 3, 8])
def test_acceptance_host_criteria(n):
    print(run_criterion(n))


@needs_bin
@pytest.mark.gpu
@pytest.mark.parametrize("n", [1, 4, 5, 9, 10])
def test_acceptance_device_criteria(n):
    print(run_criterion(n))

"""Per-rank core-phase cost at 1/P of Psi: the input of DESIGN.md's multi-GPU
model.  On the GPU box:  python scripts/core_scaling.py [config] (default 2)

For P in 1, 2, 4, 8 it times (CUDA events, sgdt_last_timing) the core phase
of a session over the config's generated tensor with a batch of M/P samples:
the replicated core always reduces all of Psi (M), the sharded one reduces
M/P per rank plus one exchange per column block (not included here: add the
stream-barrier latency per step).  Prints one JSON line per (mode, P)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main(cfg):
    import torch
    from paper_2012_03550_b200 import sgdt
    data = bench.make_data(cfg, 1.0, torch.device("cuda", 0))
    spec = data["spec"]
    order = len(spec.dims)
    J = R = spec.teacher_j
    M = bench.BATCH_M[cfg]
    trc, trv = data["train"]
    A, B = bench.init_model(spec.dims, J, R, *bench.init_stats(cfg, spec), 1)
    for mode in ("column", "blocked"):
        os.environ["SGDT_CORE"] = mode
        s = sgdt.Session(spec.dims, trc, trv, [J] * order, R, device=0)
        s.set_model(A, B)
        s.seed(2)
        for P in (1, 2, 4, 8):
            m = M // P
            ch = sgdt.CoreHyper(0.01, 0.01, m, 0, 0)
            fh = sgdt.FactorHyper(0.0, 0.01, 1.0)  # frozen factor phase: times the core alone
            s.run_epochs(ch, fh, 3)
            s.run_epochs(ch, fh, 10)
            t = s.last_timing()
            print(json.dumps({"config": cfg, "core": mode, "P": P, "m_per_rank": m, "core_ms": t.core_ms,
                              "sample_ms": t.sample_ms}), flush=True)
        del s


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 2)

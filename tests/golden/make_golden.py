"""Generate tests/golden/*.json from the REFERENCE ITSELF (oracle/_ref).

Run in the build container (where /root/reference exists):
    make -C oracle ref && python tests/golden/make_golden.py

config1.json is BASELINE config 1 exactly: synth_planted 1000x800x600, 200k nnz,
teacher J=R=5 N(0,1), noise sd 0.01, seed 1; split 0.1 seed 1; J=R=5, M=1024,
lr 0.01, lambda 0.01, 10 epochs, seed 1.  It records the
head of every generated array, the head of every Psi drawn, the per-epoch RMSE
and a checksum of the final model, all as produced by the reference.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import oracle_py as O  # noqa: E402


def config1(epochs=10):
    spec = dict(dims=[1000, 800, 600], tJ=[5, 5, 5], tR=5, nnz=200000, noise=0.01, tmean=0.0,
                tsd=1.0, seed=1)
    hyper = dict(J=[5, 5, 5], R=5, lr_a=0.01, lr_b=0.01, reg_a=0.01, reg_b=0.01, batch_m=1024,
                 seed=1, epochs=epochs)
    dims = np.array(spec["dims"], np.uint32)
    nnz = spec["nnz"]
    c = np.empty(nnz * 3, np.uint32)
    v = np.empty(nnz)
    assert O.ref().ref_synth_planted(3, dims, np.array(spec["tJ"], np.uint32), spec["tR"], nnz,
                                     spec["noise"], spec["tmean"], spec["tsd"], spec["seed"], c,
                                     v) == 0
    full = O.RefTensor(dims, c, v)
    ntest = int(round(0.1 * nnz))
    trc, trv = np.empty((nnz - ntest) * 3, np.uint32), np.empty(nnz - ntest)
    tec, tev = np.empty(ntest * 3, np.uint32), np.empty(ntest)
    assert O.ref().ref_train_test_split(full.h, 0.1, 1, trc, trv, tec, tev) == 0
    tr, te = O.RefTensor(dims, trc, trv), O.RefTensor(dims, tec, tev)
    m = O.RefModel(dims, hyper["J"], hyper["R"]).init_gaussian(0.5, 0.1, hyper["seed"])
    rng = O.RefRng(hyper["seed"] + 1)
    psi_head, tr_rmse, te_rmse, tr_mae, te_mae = [], [], [], [], []
    batch = np.empty(hyper["batch_m"], np.uint32)
    for _ in range(epochs):
        assert O.ref().ref_core_epoch(m.h, tr.h, rng.h, hyper["lr_b"], hyper["reg_b"],
                                      hyper["batch_m"], 0, 0, 0, 1, batch.ctypes.data) == 0
        psi_head.append(batch[:16].tolist())
        assert O.ref().ref_factor_epoch(m.h, tr.h, rng.h, hyper["lr_a"], hyper["reg_a"], 1.0, 0,
                                        1, None, None) == 0
        a, b = O.ref_rmse_mae(m, tr)
        tr_rmse.append(a)
        tr_mae.append(b)
        a, b = O.ref_rmse_mae(m, te)
        te_rmse.append(a)
        te_mae.append(b)
    A, B = m.params()
    return dict(
        generator="tests/golden/make_golden.py via oracle/_ref (reference compiled from source)",
        spec=spec, hyper=hyper,
        coords_head=c[:64].tolist(), values_head=v[:32].tolist(),
        values_sum=float(v.sum()), train_nnz=int(nnz - ntest), test_nnz=ntest,
        train_values_head=trv[:16].tolist(), test_values_head=tev[:16].tolist(),
        psi_head=psi_head, train_rmse=tr_rmse, test_rmse=te_rmse, train_mae=tr_mae,
        test_mae=te_mae,
        final_A_sum=[float(a.sum()) for a in A], final_B=[b.tolist() for b in B],
        final_A_head=[a[:4].tolist() for a in A],
    )


def main():
    out = os.path.dirname(os.path.abspath(__file__))
    g = config1()
    with open(os.path.join(out, "config1.json"), "w") as f:
        json.dump(g, f, indent=1)
    print("wrote config1.json; final test rmse", g["test_rmse"][-1])


if __name__ == "__main__":
    main()

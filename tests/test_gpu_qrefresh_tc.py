"""The tensor-core refresh of the Kruskal rows Q^(k) = A^(k) B^(k)
(csrc/sgdt_qrefresh_tc.cu: TMA tiles, tcgen05.mma kind::tf32 as 3xTF32, TMEM
accumulator) against A B formed on the host in fp64, against the SIMT refresh,
and inside whole epochs against the oracle.

The reference has no Q: it caches the dense core (model.cpp:36-85,116-122);
Q^(k) is its Kruskal counterpart on the device.  The bar
for Q itself is fp32 rounding of a 32-term dot product (1e-6 of sum |a||b|);
the epochs keep the 1e-4 bar of tests/test_gpu_parity.py.
"""
import numpy as np
import pytest

from oracle import oracle_py as O
from test_gpu_parity import (TOL, f32, make_case, oracle_model, rel_err, session_for, unit_sigma)

pytestmark = pytest.mark.gpu


def host_q(A, B):
    A = np.asarray(A, np.float32).astype(np.float64)
    B = np.asarray(B, np.float32).astype(np.float64)
    return A @ B, np.abs(A) @ np.abs(B)


@pytest.mark.parametrize("dims,R", [((1000, 257, 40), 32), ((128, 129, 5), 32), ((700, 3, 256), 30)])
def test_q_rows_match_host_product(monkeypatch, dims, R):
    J = (32, 32, 32)
    tr, _ = make_case(dims, J, 8, 2000, 3)
    m = oracle_model(dims, J, R, 11, sd=0.3, mean=0.1)
    A, B = m.params()
    got = {}
    for qtc in ("1", "0"):
        monkeypatch.setenv("SGDT_QTC", qtc)
        s = session_for(dims, tr, J, R)
        s.set_model(A, B)  # refreshes every Q^(k)
        got[qtc] = [s.q_rows(n) for n in range(3)]
        s.close()
    for n in range(3):
        ref, mag = host_q(A[n], B[n])
        for qtc in ("1", "0"):
            err = np.max(np.abs(got[qtc][n].astype(np.float64) - ref) / np.maximum(mag, 1e-30))
            assert err <= 1e-6, f"SGDT_QTC={qtc} mode {n}: {err}"
        # both paths agree to fp32 rounding of the accumulation
        d = np.max(np.abs(got["1"][n].astype(np.float64) - got["0"][n].astype(np.float64)) / np.maximum(mag, 1e-30))
        assert d <= 1e-6, f"mode {n}: tensor-core vs SIMT {d}"


def test_q_rows_special_values(monkeypatch):
    """Exact small integers, signed zeros and tiny values survive the hi/lo split."""
    monkeypatch.setenv("SGDT_QTC", "1")
    dims, J, R = (300, 130, 20), (32, 32, 32), 32
    tr, _ = make_case(dims, J, 8, 1500, 5)
    rng = np.random.default_rng(0)
    A = [rng.integers(-3, 4, size=(dims[n], 32)).astype(np.float64) for n in range(3)]
    B = [rng.integers(-2, 3, size=(32, R)).astype(np.float64) for n in range(3)]
    A[1] *= 2.0 ** -60
    A[2][0, :] = 0.0
    s = session_for(dims, tr, J, R)
    s.set_model(A, B)
    for n in range(3):
        ref, _ = host_q(A[n], B[n])
        assert np.array_equal(s.q_rows(n).astype(np.float64), ref), f"mode {n}"  # exact: integer products


@pytest.mark.parametrize("dims,nnz,bm", [((300, 200, 130), 20000, 500), ((129, 40, 1000), 15000, 256)])
def test_epochs_with_tensor_core_refresh_match_oracle(monkeypatch, dims, nnz, bm):
    monkeypatch.setenv("SGDT_QTC", "1")
    J, R = (32, 32, 32), 32
    sig = unit_sigma(dims, J, R)
    tr, _ = make_case(dims, J, min(J), nnz, 17, tm=0.0, ts=sig)
    t = O.Tensor(dims, *tr)
    s = session_for(dims, tr, J, R)
    m = oracle_model(dims, J, R, 23, sd=sig, mean=0.0)
    rng = O.Rng(5)
    ws = O.CoreWorkspace(nnz)
    s.set_rng(*rng.state())
    s.set_model(*m.params())
    lr, reg = 0.01, 0.01
    for epoch in range(2):
        # core phase, then the factor phase on the device's own Q (refreshed by the
        # tensor-core kernel after the cooperative kernel), teacher-forced per epoch
        s.core_epoch(lr, reg, bm)
        O.update_core_epoch(m, t, lr, reg, bm, rng, ws)
        assert np.array_equal(s.last_batch(), ws.batch())
        _, Bd = s.get_model()
        _, RB = m.params()
        for n in range(3):
            assert rel_err(Bd[n], RB[n]) <= TOL, f"core B^({n}) epoch {epoch}"
        # Q after the core phase = A B with the device's new B
        Ad, Bd = s.get_model()
        for n in range(3):
            ref, mag = host_q(Ad[n], Bd[n])
            err = np.max(np.abs(s.q_rows(n).astype(np.float64) - ref) / np.maximum(mag, 1e-30))
            assert err <= 1e-6, f"Q^({n}) after the core phase: {err}"
        up, sk = s.factor_epoch(lr, reg)
        m.set_params(*[[f32(x) for x in part] for part in (Ad, Bd)])  # oracle from the device's post-core state
        rup, rsk = O.update_factor_epoch(m, t, lr, reg, rng)
        assert (up, sk) == (rup, rsk)
        Ad, Bd = s.get_model()
        RA, RB = m.params()
        for n in range(3):
            assert rel_err(Ad[n], RA[n]) <= TOL, f"factor A^({n}) epoch {epoch}"
        m.set_params([f32(a) for a in RA], [f32(b) for b in RB])
        s.set_model(*m.params())


# ---- core phase with the per-sample state split over shared memory, registers and the
# global scratch (sgdt_core.cu "semi": configs 4 and 5 at full size), forced at test sizes
@pytest.mark.parametrize("J,R,nsm", [(32, 32, "40"), (16, 16, "1000000"), (32, 30, "17"), (20, 18, "33")])
def test_core_semi_local_state_matches_oracle(monkeypatch, J, R, nsm):
    monkeypatch.setenv("SGDT_CORE_STATE", "semi")
    monkeypatch.setenv("SGDT_CORE_NSM", nsm)  # samples beyond it sit in registers (one per thread)
    dims, nnz, bm = (60, 50, 40), 12000, 3000  # 24 CTAs x 125 samples
    Js = (J, J, J)
    sig = unit_sigma(dims, Js, R)
    tr, _ = make_case(dims, Js, min(J, 16), nnz, 17, tm=0.0, ts=sig)
    t = O.Tensor(dims, *tr)
    s = session_for(dims, tr, Js, R)
    m = oracle_model(dims, Js, R, 23, sd=sig, mean=0.0)
    rng = O.Rng(5)
    ws = O.CoreWorkspace(nnz)
    s.set_rng(*rng.state())
    for epoch in range(2):
        s.set_model(*m.params())
        s.core_epoch(0.01, 0.01, bm)
        O.update_core_epoch(m, t, 0.01, 0.01, bm, rng, ws)
        assert np.array_equal(s.last_batch(), ws.batch())
        _, Bd = s.get_model()
        RA, RB = m.params()
        for n in range(3):
            assert rel_err(Bd[n], RB[n]) <= TOL, f"core B^({n}) epoch {epoch}"
        m.set_params([f32(a) for a in RA], [f32(b) for b in RB])
    # the same phase with the state in the global scratch: bit for bit the same B when no
    # sample moved to registers (same values, same summation order, only where they live
    # differs); register samples change which thread sums which sample (fp32 association)
    out = {}
    for state in ("semi", "global"):
        monkeypatch.setenv("SGDT_CORE_STATE", state)
        monkeypatch.setenv("SGDT_CORE_SYNC", "red")
        s2 = session_for(dims, tr, Js, R)
        s2.set_model(*m.params())
        s2.set_rng(*O.Rng(9).state())
        s2.core_epoch(0.01, 0.01, bm)
        out[state] = s2.get_model()[1]
        s2.close()
    for n in range(3):
        if int(nsm) >= 125:
            assert np.array_equal(out["semi"][n], out["global"][n]), f"B^({n}): semi vs global state"
        else:
            assert rel_err(out["semi"][n], out["global"][n]) <= 1e-6, f"B^({n}): semi vs global state"


def test_blocked_core_uses_tensor_core_refresh(monkeypatch):
    """The blocked (multi-GPU) core phase hands wide modes to the same refresh kernel."""
    monkeypatch.setenv("SGDT_QTC", "1")
    monkeypatch.setenv("SGDT_CORE", "blocked")
    dims, J, R, nnz, bm = (300, 200, 130), (32, 32, 32), 32, 15000, 400
    sig = unit_sigma(dims, J, R)
    tr, _ = make_case(dims, J, 16, nnz, 17, tm=0.0, ts=sig)
    t = O.Tensor(dims, *tr)
    s = session_for(dims, tr, J, R)
    m = oracle_model(dims, J, R, 23, sd=sig, mean=0.0)
    rng = O.Rng(5)
    ws = O.CoreWorkspace(nnz)
    s.set_rng(*rng.state())
    s.set_model(*m.params())
    s.core_epoch(0.01, 0.01, bm)
    O.update_core_epoch(m, t, 0.01, 0.01, bm, rng, ws)
    Ad, Bd = s.get_model()
    _, RB = m.params()
    for n in range(3):
        assert rel_err(Bd[n], RB[n]) <= TOL, f"core B^({n})"
        ref, mag = host_q(Ad[n], Bd[n])
        err = np.max(np.abs(s.q_rows(n).astype(np.float64) - ref) / np.maximum(mag, 1e-30))
        assert err <= 1e-6, f"Q^({n}) after the blocked core phase: {err}"

"""Multi-rank factor phase (paper_2012_03550_b200/distributed.py).

CPU: the orchestration (partition_even slices, boundary export, rank-ordered
merge, row publication) on a numpy stand-in session, with in-process thread
ranks and with 2 torch.distributed gloo processes; results must equal the
single-rank run and the oracle's serial factor epoch.
GPU: real sharded sessions (2 and 3 ranks as threads on one GPU) against the
single-session device result and the oracle."""
import os
import socket
import threading

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import oracle_py as O
from paper_2012_03550_b200 import distributed as D

from cpu_shard_backend import CpuShard

DIMS, J, R = (7, 40, 30), (3, 3, 3), 3


class FH:  # FactorHyper look-alike for the CPU backend
    lr, reg, row_fraction = 0.02, 0.01, 1.0


def data(nnz=2500, seed=5):
    c, v = O.synth_planted(DIMS, J, R, nnz, 0.05, 0.0, 0.6, seed)
    m = O.Model(DIMS, J, R).init_gaussian(0.0, 0.6, seed + 1)
    return c, v, m.params()


def oracle_factor(c, v, A, B):
    m = O.Model(DIMS, J, R)
    m.set_params(A, B)
    O.update_factor_epoch(m, O.Tensor(DIMS, c, v), FH.lr, FH.reg, O.Rng(1))
    return m.params()[0]


def run_threads(c, v, A, B, world):
    groups = D.ThreadGroup.make(world)
    sess = [CpuShard(DIMS, c, v, J, R, r, world, A, B) for r in range(world)]
    errs = []

    def body(r):
        try:
            D.factor_epoch_sharded(sess[r], groups[r], FH)
        except Exception as e:  # surfaced below
            errs.append(e)
            raise

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    return sess


def test_merge_boundary_is_rank_ordered_sum():
    recs = [D.pack_boundary([5], np.array([[1.0, 2.0]]), 2),
            D.pack_boundary([5, 9], np.array([[10.0, 20.0], [1.0, 1.0]]), 2),
            D.pack_boundary([], np.zeros((0, 2)), 2),
            D.pack_boundary([9], np.array([[0.5, 0.5]]), 2)]
    m = D.merge_boundary(recs, 2)
    assert sorted(m) == [5, 9]
    assert np.array_equal(m[5], [11.0, 22.0]) and np.array_equal(m[9], [1.5, 1.5])


@pytest.mark.parametrize("world", [2, 3, 7, 16])
def test_thread_ranks_match_single_rank_and_oracle(world):
    c, v, (A, B) = data()
    one = run_threads(c, v, A, B, 1)[0]
    ref = oracle_factor(c, v, A, B)
    for n in range(3):
        assert np.max(np.abs(one.A[n] - ref[n])) <= 1e-9
    ranks = run_threads(c, v, A, B, world)
    for s in ranks:  # every rank holds the full, identical result
        for n in range(3):
            assert np.max(np.abs(s.A[n] - one.A[n])) <= 1e-12


def run_threads_p2p(c, v, A, B, world):
    groups = D.ThreadGroup.make(world)
    sess = [CpuShard(DIMS, c, v, J, R, r, world, A, B) for r in range(world)]
    errs = []

    def body(r):
        try:
            D.connect_peers(sess[r], groups[r])
            groups[r].barrier()
            D.factor_epoch_p2p(sess[r], groups[r], FH)
        except Exception as e:  # surfaced below
            errs.append(e)
            raise

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    return sess


@pytest.mark.parametrize("world", [2, 3, 7, 16])
def test_thread_ranks_peer_publication_matches_broadcast_path(world):
    """The peer-store driver (records into every rank's slot, owner-only
    finalisation of cut rows, rows stored straight into the peers) gives
    exactly the broadcast driver's result on every rank."""
    c, v, (A, B) = data()
    want = run_threads(c, v, A, B, world)[0]
    for s in run_threads_p2p(c, v, A, B, world):
        for n in range(3):
            assert np.array_equal(s.A[n], want.A[n])


def _gloo_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c, v, (A, B) = data()
    s = CpuShard(DIMS, c, v, J, R, rank, world, A, B)
    D.factor_epoch_sharded(s, D.TorchGroup(), FH)
    np.save(os.path.join(out_dir, f"A_{rank}.npy"), np.concatenate([a.ravel() for a in s.A]))
    dist.destroy_process_group()


def test_gloo_two_processes(tmp_path):
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mp.spawn(_gloo_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    c, v, (A, B) = data()
    one = run_threads(c, v, A, B, 1)[0]
    want = np.concatenate([a.ravel() for a in one.A])
    for r in range(2):
        got = np.load(tmp_path / f"A_{r}.npy")
        assert np.max(np.abs(got - want)) <= 1e-12


# ---------------------------------------------------------------- sharded core phase
class CH:  # CoreHyper look-alike
    lr, reg, batch_m, resample_per_mode, incremental_residual = 0.02, 0.01, 300, 0, 0


def oracle_core(c, v, A, B, seed):
    m = O.Model(DIMS, J, R)
    m.set_params(A, B)
    O.update_core_epoch(m, O.Tensor(DIMS, c, v), CH.lr, CH.reg, CH.batch_m, O.Rng(seed),
                        O.CoreWorkspace(len(v)))
    return m.params()[1]


def run_core_threads(c, v, A, B, world, block, seed=3):
    groups = D.ThreadGroup.make(world)
    sess = [CpuShard(DIMS, c, v, J, R, r, world, A, B) for r in range(world)]
    errs = []

    def body(r):
        try:
            sess[r].seed(seed)
            D.core_epoch_sharded(sess[r], groups[r], CH, block)
        except Exception as e:  # surfaced below
            errs.append(e)
            raise

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    return sess


@pytest.mark.parametrize("world", [1, 2, 3, 7])
@pytest.mark.parametrize("block", [1, 2, 3])
def test_sharded_core_thread_ranks_match_oracle(world, block):
    """The blocked algebra (V0 + in-block Gram, rank-ordered sums, T exact
    Gauss-Seidel steps) equals the reference's column-by-column update."""
    c, v, (A, B) = data(seed=11)
    want = oracle_core(c, v, A, B, 3)
    sess = run_core_threads(c, v, A, B, world, block)
    for s in sess:
        for n in range(3):
            assert np.max(np.abs(s.B[n] - want[n])) <= 1e-11
    for s in sess[1:]:
        for n in range(3):
            assert np.array_equal(s.B[n], sess[0].B[n])


def _gloo_core_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c, v, (A, B) = data(seed=11)
    s = CpuShard(DIMS, c, v, J, R, rank, world, A, B)
    s.seed(3)
    D.core_epoch_sharded(s, D.TorchGroup(), CH, 2)
    np.save(os.path.join(out_dir, f"B_{rank}.npy"), np.concatenate([b.ravel() for b in s.B]))
    dist.destroy_process_group()


def test_sharded_core_gloo_two_processes(tmp_path):
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mp.spawn(_gloo_core_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    c, v, (A, B) = data(seed=11)
    want = np.concatenate([b.ravel() for b in oracle_core(c, v, A, B, 3)])
    got = [np.load(tmp_path / f"B_{r}.npy") for r in range(2)]
    assert np.array_equal(got[0], got[1])
    assert np.max(np.abs(got[0] - want)) <= 1e-11


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_gpu_sharded_sessions_match_single_session(world):
    from paper_2012_03550_b200 import sgdt
    c, v, (A, B) = data(nnz=6000, seed=9)
    A = [a.astype(np.float32).astype(np.float64) for a in A]
    B = [b.astype(np.float32).astype(np.float64) for b in B]
    fh = sgdt.FactorHyper(FH.lr, FH.reg, 1.0)
    ch = sgdt.CoreHyper(0.01, 0.01, 256, 0, 0)
    single = sgdt.Session(DIMS, c, v, J, R)
    single.set_model(A, B)
    single.seed(4)
    single.core_epoch(ch.lr, ch.reg, ch.batch_m)
    single.factor_epoch(fh.lr, fh.reg)
    SA, SB = single.get_model()
    groups = D.ThreadGroup.make(world)
    sess = [D.ShardedSession(DIMS, c, v, J, R, r, world) for r in range(world)]
    for s in sess:
        s.set_model(A, B)
        s.seed(4)
    errs = []

    def body(r):
        try:
            D.run_epochs_sharded(sess[r], groups[r], ch, fh, 1)
        except Exception as e:
            errs.append(e)
            raise

    th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for s in sess:
        GA, GB = s.get_model()
        for n in range(3):
            assert np.array_equal(GB[n], SB[n])  # replicated core phase: bit-identical
            assert np.max(np.abs(GA[n] - SA[n]) / np.maximum(1, np.abs(SA[n]))) <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_gpu_peer_publication_matches_broadcast_path(world):
    """Sharded sessions publishing through peer stores (ranks as threads on one
    GPU: the peers' buffers are plain device pointers of the same process)
    give exactly the host-merge + broadcast driver's model on every rank."""
    from paper_2012_03550_b200 import sgdt
    c, v, (A, B) = data(nnz=6000, seed=9)
    A = [a.astype(np.float32).astype(np.float64) for a in A]
    B = [b.astype(np.float32).astype(np.float64) for b in B]
    fh = sgdt.FactorHyper(FH.lr, FH.reg, 1.0)
    ch = sgdt.CoreHyper(0.01, 0.01, 256, 0, 0)
    results = {}
    for mode in ("broadcast", "p2p"):
        groups = D.ThreadGroup.make(world)
        sess = [D.ShardedSession(DIMS, c, v, J, R, r, world) for r in range(world)]
        for s in sess:
            s.set_model(A, B)
            s.seed(4)
        errs = []

        def body(r):
            try:
                if mode == "p2p":
                    D.run_epochs_p2p(sess[r], groups[r], ch, fh, 2)
                else:
                    D.run_epochs_sharded(sess[r], groups[r], ch, fh, 2)
            except Exception as e:
                errs.append(e)
                raise

        th = [threading.Thread(target=body, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errs, errs
        results[mode] = [s.get_model() for s in sess]
    for r in range(world):
        for n in range(3):
            assert np.array_equal(results["p2p"][r][0][n], results["broadcast"][0][0][n])
            assert np.array_equal(results["p2p"][r][1][n], results["broadcast"][0][1][n])


def _ipc_worker(rank, world, port, out_dir):
    """One process per rank on the same GPU: peers mapped through CUDA IPC
    handles, host (gloo) barriers -- no kernel waits on another rank."""
    import torch
    import torch.distributed as dist
    from paper_2012_03550_b200 import sgdt
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    c, v, (A, B) = data(nnz=6000, seed=9)
    A = [a.astype(np.float32).astype(np.float64) for a in A]
    B = [b.astype(np.float32).astype(np.float64) for b in B]
    s = D.ShardedSession(DIMS, c, v, J, R, rank, world, device=0)
    s.set_model(A, B)
    s.seed(4)
    D.run_epochs_p2p(s, D.TorchGroup(), sgdt.CoreHyper(0.01, 0.01, 256, 0, 0), sgdt.FactorHyper(FH.lr, FH.reg, 1.0), 2)
    GA, GB = s.get_model()
    np.save(os.path.join(out_dir, f"P_{rank}.npy"), np.concatenate([x.ravel() for x in GA + GB]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_gpu_ipc_peer_publication_two_processes(tmp_path):
    """The cross-process form of the peer-store driver (sgdt_peer_ipc_handles /
    sgdt_ipc_open) gives the single-process result on both ranks."""
    from paper_2012_03550_b200 import sgdt
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mp.spawn(_ipc_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    c, v, (A, B) = data(nnz=6000, seed=9)
    A = [a.astype(np.float32).astype(np.float64) for a in A]
    B = [b.astype(np.float32).astype(np.float64) for b in B]
    groups = D.ThreadGroup.make(2)
    sess = [D.ShardedSession(DIMS, c, v, J, R, r, 2) for r in range(2)]
    for x in sess:
        x.set_model(A, B)
        x.seed(4)
    th = [threading.Thread(target=D.run_epochs_sharded,
                           args=(sess[r], groups[r], sgdt.CoreHyper(0.01, 0.01, 256, 0, 0),
                                 sgdt.FactorHyper(FH.lr, FH.reg, 1.0), 2)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    GA, GB = sess[0].get_model()
    want = np.concatenate([x.ravel() for x in GA + GB])
    for r in range(2):
        assert np.array_equal(np.load(tmp_path / f"P_{r}.npy"), want)


@pytest.mark.gpu
def test_gpu_nccl_path_single_rank():
    """The NCCL publication path (torch tensor aliasing the session's A^(n),
    dist.broadcast on it) at world size 1."""
    import torch
    import torch.distributed as dist
    from paper_2012_03550_b200 import sgdt
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        c, v, (A, B) = data(nnz=6000, seed=9)
        fh = sgdt.FactorHyper(FH.lr, FH.reg, 1.0)
        ch = sgdt.CoreHyper(0.01, 0.01, 256, 0, 0)
        single = sgdt.Session(DIMS, c, v, J, R)
        single.set_model(A, B)
        single.seed(4)
        single.run_epochs(ch, fh, 2)
        s = D.ShardedSession(DIMS, c, v, J, R, 0, 1)
        s.set_model(A, B)
        s.seed(4)
        g = D.TorchGroup()
        assert g.nccl
        D.run_epochs_sharded(s, g, ch, fh, 2)
        a = s.factor_tensor(0)
        assert a.is_cuda and tuple(a.shape) == (DIMS[0], J[0])
        SA, SB = single.get_model()
        GA, GB = s.get_model()
        for n in range(3):
            assert np.array_equal(GA[n], SA[n]) and np.array_equal(GB[n], SB[n])
        # the peer-store driver over the NCCL stream barrier (no peers at P = 1)
        p = D.ShardedSession(DIMS, c, v, J, R, 0, 1)
        p.set_model(A, B)
        p.seed(4)
        D.run_epochs_p2p(p, g, ch, fh, 2)
        PA, PB = p.get_model()
        for n in range(3):
            assert np.array_equal(PA[n], SA[n]) and np.array_equal(PB[n], SB[n])
    finally:
        dist.destroy_process_group()

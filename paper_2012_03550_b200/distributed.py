"""Multi-GPU SGD_Tucker epochs: the factor phase is sharded over ranks, the
core phase is sharded or replicated.

One process (or thread) per GPU, each holding a sharded session
(`sgdt_session_create_shard`).  Per epoch:

* Core phase.  Every rank draws the identical Psi (same RNG state, same pool,
  bit-exact sampler).
  - sharded (core="sharded", `core_epoch_sharded`): rank r reduces only its
    slice partition_even(M, P)[r] (the reference's worker slices,
    scheduler.cpp:34-46).  The columns of B^(n) go in blocks of T; per block
    each rank stores its B^(n)-gradient vector (V0 and the in-block Gram
    terms, sgdt.h "sharded core phase") into slot `rank` of every rank's
    exchange buffer, and after a barrier every rank sums the slots in rank
    order (core_optimizer.cpp:225-243) and replays the block's Gauss-Seidel
    column steps, so B^(n) stays bit-identical everywhere.  N ceil(R/T)
    exchanges per epoch, of ~T^2 J^2 / 2 doubles each.
  - replicated (core="replicated"): every rank runs the identical core kernel
    on the identical model; no collective at all.
* Factor phase, sharded.  For each mode n, in order (Gauss-Seidel):
  1. each rank runs the factor kernel over its slice partition_even(nnz, P)
     of the mode-n order (the `improved` slices of factor_optimizer.cpp:
     209-210) and finalises every row inside it;
  2. the <= 2 rows cut by its slice edges are exported as fp64 partial
     gradients; an all-gather plus a rank-ordered sum reproduces the
     reference's boundary merge (factor_optimizer.cpp:247-270);
  3. the ranks that hold a cut row finalise it from the merged gradient;
  4. every rank broadcasts its row block [row_lo, row_hi) of A^(n) and all
     ranks refresh Q^(n) = A^(n) B^(n) for the next mode's gathers.

Collectives go through a `Group`: `TorchGroup` wraps torch.distributed (NCCL
on GPUs -- the row blocks move device to device over NVLink; gloo for CPU
tests), `ThreadGroup` runs several ranks as threads of one process (tests on
one GPU, where no kernel ever waits on another).
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import sgdt


# ----------------------------------------------------------------------------
# groups
# ----------------------------------------------------------------------------
class Group:
    rank: int
    world: int

    def all_gather(self, arr: np.ndarray) -> list[np.ndarray]:
        raise NotImplementedError

    def broadcast(self, arr: np.ndarray, src: int) -> np.ndarray:
        raise NotImplementedError

    def barrier(self) -> None:
        raise NotImplementedError

    def max(self, x: float) -> float:
        return float(max(a[0] for a in self.all_gather(np.array([x], np.float64))))


class ThreadGroup(Group):
    """Ranks as threads of one process; host-side rendezvous only."""

    class _Shared:
        def __init__(self, world):
            self.world = world
            self.bar = threading.Barrier(world)
            self.slots = [None] * world

    def __init__(self, shared: "_Shared", rank: int):
        self.s, self.rank, self.world = shared, rank, shared.world

    @classmethod
    def make(cls, world: int) -> list["ThreadGroup"]:
        sh = cls._Shared(world)
        return [cls(sh, r) for r in range(world)]

    def all_gather(self, arr):
        self.s.slots[self.rank] = np.array(arr, copy=True)
        self.s.bar.wait()
        out = [np.array(x, copy=True) for x in self.s.slots]
        self.s.bar.wait()
        return out

    def broadcast(self, arr, src):
        if self.rank == src:
            self.s.slots[src] = np.array(arr, copy=True)
        self.s.bar.wait()
        out = np.array(self.s.slots[src], copy=True)
        self.s.bar.wait()
        return out

    def barrier(self):
        self.s.bar.wait()

    def stream_barrier(self, sess) -> None:
        """Order every rank's queued device work before any rank's next work."""
        sess.synchronize()
        self.s.bar.wait()


class TorchGroup(Group):
    """torch.distributed process group (NCCL for GPU ranks, gloo on CPU)."""

    def __init__(self, device=None):
        import torch
        import torch.distributed as dist
        self.dist, self.torch = dist, torch
        self.rank, self.world = dist.get_rank(), dist.get_world_size()
        self.nccl = dist.get_backend() == "nccl"
        self.device = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if self.nccl else torch.device("cpu"))

    def _t(self, arr):
        return self.torch.as_tensor(np.ascontiguousarray(arr)).to(self.device)

    def all_gather(self, arr):
        t = self._t(arr)
        out = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t)
        return [o.cpu().numpy() for o in out]

    def broadcast(self, arr, src):
        t = self._t(arr)
        self.dist.broadcast(t, src=src)
        return t.cpu().numpy()

    def barrier(self):
        self.dist.barrier()

    def stream_barrier(self, sess) -> None:
        """NCCL: a one-element all-reduce enqueued on the session's stream --
        it completes on a rank only after every rank's earlier kernels (and
        their peer stores) completed, with no host synchronisation.  gloo:
        synchronise, then a host barrier."""
        if not self.nccl:
            sess.synchronize()
            self.dist.barrier()
            return
        torch = self.torch
        if not hasattr(self, "_tok"):
            self._tok = torch.zeros(1, device=self.device)
            self._streams = {}
        st = self._streams.get(sess.stream)
        if st is None:
            st = self._streams[sess.stream] = torch.cuda.ExternalStream(sess.stream)
        with torch.cuda.stream(st):
            self.dist.all_reduce(self._tok)


# ----------------------------------------------------------------------------
# the sharded GPU session
# ----------------------------------------------------------------------------
class _ShardInfo(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("entry_begin", C.c_uint64),
                ("entry_end", C.c_uint64), ("row_lo", C.c_uint32), ("row_hi", C.c_uint32),
                ("n_export", C.c_uint32), ("export_rows", C.c_uint32 * 2)]


def _bind():
    L = sgdt.load()
    if getattr(L, "_shard_bound", False):
        return L
    vp = C.c_void_p
    L.sgdt_session_create_shard.argtypes = [C.POINTER(sgdt._TensorDesc), C.POINTER(sgdt._TensorDesc),
                                            C.POINTER(C.c_uint32), C.c_uint32, C.c_int, C.c_int, C.c_int,
                                            C.POINTER(vp)]
    L.sgdt_get_shard_info.argtypes = [vp, C.c_int, C.POINTER(_ShardInfo)]
    L.sgdt_factor_mode_local.argtypes = [vp, C.c_int, C.POINTER(sgdt.FactorHyper), C.POINTER(C.c_double)]
    L.sgdt_factor_mode_finish.argtypes = [vp, C.c_int, C.POINTER(sgdt.FactorHyper), C.c_uint32,
                                          C.POINTER(C.c_uint32), C.POINTER(C.c_double)]
    L.sgdt_factor_rows.argtypes = [vp, C.c_int, C.c_uint32, C.c_uint32, C.c_void_p, C.c_int, C.c_int]
    L.sgdt_factor_device_ptr.argtypes = [vp, C.c_int, C.POINTER(C.c_void_p)]
    L.sgdt_refresh_q.argtypes = [vp, C.c_int]
    L.sgdt_synchronize.argtypes = [vp]
    L.sgdt_peer_buffers.argtypes = [vp, C.POINTER(vp)]
    L.sgdt_peer_ipc_handles.argtypes = [vp, vp]
    L.sgdt_ipc_open.argtypes = [vp, C.c_int, C.POINTER(vp)]
    L.sgdt_set_peers.argtypes = [vp, C.POINTER(vp)]
    L.sgdt_core_epoch_async.argtypes = [vp, C.POINTER(sgdt.CoreHyper)]
    L.sgdt_sample_ahead.argtypes = [vp, C.POINTER(sgdt.CoreHyper)]
    L.sgdt_factor_mode_p2p.argtypes = [vp, C.c_int, C.POINTER(sgdt.FactorHyper)]
    L.sgdt_factor_merge_p2p.argtypes = [vp, C.c_int, C.POINTER(sgdt.FactorHyper)]
    L.sgdt_check.argtypes = [vp]
    L.sgdt_core_plan.argtypes = [vp, C.POINTER(sgdt.CoreHyper), C.c_uint32, C.POINTER(C.c_uint32),
                                 C.POINTER(C.c_uint32)]
    L.sgdt_core_step.argtypes = [vp, C.c_uint32]
    L._shard_bound = True
    return L


class _CudaArray:
    """Zero-copy view of library-owned device memory for torch (NCCL)."""

    def __init__(self, ptr: int, shape, typestr="<f4"):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class ShardedSession(sgdt.Session):
    """A session holding rank `rank`'s slices of every mode-sorted order."""

    row_dtype = np.float32

    def __init__(self, dims, coords, values, J, R, rank, world, test=None, perms=None, device=-1):
        L = _bind()
        self._tr = sgdt._Tensor(dims, coords, values, perms)
        self._te = sgdt._Tensor(dims, *test) if test is not None else None
        self.order = self._tr.order
        self.dims = [int(d) for d in self._tr.dims]
        self.J = np.ascontiguousarray(J, np.uint32)
        self.R = int(R)
        self.nnz = len(self._tr.values)
        self.rank, self.world = rank, world
        self.device = device
        h = C.c_void_p()
        sgdt._ck(L.sgdt_session_create_shard(C.byref(self._tr.desc), C.byref(self._te.desc) if self._te else None,
                                             sgdt._p(self.J, C.c_uint32), self.R, device, rank, world, C.byref(h)))
        self.h = h
        self._tr = self._te = None

    def shard_info(self, n: int) -> _ShardInfo:
        info = _ShardInfo()
        sgdt._ck(_bind().sgdt_get_shard_info(self.h, n, C.byref(info)))
        return info

    def factor_mode_local(self, n: int, fh: sgdt.FactorHyper):
        info = self.shard_info(n)
        g = np.zeros((2, self.R))
        sgdt._ck(_bind().sgdt_factor_mode_local(self.h, n, C.byref(fh), sgdt._p(g, C.c_double)))
        k = int(info.n_export)
        return np.array(info.export_rows[:k], np.uint32), g[:k].copy()

    def factor_mode_finish(self, n: int, fh: sgdt.FactorHyper, rows, g) -> None:
        rows = np.ascontiguousarray(rows, np.uint32)
        g = np.ascontiguousarray(g, np.float64).reshape(len(rows), self.R)
        sgdt._ck(_bind().sgdt_factor_mode_finish(self.h, n, C.byref(fh), len(rows), sgdt._p(rows, C.c_uint32),
                                                 sgdt._p(g, C.c_double)))

    def get_rows(self, n: int, lo: int, hi: int) -> np.ndarray:
        out = np.empty((hi - lo, int(self.J[n])), np.float32)
        sgdt._ck(_bind().sgdt_factor_rows(self.h, n, lo, hi, out.ctypes.data_as(C.c_void_p), 0, 0))
        return out

    def set_rows(self, n: int, lo: int, block: np.ndarray) -> None:
        block = np.ascontiguousarray(block, np.float32)
        sgdt._ck(_bind().sgdt_factor_rows(self.h, n, lo, lo + block.shape[0], block.ctypes.data_as(C.c_void_p),
                                          1, 0))

    def factor_tensor(self, n: int):
        """A^(n) as a torch CUDA tensor aliasing the session's memory."""
        import torch
        p = C.c_void_p()
        sgdt._ck(_bind().sgdt_factor_device_ptr(self.h, n, C.byref(p)))
        return torch.as_tensor(_CudaArray(p.value, (self.dims[n], int(self.J[n]))), device="cuda")

    def refresh_q(self, n: int) -> None:
        sgdt._ck(_bind().sgdt_refresh_q(self.h, n))

    def synchronize(self) -> None:
        sgdt._ck(_bind().sgdt_synchronize(self.h))

    # ---- peer-memory publication (NVLink P2P) ------------------------------
    @property
    def n_peer_buffers(self) -> int:
        return 2 * self.order + 2

    def peer_buffers(self) -> list[int]:
        out = (C.c_void_p * self.n_peer_buffers)()
        sgdt._ck(_bind().sgdt_peer_buffers(self.h, out))
        return [int(p or 0) for p in out]

    def peer_ipc_handles(self) -> np.ndarray:
        out = np.zeros(self.n_peer_buffers * 64, np.uint8)
        sgdt._ck(_bind().sgdt_peer_ipc_handles(self.h, out.ctypes.data_as(C.c_void_p)))
        return out

    def set_peers(self, table) -> None:
        """table: world x (2N+2) device pointers valid in this process."""
        flat = [int(p) for row in table for p in row]
        arr = (C.c_void_p * len(flat))(*flat)
        sgdt._ck(_bind().sgdt_set_peers(self.h, arr))
        self.peers_set = True

    def core_epoch_async(self, ch: sgdt.CoreHyper) -> None:
        sgdt._ck(_bind().sgdt_core_epoch_async(self.h, C.byref(ch)))

    def sample_ahead(self, ch: sgdt.CoreHyper) -> None:
        sgdt._ck(_bind().sgdt_sample_ahead(self.h, C.byref(ch)))

    def core_plan(self, ch: sgdt.CoreHyper, block: int = 0) -> tuple[int, int]:
        """Begin a sharded core phase; returns (steps, T)."""
        steps, T = C.c_uint32(), C.c_uint32()
        sgdt._ck(_bind().sgdt_core_plan(self.h, C.byref(ch), block, C.byref(steps), C.byref(T)))
        return int(steps.value), int(T.value)

    def core_step(self, k: int) -> None:
        sgdt._ck(_bind().sgdt_core_step(self.h, k))

    def factor_mode_p2p(self, n: int, fh: sgdt.FactorHyper) -> None:
        sgdt._ck(_bind().sgdt_factor_mode_p2p(self.h, n, C.byref(fh)))

    def factor_merge_p2p(self, n: int, fh: sgdt.FactorHyper) -> None:
        sgdt._ck(_bind().sgdt_factor_merge_p2p(self.h, n, C.byref(fh)))

    def check(self) -> None:
        sgdt._ck(_bind().sgdt_check(self.h))


# ----------------------------------------------------------------------------
# the epoch driver (backend-agnostic: tests run it on a CPU backend too)
# ----------------------------------------------------------------------------
def merge_boundary(records: list[np.ndarray], R: int) -> dict[int, np.ndarray]:
    """Rank-ordered fp64 sum of every exported row (factor_optimizer.cpp:247-270).

    records[r] = [n_export, row0, row1, g0 (R), g1 (R)] from rank r."""
    merged: dict[int, np.ndarray] = {}
    for rec in records:  # ascending rank
        k = int(rec[0])
        for i in range(k):
            row = int(rec[1 + i])
            g = np.asarray(rec[3 + i * R: 3 + (i + 1) * R], np.float64)
            merged[row] = merged[row] + g if row in merged else g.copy()
    return merged


def pack_boundary(rows, g, R: int) -> np.ndarray:
    rec = np.zeros(3 + 2 * R, np.float64)
    rec[0] = len(rows)
    for i, row in enumerate(rows):
        rec[1 + i] = row
        rec[3 + i * R: 3 + (i + 1) * R] = g[i]
    return rec


def publish_rows(sess, group: Group, n: int, ranges: list[tuple[int, int]]) -> None:
    """Every rank ends up with every rank's block of A^(n)."""
    if isinstance(group, TorchGroup) and group.nccl and hasattr(sess, "factor_tensor"):
        import torch
        sess.synchronize()
        A = sess.factor_tensor(n)
        for r, (lo, hi) in enumerate(ranges):
            if hi > lo:
                group.dist.broadcast(A[lo:hi], src=r)
        torch.cuda.synchronize()
        return
    for r, (lo, hi) in enumerate(ranges):
        if hi <= lo:
            continue
        dt = getattr(sess, "row_dtype", np.float32)
        block = sess.get_rows(n, lo, hi) if group.rank == r else np.empty((hi - lo, int(sess.J[n])), dt)
        block = group.broadcast(block, r)
        if group.rank != r:
            sess.set_rows(n, lo, block)


def factor_epoch_sharded(sess, group: Group, fh) -> None:
    """update_factor_epoch (factor_optimizer.cpp:101-273) over P ranks."""
    R = sess.R
    for n in range(sess.order):
        rows, g = sess.factor_mode_local(n, fh)
        merged = merge_boundary(group.all_gather(pack_boundary(rows, g, R)), R)
        mine = [int(r) for r in rows]
        if mine:
            sess.factor_mode_finish(n, fh, np.array(mine, np.uint32), np.stack([merged[r] for r in mine]))
        info = sess.shard_info(n)
        ranges = [(int(a[0]), int(a[1])) for a in group.all_gather(np.array([info.row_lo, info.row_hi], np.int64))]
        publish_rows(sess, group, n, ranges)
        sess.refresh_q(n)


def run_epochs_sharded(sess, group: Group, ch, fh, epochs: int = 1) -> None:
    """`epochs` x (replicated core phase; sharded factor phase)."""
    for _ in range(epochs):
        sess.core_epoch(ch.lr, ch.reg, ch.batch_m, bool(ch.resample_per_mode), bool(ch.incremental_residual))
        factor_epoch_sharded(sess, group, fh)


# ----------------------------------------------------------------------------
# peer-memory publication: the finaliser's stores are the all-gather
# ----------------------------------------------------------------------------
def connect_peers(sess, group: Group) -> None:
    """Give every rank the other ranks' A^(n)/Q^(n)/record buffers.  Ranks in
    one process (ThreadGroup) exchange raw device pointers; ranks in separate
    processes exchange CUDA IPC handles and map them (sgdt_ipc_open)."""
    if isinstance(group, ThreadGroup):
        table = group.all_gather(np.array(sess.peer_buffers(), np.uint64))
        sess.set_peers([[int(p) for p in row] for row in table])
        return
    L = _bind()
    handles = group.all_gather(sess.peer_ipc_handles())
    own = sess.peer_buffers()
    dev = sess.device if hasattr(sess, "device") else -1
    table = []
    for r, hs in enumerate(handles):
        if r == group.rank:
            table.append(own)
            continue
        row = []
        for i in range(sess.n_peer_buffers):
            p = C.c_void_p()
            h = np.ascontiguousarray(hs[i * 64:(i + 1) * 64], np.uint8)
            sgdt._ck(L.sgdt_ipc_open(h.ctypes.data_as(C.c_void_p), dev, C.byref(p)))
            row.append(int(p.value))
        table.append(row)
    sess.set_peers(table)


def factor_epoch_p2p(sess, group: Group, fh) -> None:
    """update_factor_epoch over P ranks with peer-memory publication: per
    mode, the local pass (every finalised row stored into every rank's A^(n)
    and Q^(n), the cut rows' partials into every rank's record slot), a
    barrier, the owner's merge + finalisation of its cut row (stored
    everywhere), a barrier.  No host round trip, no broadcast, no Q refresh.
    The leading barrier orders the peers' stores after every rank's core
    phase, which reads every A^(k) row and rewrites every Q^(k) row."""
    group.stream_barrier(sess)
    for n in range(sess.order):
        sess.factor_mode_p2p(n, fh)
        group.stream_barrier(sess)
        sess.factor_merge_p2p(n, fh)
        group.stream_barrier(sess)


def core_epoch_sharded(sess, group: Group, ch, block: int = 0) -> int:
    """update_core_epoch (core_optimizer.cpp:112-257) over P ranks: each rank
    reduces its Psi slice per column block and publishes the block vector into
    every rank's exchange slot (P2P stores by the producing kernel); a
    barrier separates the steps, and the next step sums the slots in rank
    order.  Backends without peer memory (the CPU stand-in) exchange the
    vectors through the group instead.  Returns T."""
    steps, T = sess.core_plan(ch, block)
    host = getattr(sess, "core_exchange_host", False)
    for k in range(steps):
        sess.core_step(k)
        if k + 1 < steps and group.world > 1:
            if host:
                sess.core_receive(group.all_gather(sess.core_vector()))
            else:
                group.stream_barrier(sess)
    return T


def run_epochs_p2p(sess, group: Group, ch, fh, epochs: int = 1, core: str = "replicated",
                   block: int = 0) -> None:
    """`epochs` x (core phase, replicated or sharded; peer-published sharded
    factor phase), one host synchronisation (the numeric check) at the end."""
    if core not in ("replicated", "sharded"):
        raise ValueError(f"core must be 'replicated' or 'sharded', not {core!r}")
    if not getattr(sess, "peers_set", False):
        connect_peers(sess, group)
    for e in range(epochs):
        if core == "sharded":
            core_epoch_sharded(sess, group, ch, block)
        else:
            sess.core_epoch_async(ch)
        if e + 1 < epochs:  # next epoch's Psi on the side stream, under this factor phase
            sess.sample_ahead(ch)
        factor_epoch_p2p(sess, group, fh)
    sess.check()

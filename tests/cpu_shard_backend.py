"""CPU stand-in for a sharded device session -- TEST INFRASTRUCTURE ONLY.

It implements the sharded-session surface that distributed.py drives
(shard_info / factor_mode_local / factor_mode_finish / get_rows / set_rows /
refresh_q) in numpy fp64 with the Kruskal route, so the multi-rank
orchestration (slices, boundary export, rank-ordered merge, row publication)
can be exercised under torch.distributed gloo on CPU, where no GPU exists.

It also restates the blocked / sharded core phase (sgdt_core_blocked.cu,
sgdt.h "sharded core phase") in numpy fp64: Psi from the oracle sampler,
this rank's partition_even(M, P) slice, per column block the vector of V0
and the in-block Gram matrices, the rank-ordered sum and the T Gauss-Seidel
column steps.  Vectors travel through the group (core_exchange_host), since
there is no peer memory on CPU.
"""
from __future__ import annotations

import numpy as np


class _Info:
    def __init__(self, **kw):
        self.__dict__.update(kw)


def partition_even(count, workers):
    base, rem = divmod(count, workers)
    out, at = [], 0
    for w in range(workers):
        ln = base + (1 if w < rem else 0)
        out.append((at, at + ln))
        at += ln
    return out


class CpuShard:
    row_dtype = np.float64

    def __init__(self, dims, coords, values, J, R, rank, world, A, B):
        self.dims = [int(d) for d in dims]
        self.order = len(dims)
        self.coords = np.asarray(coords, np.int64).reshape(-1, self.order) - 1
        self.values = np.asarray(values, np.float64)
        self.J = np.asarray(J)
        self.R = int(R)
        self.rank, self.world = rank, world
        self.A = [np.array(a, np.float64) for a in A]
        self.B = [np.array(b, np.float64) for b in B]
        nnz = len(self.values)
        self.perm, self.off = [], []
        for n in range(self.order):
            p = np.argsort(self.coords[:, n], kind="stable")
            self.perm.append(p)
            cnt = np.bincount(self.coords[:, n], minlength=self.dims[n])
            self.off.append(np.concatenate([[0], np.cumsum(cnt)]))
        self.slices = [partition_even(nnz, world)[rank] for _ in range(self.order)]

    # -- the sharded-session surface --------------------------------------
    def shard_info(self, n):
        qb, qe = self.slices[n]
        off = self.off[n]
        if qb >= qe:
            return _Info(row_lo=0, row_hi=0, n_export=0, export_rows=[0, 0])
        r0 = int(np.searchsorted(off, qb, side="right") - 1)
        r1 = int(np.searchsorted(off, qe - 1, side="right") - 1)
        rows = []
        for r in sorted({r0, r1}):
            if off[r] < qb or off[r + 1] > qe:
                rows.append(r)
        return _Info(row_lo=r0 + 1 if off[r0] < qb else r0, row_hi=r1 + 1, n_export=len(rows),
                     export_rows=rows + [0] * (2 - len(rows)))

    def _q(self, k):
        return self.A[k] @ self.B[k]

    def _finalize(self, n, row, g, fh):
        cnt = self.off[n][row + 1] - self.off[n][row]
        a = self.A[n][row]
        F = self.B[n] @ g
        self.A[n][row] = a - fh.lr * (F / cnt + fh.reg * a)

    def factor_mode_local(self, n, fh):
        qb, qe = self.slices[n]
        info = self.shard_info(n)
        if qb >= qe:
            return np.zeros(0, np.uint32), np.zeros((0, self.R))
        ids = self.perm[n][qb:qe]
        rows = self.coords[ids, n]
        c = np.ones((len(ids), self.R))
        for k in range(self.order):
            if k != n:
                c *= self._q(k)[self.coords[ids, k]]
        p = (self._q(n)[rows] * c).sum(1)
        v = (p - self.values[ids])[:, None] * c
        starts = np.flatnonzero(np.concatenate([[True], rows[1:] != rows[:-1]]))
        sums = np.add.reduceat(v, starts, axis=0)
        exported = list(info.export_rows[: info.n_export])
        out_g = []
        for row, g in zip(rows[starts], sums):
            if int(row) in exported:
                out_g.append((int(row), g))
            else:
                self._finalize(n, int(row), g, fh)
        out_g.sort(key=lambda t: exported.index(t[0]))
        return np.array([r for r, _ in out_g], np.uint32), np.array([g for _, g in out_g]).reshape(-1, self.R)

    def factor_mode_finish(self, n, fh, rows, g):
        for row, gg in zip(rows, g):
            self._finalize(n, int(row), np.asarray(gg, np.float64), fh)

    def get_rows(self, n, lo, hi):
        return self.A[n][lo:hi].copy()

    def set_rows(self, n, lo, block):
        self.A[n][lo:lo + block.shape[0]] = block

    def refresh_q(self, n):
        pass  # Q is recomputed from A on demand

    # -- peer-memory publication (emulated: peers are in-process objects) ---
    _registry: dict = {}

    @property
    def n_peer_buffers(self):
        return 2 * self.order + 2

    def peer_buffers(self):
        tok = id(self)
        CpuShard._registry[tok] = self
        return [tok] * self.n_peer_buffers

    def set_peers(self, table):
        self.peers = [CpuShard._registry[int(row[0])] for r, row in enumerate(table) if r != self.rank]
        self.rec = {}
        self.peers_set = True

    def synchronize(self):
        pass

    def _publish_row(self, n, row):
        for p in self.peers:
            p.A[n][row] = self.A[n][row]

    def factor_mode_p2p(self, n, fh):
        rows, g = self.factor_mode_local(n, fh)
        info = self.shard_info(n)
        qb, qe = self.slices[n]
        if qb < qe:  # every row this rank finalised locally, published
            ids = self.perm[n][qb:qe]
            for row in np.unique(self.coords[ids, n]):
                if int(row) not in list(info.export_rows[: info.n_export]):
                    self._publish_row(n, int(row))
        record = (list(int(r) for r in rows), [np.array(x) for x in g])
        for dst in [self] + self.peers:
            dst.rec[self.rank] = record

    def factor_merge_p2p(self, n, fh):
        info = self.shard_info(n)
        own = [int(r) for r in info.export_rows[: info.n_export] if info.row_lo <= r < info.row_hi]
        for row in own:
            g = None
            for w in range(self.world):
                rows, gs = self.rec.get(w, ([], []))
                for r, gg in zip(rows, gs):
                    if r == row:
                        g = gg.copy() if g is None else g + gg
            self._finalize(n, row, g, fh)
            self._publish_row(n, row)

    # -- sharded core phase (numpy fp64 restatement of sgdt_core_blocked.cu) --
    core_exchange_host = True

    def seed(self, seed):
        from oracle import oracle_py as O
        self.rng = O.Rng(seed)
        self.ws = O.CoreWorkspace(len(self.values))

    def core_plan(self, ch, block=0):
        from oracle import oracle_py as O
        nnz = len(self.values)
        m = int(ch.batch_m) or nnz
        if ch.batch_m:
            self.psi = O.sample_batch(nnz, m, self.rng, self.ws).astype(np.int64)
        else:
            self.psi = np.arange(nnz)
        self.m = m
        self.lo, self.hi = partition_even(m, self.world)[self.rank]
        self.lr, self.reg = float(ch.lr), float(ch.reg)
        T = min(int(block) if block else self.R, self.R)
        self.T = T
        self.blocks = [(n, r0, min(T, self.R - r0)) for n in range(self.order) for r0 in range(0, self.R, T)]
        self.steps = len(self.blocks) + 1
        self._vec, self._sum = None, None
        return self.steps, T

    def _block_vector(self, n, r0, T):
        ids = self.psi[self.lo:self.hi]
        co = self.coords[ids]
        c = np.ones((len(ids), self.R))
        for k in range(self.order):
            if k != n:
                c *= self.A[k][co[:, k]] @ self.B[k]
        a = self.A[n][co[:, n]]
        xhat = (c * (a @ self.B[n])).sum(1)
        res = xhat - self.values[ids]
        cb = c[:, r0:r0 + T]
        V0 = np.einsum("st,s,sj->tj", cb, res, a)
        G = np.einsum("st,su,sj,sk->tujk", cb, cb, a, a)
        return np.concatenate([V0.ravel(), G.ravel()])

    def _replay(self, n, r0, T, v):
        J = int(self.J[n])
        V0 = v[:T * J].reshape(T, J)
        G = v[T * J:].reshape(T, T, J, J)
        db = np.zeros((T, J))
        for t in range(T):
            V = V0[t] + sum(G[t, u] @ db[u] for u in range(t))
            old = self.B[n][:, r0 + t].copy()
            self.B[n][:, r0 + t] = old - self.lr * (V / self.m + self.reg * old)
            db[t] = self.B[n][:, r0 + t] - old

    def core_step(self, k):
        if k > 0:
            v = self._sum if self._sum is not None else self._vec
            self._replay(*self.blocks[k - 1], v)
            self._sum = None
        self._vec = self._block_vector(*self.blocks[k]) if k + 1 < self.steps else None

    def core_vector(self):
        return self._vec

    def core_receive(self, vecs):
        acc = np.zeros_like(vecs[0])
        for v in vecs:  # ascending rank
            acc = acc + v
        self._sum = acc

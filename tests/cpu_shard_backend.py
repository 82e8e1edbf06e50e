"""CPU stand-in for a sharded device session -- TEST INFRASTRUCTURE ONLY.

It implements the sharded-session surface that distributed.py drives
(shard_info / factor_mode_local / factor_mode_finish / get_rows / set_rows /
refresh_q) in numpy fp64 with the Kruskal route, so the multi-rank
orchestration (slices, boundary export, rank-ordered merge, row publication)
can be exercised under torch.distributed gloo on CPU, where no GPU exists.
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
        return 2 * self.order + 1

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

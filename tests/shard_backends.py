"""CPU shard backend for testing paper_1802_00330_b200.dist.solve_sharded under gloo.

TEST INFRASTRUCTURE: restates one rank's round operations with the oracle
(oracle/rootbox_oracle.c) and numpy, with the same interface as
dist.CudaShardBackend, so the multi-rank driver logic (global HS trigger,
owner routing, global dedup, statistics and termination) is exercised on CPU.
"""
import numpy as np

from oracle import oracle as O
from paper_1802_00330_b200.dist import row_owner, thin_rows


def _width(lo, hi):
    return (hi - lo).max(axis=1) if lo.shape[0] else np.zeros(0)


def _mid(lo, hi):
    m = 0.5 * (lo + hi)
    bad = np.isinf(m)
    if bad.any():
        m = np.where(bad, 0.5 * lo + 0.5 * hi, m)
    return np.clip(m, lo, hi)


class OracleShardBackend:
    device_exchange = False
    device = -1

    def __init__(self, spec, jac):
        self.n = spec.n
        self.osys = O.OSystem(spec.n, spec.eqs, jac)
        self.lo = np.zeros((0, self.n)); self.hi = np.zeros((0, self.n))
        self.c = np.zeros(0, bool); self.u = np.zeros(0, bool)

    def load(self, lo, hi, cert, uns, target):
        self.lo = np.asarray(lo, float).reshape(-1, self.n).copy()
        self.hi = np.asarray(hi, float).reshape(-1, self.n).copy()
        self.c = np.asarray(cert).astype(bool).copy(); self.u = np.asarray(uns).astype(bool).copy()
        self.target = target

    def size(self):
        return self.lo.shape[0]

    def round_filter(self, round_no):
        done = (_width(self.lo, self.hi) <= self.target) | self.u
        alo, ahi = self.lo[~done], self.hi[~done]
        m = _mid(alo, ahi)
        deg = ((m == alo) | (m == ahi)).any(axis=1) if alo.shape[0] else np.zeros(0, bool)
        self.keep = (np.concatenate([self.lo[done], alo[deg]]), np.concatenate([self.hi[done], ahi[deg]]),
                     np.concatenate([self.c[done], np.zeros(deg.sum(), bool)]),
                     np.concatenate([self.u[done], np.ones(deg.sum(), bool)]))
        plo, phi = alo[~deg], ahi[~deg]
        if plo.shape[0]:
            slo, shi = self.osys.chunk_filter(plo, phi)
        else:
            slo, shi = np.zeros((0, self.n)), np.zeros((0, self.n))
        self.surv = (slo, shi)
        cw = float(_width(slo, shi).max()) if slo.shape[0] else 0.0
        return self.keep[0].shape[0], slo.shape[0], cw, plo.shape[0] << self.n

    def round_hs(self, hs_on, contract):
        slo, shi = self.surv
        calls = 0
        if hs_on and slo.shape[0]:
            slo, shi, sc = self.osys.hs_pass(slo, shi, contract)
            calls = self.surv[0].shape[0]
        else:
            sc = np.zeros(slo.shape[0], bool)
        klo, khi, kc, ku = self.keep
        self.lo = np.concatenate([klo, slo]); self.hi = np.concatenate([khi, shi])
        self.c = np.concatenate([kc, sc]); self.u = np.concatenate([ku, np.zeros(slo.shape[0], bool)])
        w = float(_width(self.lo, self.hi).max()) if self.lo.shape[0] else 0.0
        return self.lo.shape[0], w, calls

    def route_count(self, world):
        """rb_shard_route_count: thin rows per hash owner, count of the others."""
        self._thin = thin_rows(self.lo, self.hi)
        own = row_owner(self.lo, self.hi, world) if self.lo.shape[0] else np.zeros(0, np.int64)
        self._dest = np.where(self._thin, own, -1)
        thin = np.bincount(own[self._thin], minlength=world).astype(np.int64)
        return thin, int((~self._thin).sum())

    def route(self, world, rank, move):
        """rb_shard_route: non-thin rows fill move[d] in rank order (the device takes
        them in any order; the solve does not depend on which rows move), the rest
        stay; rows ordered [own | rank 0 | rank 1 | ...]."""
        dest = self._dest.copy()
        free = np.nonzero(dest < 0)[0]
        k = 0
        for d in range(world):
            m = 0 if d == rank else int(move[d])
            dest[free[k:k + m]] = d
            k += m
        dest[dest < 0] = rank
        key = np.where(dest == rank, -1, dest)
        order = np.argsort(key, kind="stable")
        self.lo, self.hi, self.c, self.u = self.lo[order], self.hi[order], self.c[order], self.u[order]
        return np.bincount(dest, minlength=world).astype(np.int64)

    def export_packed(self, torch, start, count):
        s = slice(start, start + count)
        f = (self.c[s].astype(np.float64) + 2.0 * self.u[s].astype(np.float64)).reshape(-1, 1)
        return torch.from_numpy(np.concatenate([self.lo[s], self.hi[s], f], axis=1))

    def import_packed(self, torch, keep, rows):
        r = rows.numpy()
        n = self.n
        self.lo = np.concatenate([self.lo[:keep], r[:, :n]]); self.hi = np.concatenate([self.hi[:keep], r[:, n:2 * n]])
        self.c = np.concatenate([self.c[:keep], np.remainder(r[:, 2 * n], 2.0) == 1.0])
        self.u = np.concatenate([self.u[:keep], np.floor(r[:, 2 * n] / 2.0) == 1.0])

    def dedup(self):
        n = self.n
        N = self.lo.shape[0]
        if N == 0:
            return 0, 0.0
        keys = tuple(self.hi[:, i] for i in reversed(range(n))) + tuple(self.lo[:, i] for i in reversed(range(n)))
        o = np.lexsort(keys)
        lo, hi, c, u = self.lo[o], self.hi[o], self.c[o], self.u[o]
        same = np.all(lo[1:] == lo[:-1], axis=1) & np.all(hi[1:] == hi[:-1], axis=1)
        starts = np.nonzero(np.concatenate(([True], ~same)))[0]
        self.lo, self.hi = lo[starts], hi[starts]
        self.c = np.logical_or.reduceat(c, starts); self.u = np.logical_or.reduceat(u, starts)
        return N - starts.size, float(_width(self.lo, self.hi).max())

    def finalize(self):
        n = self.n
        keys = tuple(self.hi[:, i] for i in reversed(range(n))) + tuple(self.lo[:, i] for i in reversed(range(n)))
        o = np.lexsort(keys) if self.lo.shape[0] else np.zeros(0, np.int64)
        return self.lo[o], self.hi[o], self.c[o], self.u[o]

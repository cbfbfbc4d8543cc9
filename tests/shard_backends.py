"""CPU shard backend for testing paper_1802_00330_b200.dist.solve_sharded under gloo.

TEST INFRASTRUCTURE: restates one rank's round operations with the oracle
(oracle/rootbox_oracle.c) and numpy, with the same interface as
dist.CudaShardBackend, so the multi-rank driver logic (global HS trigger,
owner routing, global dedup, statistics and termination) is exercised on CPU.
"""
import numpy as np

from oracle import oracle as O
from paper_1802_00330_b200.dist import row_owner


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

    def partition(self, world):
        own = row_owner(self.lo, self.hi, world) if self.lo.shape[0] else np.zeros(0, np.int64)
        order = np.argsort(own, kind="stable")
        self.lo, self.hi, self.c, self.u = self.lo[order], self.hi[order], self.c[order], self.u[order]
        return np.bincount(own, minlength=world).astype(np.int64)

    def export_rows(self, torch, start, count):
        s = slice(start, start + count)
        fl = np.stack([self.c[s], self.u[s]], axis=1).astype(np.uint8)
        return (torch.from_numpy(np.ascontiguousarray(self.lo[s])), torch.from_numpy(np.ascontiguousarray(self.hi[s])),
                torch.from_numpy(np.ascontiguousarray(fl)))

    def import_rows(self, torch, keep, lo, hi, fl):
        fl = fl.numpy()
        self.lo = np.concatenate([self.lo[:keep], lo.numpy()]); self.hi = np.concatenate([self.hi[:keep], hi.numpy()])
        self.c = np.concatenate([self.c[:keep], fl[:, 0].astype(bool)])
        self.u = np.concatenate([self.u[:keep], fl[:, 1].astype(bool)])

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

    def export_host(self):
        return self.lo, self.hi, self.c, self.u

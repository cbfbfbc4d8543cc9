"""Frontier sharding across GPUs (one process per GPU, torch.distributed).

``solve_sharded(s, cfg)`` runs rootbox.bnb.solve (bnb.py:224-354) with the
frontier partitioned across the ranks of the default process group.  Boxes are
independent inside a round (the paper's "no message communication ... between
different threads"), so each rank runs the same kernels as
``rb_solve`` on its own rows.  The exchanges are exactly the reference's global
decisions plus an ownership shuffle:

  1. after the filter: all-reduce of the survivor count and their max width
     -> the HS trigger (bnb.py:289-296) is decided identically on every rank;
  2. after HS: every row moves to its owner rank = row_hash(row) % world
     (all_to_all).  Exact duplicates therefore always meet on one shard, so the
     per-shard dedup is the global dedup (bnb.py:322-326), and the hash spreads
     the frontier evenly (the rebalancing of SURVEY §8(e));
  3. all-reduce of the round statistics -> RoundStats and the termination test
     (bnb.py:339-352) are global; max_seconds is decided by rank 0's clock.

The final frontier is gathered on rank 0 and put in canonical order
(_batch.canonical_order, _batch.py:244-250).  With NCCL the rows travel as
device tensors (rb_shard_export_device / rb_shard_import_device); with gloo
through host memory.
"""
from __future__ import annotations

import ctypes as C
import math
import time

import numpy as np

from . import _native
from .bnb import (BUDGET_EXHAUSTED, NO_REAL_SOLUTION, WIDTH_REACHED, Box, Interval, RootBox, RoundStats,
                  SolveResult, SolverConfig, native_config, validate_config)
from .system import as_spec, compile_tables

__all__ = ["solve_sharded", "CudaShardBackend", "row_owner"]

_M1 = np.uint64(0xFF51AFD7ED558CCD)
_M2 = np.uint64(0xC4CEB9FE1A85EC53)
_SEED = np.uint64(0x9E3779B97F4A7C15)


def _mix64(x):
    x = x ^ (x >> np.uint64(33))
    x = x * _M1
    x = x ^ (x >> np.uint64(33))
    x = x * _M2
    x = x ^ (x >> np.uint64(33))
    return x


def row_owner(lo: np.ndarray, hi: np.ndarray, world: int) -> np.ndarray:
    """Owner rank of each row (row-major lo/hi) -- the host twin of the device
    row_hash (kernels.cuh): mix64 over the canonical (+0.0) bit patterns,
    lo_j then hi_j for j ascending."""
    lo = np.where(lo == 0.0, 0.0, lo)
    hi = np.where(hi == 0.0, 0.0, hi)
    lb = np.ascontiguousarray(lo, np.float64).view(np.uint64)
    hb = np.ascontiguousarray(hi, np.float64).view(np.uint64)
    h = np.full(lo.shape[0], _SEED, dtype=np.uint64)
    with np.errstate(over="ignore"):
        for j in range(lo.shape[1]):
            h = _mix64(h ^ lb[:, j])
            h = _mix64(h ^ hb[:, j])
    return (h % np.uint64(world)).astype(np.int64)


class CudaShardBackend:
    """One rank's shard on its GPU (librootbox_b200.so handle)."""

    def __init__(self, spec, device: int = 0, device_exchange: bool = True):
        self.n = spec.n
        self.device = device
        self.eng = _native.Engine(compile_tables(spec), device)
        self.device_exchange = device_exchange
        self._L = _native.lib()

    def _ck(self, rc, what):
        _native._check(rc, self.eng.h, what)

    def load(self, lo, hi, cert, uns, target):
        lo = np.ascontiguousarray(lo, np.float64).reshape(-1, self.n)
        hi = np.ascontiguousarray(hi, np.float64).reshape(-1, self.n)
        c = np.ascontiguousarray(cert, np.uint8)
        u = np.ascontiguousarray(uns, np.uint8)
        p = _native._p
        self._ck(self._L.rb_shard_load(self.eng.h, p(lo), p(hi), p(c), p(u), lo.shape[0], float(target)),
                 "rb_shard_load")

    def size(self) -> int:
        return int(self._L.rb_shard_size(self.eng.h))

    def round_filter(self, round_no):
        car, surv, ch = C.c_int64(), C.c_int64(), C.c_int64()
        cw = C.c_double()
        self._ck(self._L.rb_round_filter(self.eng.h, int(round_no), C.byref(car), C.byref(surv), C.byref(cw),
                                         C.byref(ch)), "rb_round_filter")
        return car.value, surv.value, cw.value, ch.value

    def round_hs(self, hs_on, contract):
        n_out, calls = C.c_int64(), C.c_int64()
        w = C.c_double()
        self._ck(self._L.rb_round_hs(self.eng.h, int(bool(hs_on)), int(bool(contract)), C.byref(n_out), C.byref(w),
                                     C.byref(calls)), "rb_round_hs")
        return n_out.value, w.value, calls.value

    def partition(self, world):
        counts = np.zeros(world, np.int64)
        self._ck(self._L.rb_shard_partition(self.eng.h, int(world), _native._p(counts)), "rb_shard_partition")
        return counts

    def dedup(self):
        d = C.c_int64()
        w = C.c_double()
        self._ck(self._L.rb_shard_dedup(self.eng.h, C.byref(d), C.byref(w)), "rb_shard_dedup")
        return d.value, w.value

    # -- row transport (torch tensors: CUDA for NCCL, CPU for gloo)
    def export_rows(self, torch, start, count):
        n = self.n
        if self.device_exchange:
            dev = torch.device("cuda", self.device)
            lo = torch.empty((count, n), dtype=torch.float64, device=dev)
            hi = torch.empty((count, n), dtype=torch.float64, device=dev)
            fl = torch.empty((count, 2), dtype=torch.uint8, device=dev)
            if count:
                torch.cuda.synchronize(dev)
                self._ck(self._L.rb_shard_export_device(self.eng.h, start, count, C.c_void_p(lo.data_ptr()),
                                                        C.c_void_p(hi.data_ptr()), C.c_void_p(fl.data_ptr()),
                                                        C.c_void_p(fl.data_ptr() + count)), "export")
            # cert / unsplit were written as two planes; present them as columns
            fl = fl.reshape(2, count).t().contiguous() if count else fl
            return lo, hi, fl
        lo = np.empty((count, n)); hi = np.empty((count, n))
        c = np.empty(count, np.uint8); u = np.empty(count, np.uint8)
        if count:
            p = _native._p
            self._ck(self._L.rb_shard_export(self.eng.h, start, count, p(lo), p(hi), p(c), p(u)), "export")
        fl = np.stack([c, u], axis=1) if count else np.zeros((0, 2), np.uint8)
        return torch.from_numpy(lo), torch.from_numpy(hi), torch.from_numpy(np.ascontiguousarray(fl))

    def import_rows(self, torch, keep, lo, hi, fl):
        count = int(lo.shape[0])
        if self.device_exchange:
            if count:
                planes = fl.t().contiguous()  # [2, count]: cert plane then unsplit plane
                torch.cuda.synchronize(lo.device)
                self._ck(self._L.rb_shard_import_device(self.eng.h, keep, C.c_void_p(lo.data_ptr()),
                                                        C.c_void_p(hi.data_ptr()), C.c_void_p(planes.data_ptr()),
                                                        C.c_void_p(planes.data_ptr() + count), count), "import")
            else:
                self._ck(self._L.rb_shard_import_device(self.eng.h, keep, None, None, None, None, 0), "import")
            return
        p = _native._p
        lo = np.ascontiguousarray(lo.numpy()); hi = np.ascontiguousarray(hi.numpy())
        fl = np.ascontiguousarray(fl.numpy())
        c = np.ascontiguousarray(fl[:, 0]); u = np.ascontiguousarray(fl[:, 1])
        self._ck(self._L.rb_shard_import(self.eng.h, keep, p(lo) if count else None, p(hi) if count else None,
                                         p(c) if count else None, p(u) if count else None, count), "import")

    def export_host(self):
        n, N = self.n, self.size()
        lo = np.empty((N, n)); hi = np.empty((N, n)); c = np.empty(N, np.uint8); u = np.empty(N, np.uint8)
        if N:
            p = _native._p
            self._ck(self._L.rb_shard_export(self.eng.h, 0, N, p(lo), p(hi), p(c), p(u)), "export")
        return lo, hi, c.astype(bool), u.astype(bool)


def _exchange(torch, dist, backend, world, counts, group):
    """Route rows to their owners: all_to_all of (lo, hi, flags)."""
    total = int(counts.sum())
    dev = torch.device("cuda", backend.device) if getattr(backend, "device_exchange", False) else torch.device("cpu")
    send_counts = torch.tensor(counts, dtype=torch.int64, device=dev)
    recv_counts = torch.empty_like(send_counts)
    dist.all_to_all_single(recv_counts, send_counts, group=group)
    rc = [int(v) for v in recv_counts.tolist()]
    sc = [int(v) for v in counts.tolist()]
    lo, hi, fl = backend.export_rows(torch, 0, total)
    rlo = torch.empty((sum(rc), backend.n), dtype=torch.float64, device=lo.device)
    rhi = torch.empty_like(rlo)
    rfl = torch.empty((sum(rc), 2), dtype=torch.uint8, device=lo.device)
    dist.all_to_all_single(rlo, lo, rc, sc, group=group)
    dist.all_to_all_single(rhi, hi, rc, sc, group=group)
    dist.all_to_all_single(rfl, fl, rc, sc, group=group)
    backend.import_rows(torch, 0, rlo, rhi, rfl)


def solve_sharded(s, cfg=None, backend=None, group=None, device: int | None = None):
    """bnb.solve over the ranks of `group` (default: the world).  Every rank
    calls it; rank 0 returns the SolveResult (canonical order), others None."""
    import torch
    import torch.distributed as dist
    cfg = cfg or SolverConfig()
    validate_config(cfg)
    spec = as_spec(s)
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if backend is None:
        dev = device if device is not None else (torch.cuda.current_device() if torch.cuda.is_available() else 0)
        nccl = dist.is_initialized() and dist.get_backend(group) == "nccl"
        backend = CudaShardBackend(spec, dev, device_exchange=nccl or not dist.is_initialized())
    comm_dev = (torch.device("cuda", backend.device) if getattr(backend, "device_exchange", False)
                else torch.device("cpu"))

    def allreduce(vals, op):
        t = torch.tensor(vals, dtype=torch.float64, device=comm_dev)
        if world > 1:
            dist.all_reduce(t, op=op, group=group)
        return t.tolist()

    SUM = dist.ReduceOp.SUM if dist.is_initialized() else None
    MAX = dist.ReduceOp.MAX if dist.is_initialized() else None
    n = spec.n
    ilo, ihi = spec.init_lo, spec.init_hi
    init_width = float(np.max(ihi - ilo))
    target = cfg.target_width if cfg.target_width is not None else init_width * 2.0 ** -10
    hs_possible = cfg.hs_enable_round is not None or cfg.hs_enable_width is not None
    if init_width <= target:
        if rank != 0:
            return None
        return SolveResult(WIDTH_REACHED, (RootBox(Box.from_bounds(ilo, ihi), False, False),), ())
    if rank == 0:
        backend.load(ilo.reshape(1, n), ihi.reshape(1, n), np.zeros(1, np.uint8), np.zeros(1, np.uint8), target)
    else:
        backend.load(np.zeros((0, n)), np.zeros((0, n)), np.zeros(0, np.uint8), np.zeros(0, np.uint8), target)
    stats = []
    status = BUDGET_EXHAUSTED
    t_start = time.perf_counter()
    for round_no in range(1, cfg.max_rounds + 1):
        t0 = time.perf_counter()
        n_in = backend.size()
        carried, surv, cw, children = backend.round_filter(round_no)
        g_in, g_after_filter, g_surv = allreduce([n_in, carried + surv, surv], SUM)
        (g_cw,) = allreduce([cw if surv > 0 else 0.0], MAX)
        hs_on = False
        if g_surv > 0 and hs_possible:  # bnb.py:289-296 on the global survivors
            if cfg.hs_enable_round is not None and round_no >= cfg.hs_enable_round:
                hs_on = True
            if cfg.hs_enable_width is not None and g_cw <= cfg.hs_enable_width:
                hs_on = True
        backend.round_hs(hs_on, cfg.hs_contract)
        counts = backend.partition(world)
        if world > 1:
            _exchange(torch, dist, backend, world, counts, group)
        _dups, width = backend.dedup()
        after_local = backend.size()
        (g_after,) = allreduce([after_local], SUM)
        (g_width,) = allreduce([width if after_local else 0.0], MAX)
        stop_clock = 0.0
        if rank == 0 and cfg.max_seconds is not None and time.perf_counter() - t_start > cfg.max_seconds:
            stop_clock = 1.0
        (stop_clock,) = allreduce([stop_clock], MAX)
        stats.append(RoundStats(round=round_no, boxes_in=int(g_in), boxes_after_filter=int(g_after_filter),
                                boxes_after_hs=int(g_after), width=float(g_width) if g_after else 0.0,
                                elapsed_seconds=time.perf_counter() - t0))
        if g_after == 0:
            status = NO_REAL_SOLUTION
            break
        if g_width <= target:
            status = WIDTH_REACHED
            break
        if g_after > cfg.max_boxes:
            status = BUDGET_EXHAUSTED
            break
        if stop_clock:
            status = BUDGET_EXHAUSTED
            break
    # gather the final frontier on rank 0
    lo, hi, c, u = backend.export_host()
    if world > 1:
        parts = [None] * world if rank == 0 else None
        dist.gather_object((lo, hi, c, u), parts, dst=0, group=group)
        if rank != 0:
            return None
        lo = np.concatenate([p[0] for p in parts]).reshape(-1, n)
        hi = np.concatenate([p[1] for p in parts]).reshape(-1, n)
        c = np.concatenate([p[2] for p in parts])
        u = np.concatenate([p[3] for p in parts])
    keys = tuple(hi[:, i] for i in reversed(range(n))) + tuple(lo[:, i] for i in reversed(range(n)))
    order = np.lexsort(keys) if lo.shape[0] else np.zeros(0, np.int64)
    lo, hi, c, u = lo[order], hi[order], c[order], u[order]
    boxes = tuple(RootBox(Box(tuple(Interval(a, b) for a, b in zip(lo[r].tolist(), hi[r].tolist()))), bool(c[r]),
                          bool(u[r])) for r in range(lo.shape[0]))
    return SolveResult(status, boxes, tuple(stats))

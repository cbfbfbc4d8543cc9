"""Frontier sharding across GPUs (one process per GPU, torch.distributed).

``solve_sharded(s, cfg)`` runs rootbox.bnb.solve (bnb.py:224-354) with the
frontier partitioned across the ranks of a process group.  Boxes are
independent inside a round (the paper's "no message communication ... between
different threads"); the reference's only parallelism is a
thread pool over chunks of one frontier (bnb.py:183-187, 271-313).  Each rank
runs the engine's own round kernels on its rows; per round the ranks exchange:

  1. after the filter, one all_gather of (survivors, max survivor width, rows
     at round start): the global HS trigger (bnb.py:289-296) and the previous
     round's boxes_after_hs;
  2. after HS, one all_gather of (rows, max row width, thin rows per owner, other
     rows, rank 0's clock verdict): the termination test (bnb.py:339-352) and
     the routing plan, computed identically on every rank;
  3. only when the plan moves rows, one all_to_all of packed rows:
       - a row with a component at most 64 ulps wide goes to its hash owner
         (row_hash % world): only such rows can have an exact duplicate on
         another shard (kThinUlps, kernels.cuh), so the per-shard dedup that
         follows is the global dedup of bnb.py:322-326;
       - when the largest shard exceeds the smallest by more than 1.25x (or a
         shard is empty), the surplus over total/world moves to the deficit
         ranks in rank order.

The width of a round is invariant under moving rows and under removing exact
duplicates, so it comes from exchange 2; boxes_after_hs of round r is the sum of
the shard sizes at the start of round r + 1 (exchange 1), and one last
all_gather closes the final round.  The result is independent of the number of
ranks: rows are gathered on rank 0 and put in canonical order on its device
(rb_shard_finalize, _batch.canonical_order, _batch.py:244-250).

At world size 1 there is nothing to exchange and ``solve_sharded`` is the
engine's own solve (device-resident round loop).
"""
from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _native
from .bnb import (BUDGET_EXHAUSTED, NO_REAL_SOLUTION, WIDTH_REACHED, Box, RootBox, RoundStats, SolveResult,
                  SolverConfig, _own_result, _reference_types, native_config, validate_config)
from .system import as_spec, compile_tables

__all__ = ["solve_sharded", "CudaShardBackend", "row_owner", "rebalance_plan", "REBALANCE_RATIO"]

_M1 = np.uint64(0xFF51AFD7ED558CCD)
_M2 = np.uint64(0xC4CEB9FE1A85EC53)
_SEED = np.uint64(0x9E3779B97F4A7C15)
THIN_ULPS = 64          # kThinUlps (kernels.cuh)
REBALANCE_RATIO = 1.25  # move surplus rows when max/min shard size exceeds this


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


def _ordkey(x):
    b = np.ascontiguousarray(x, np.float64).view(np.int64)
    return np.where(b >= 0, b, np.int64(-0x8000000000000000) - b)


def thin_rows(lo: np.ndarray, hi: np.ndarray) -> np.ndarray:
    """Host twin of thin_comp (kernels.cuh): some component at most 64 ulps wide."""
    if lo.shape[0] == 0:
        return np.zeros(0, bool)
    return np.any(_ordkey(hi) - _ordkey(lo) <= THIN_ULPS, axis=1)


def rebalance_plan(sizes, movable, ratio: float = REBALANCE_RATIO):
    """move[r][d] = non-thin rows rank r sends to rank d so every shard is near
    total/world.  Runs identically on every rank from the all_gathered sizes.
    Nothing moves while max/min <= ratio and no shard is empty (or there are
    fewer rows than ranks)."""
    sizes = [int(v) for v in sizes]
    world = len(sizes)
    move = [[0] * world for _ in range(world)]
    total = sum(sizes)
    if world == 1 or total < world:
        return move
    if min(sizes) > 0 and max(sizes) <= ratio * min(sizes):
        return move
    target = [total // world + (1 if r < total % world else 0) for r in range(world)]
    give = [max(0, min(sizes[r] - target[r], int(movable[r]))) for r in range(world)]
    need = [max(0, target[r] - sizes[r]) for r in range(world)]
    d = 0
    for r in range(world):
        while give[r] > 0:
            while d < world and need[d] == 0:
                d += 1
            if d == world:
                return move
            k = min(give[r], need[d])
            move[r][d] += k
            give[r] -= k
            need[d] -= k
    return move


class CudaShardBackend:
    """One rank's shard on its GPU (librootbox_b200.so handle).  device_exchange:
    rows travel as CUDA tensors (NCCL); otherwise through host memory (gloo)."""

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

    def route_count(self, world):
        thin = np.zeros(world, np.int64)
        other = C.c_int64()
        self._ck(self._L.rb_shard_route_count(self.eng.h, int(world), _native._p(thin), C.byref(other)),
                 "rb_shard_route_count")
        return thin, other.value

    def route(self, world, rank, move):
        mv = np.ascontiguousarray(move, np.int64)
        sc = np.zeros(world, np.int64)
        self._ck(self._L.rb_shard_route(self.eng.h, int(world), int(rank), _native._p(mv), _native._p(sc)),
                 "rb_shard_route")
        return sc

    def dedup(self):
        d = C.c_int64()
        w = C.c_double()
        self._ck(self._L.rb_shard_dedup(self.eng.h, C.byref(d), C.byref(w)), "rb_shard_dedup")
        return d.value, w.value

    # -- rows as one packed [count, 2n + 1] float64 tensor: lo | hi | cert + 2 unsplit
    def export_packed(self, torch, start, count):
        n = self.n
        if self.device_exchange:
            dev = torch.device("cuda", self.device)
            lo = torch.empty((count, n), dtype=torch.float64, device=dev)
            hi = torch.empty((count, n), dtype=torch.float64, device=dev)
            fl = torch.empty((2, count), dtype=torch.uint8, device=dev)
            if count:
                torch.cuda.synchronize(dev)
                self._ck(self._L.rb_shard_export_device(self.eng.h, start, count, C.c_void_p(lo.data_ptr()),
                                                        C.c_void_p(hi.data_ptr()), C.c_void_p(fl.data_ptr()),
                                                        C.c_void_p(fl.data_ptr() + count)), "export")
            f = fl[0].to(torch.float64) + 2.0 * fl[1].to(torch.float64)
            return torch.cat([lo, hi, f.reshape(count, 1)], dim=1)
        lo = np.empty((count, n)); hi = np.empty((count, n))
        c = np.empty(count, np.uint8); u = np.empty(count, np.uint8)
        if count:
            p = _native._p
            self._ck(self._L.rb_shard_export(self.eng.h, start, count, p(lo), p(hi), p(c), p(u)), "export")
        f = (c.astype(np.float64) + 2.0 * u.astype(np.float64)).reshape(count, 1)
        return torch.from_numpy(np.concatenate([lo, hi, f], axis=1))

    def import_packed(self, torch, keep, rows):
        n = self.n
        count = int(rows.shape[0])
        lo = rows[:, :n].contiguous()
        hi = rows[:, n:2 * n].contiguous()
        f = rows[:, 2 * n]
        if self.device_exchange:
            planes = torch.stack([torch.remainder(f, 2.0), torch.floor(f / 2.0)]).to(torch.uint8).contiguous()
            torch.cuda.synchronize(rows.device)
            if count:
                self._ck(self._L.rb_shard_import_device(self.eng.h, keep, C.c_void_p(lo.data_ptr()),
                                                        C.c_void_p(hi.data_ptr()), C.c_void_p(planes.data_ptr()),
                                                        C.c_void_p(planes.data_ptr() + count), count), "import")
            else:
                self._ck(self._L.rb_shard_import_device(self.eng.h, keep, None, None, None, None, 0), "import")
            return
        p = _native._p
        lo = np.ascontiguousarray(lo.numpy()); hi = np.ascontiguousarray(hi.numpy())
        fv = f.numpy()
        c = np.ascontiguousarray(np.remainder(fv, 2.0).astype(np.uint8))
        u = np.ascontiguousarray(np.floor(fv / 2.0).astype(np.uint8))
        self._ck(self._L.rb_shard_import(self.eng.h, keep, p(lo) if count else None, p(hi) if count else None,
                                         p(c) if count else None, p(u) if count else None, count), "import")

    def finalize(self):
        """Canonical order of the shard's rows on the device; returns the result arrays."""
        nb = C.c_int64()
        with self.eng._lock:
            self._ck(self._L.rb_shard_finalize(self.eng.h, C.byref(nb)), "rb_shard_finalize")
            N, n = nb.value, self.n
            lo = np.empty((N, n)); hi = np.empty((N, n)); fl = np.empty((2, N), np.uint8)
            self._ck(self._L.rb_fetch(self.eng.h, lo.ctypes.data, hi.ctypes.data, fl.ctypes.data,
                                      fl[1].ctypes.data, None), "rb_fetch")
        return lo, hi, fl[0].astype(bool), fl[1].astype(bool)

    def solve_single(self, cfg):
        """World size 1: the engine's own solve (nothing to exchange)."""
        return self.eng.solve(native_config(cfg), stats_rows=True)


def _exchange(torch, dist, backend, rank, world, send, group):
    """One all_to_all of packed rows: send[d] rows to rank d, taken from the shard
    after its own rows (rb_shard_route order); received rows are appended."""
    keep = int(send[rank])
    sc = [0 if d == rank else int(send[d]) for d in range(world)]
    rows = backend.export_packed(torch, keep, sum(sc))
    return rows, sc, keep


def solve_sharded(s, cfg=None, backend=None, group=None, device: int | None = None, force_protocol=False,
                  arrays=False):
    """bnb.solve over the ranks of `group` (default: the world).  Every rank calls
    it; rank 0 returns the SolveResult (canonical order), the others None.  The
    boxes and statistics are those of the single-process solve, bit for bit.
    force_protocol: run the exchange protocol even at world size 1 (tests).  arrays:
    return the engine arrays and per-round statistics (with children and hs_calls)
    instead of SolveResult objects."""
    import torch
    import torch.distributed as dist
    cfg = cfg or SolverConfig()
    validate_config(cfg)
    spec = as_spec(s)
    on = dist.is_available() and dist.is_initialized()
    rank = dist.get_rank(group) if on else 0
    world = dist.get_world_size(group) if on else 1
    if world == 1 and backend is None and not force_protocol:  # the engine's own solve (cached engine)
        from .bnb import solve, solve_arrays
        return solve_arrays(s, cfg, device) if arrays else solve(s, cfg)
    if backend is None:
        dev = device if device is not None else (torch.cuda.current_device() if torch.cuda.is_available() else 0)
        nccl = on and dist.get_backend(group) == "nccl"
        backend = CudaShardBackend(spec, dev, device_exchange=nccl or not on)
    if world == 1 and hasattr(backend, "solve_single") and not force_protocol:
        if arrays:
            return backend.eng.solve(native_config(cfg))
        return _result(s, backend.solve_single(cfg))
    comm_dev = (torch.device("cuda", backend.device) if getattr(backend, "device_exchange", False)
                else torch.device("cpu"))

    def gather(vals):
        """all_gather of one float64 vector per rank -> [world, len] numpy array."""
        t = torch.tensor(vals, dtype=torch.float64, device=comm_dev)
        if world == 1:
            return t.reshape(1, -1).cpu().numpy()
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        return torch.stack(parts).cpu().numpy()

    def all_to_all(rows, sc, rc):
        out = torch.empty((sum(rc), rows.shape[1]), dtype=torch.float64, device=rows.device)
        dist.all_to_all_single(out, rows, rc, sc, group=group)
        return out

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
    rows_stats = []      # [round, boxes_in, after_filter, after_hs, width, elapsed]
    status = BUDGET_EXHAUSTED
    t_start = time.perf_counter()
    for round_no in range(1, cfg.max_rounds + 1):
        t0 = time.perf_counter()
        n_in = backend.size()
        carried, surv, cw, children = backend.round_filter(round_no)
        g1 = gather([float(surv), cw if surv > 0 else 0.0, float(n_in)])      # exchange 1
        g_surv, g_cw, g_in = g1[:, 0].sum(), g1[:, 1].max(), int(g1[:, 2].sum())
        if rows_stats:
            rows_stats[-1][3] = g_in  # previous round's boxes_after_hs (after its dedup)
        hs_on = False
        if g_surv > 0 and hs_possible:  # bnb.py:289-296 on the global survivors
            if cfg.hs_enable_round is not None and round_no >= cfg.hs_enable_round:
                hs_on = True
            if cfg.hs_enable_width is not None and g_cw <= cfg.hs_enable_width:
                hs_on = True
        size, width, calls = backend.round_hs(hs_on, cfg.hs_contract)
        thin, other = backend.route_count(world)
        stop = 1.0 if (rank == 0 and cfg.max_seconds is not None and
                       time.perf_counter() - t_start > cfg.max_seconds) else 0.0
        g2 = gather([float(size), width if size else 0.0, float(other), stop, float(carried + surv),
                     float(children), float(calls)] + [float(v) for v in thin])  # exchange 2
        sizes, g_width = g2[:, 0].astype(np.int64), float(g2[:, 1].max())
        g_after_filter = int(g2[:, 4].sum())
        g_children, g_calls = int(g2[:, 5].sum()), int(g2[:, 6].sum())
        thin_m = g2[:, 7:7 + world].astype(np.int64)            # thin_m[r][d]: thin rows r -> d
        movable = g2[:, 2].astype(np.int64)
        stay = np.array([movable[r] + thin_m[r][r] for r in range(world)])
        after_thin = stay + np.array([thin_m[:, d].sum() - thin_m[d][d] for d in range(world)])
        move = rebalance_plan(after_thin, movable)
        send = np.array([[thin_m[r][d] + move[r][d] if d != r else 0 for d in range(world)]
                         for r in range(world)])
        if send.sum() > 0:                                                    # exchange 3
            sc_all = backend.route(world, rank, move[rank])
            rows, sc, keep = _exchange(torch, dist, backend, rank, world, sc_all, group)
            rc = [int(send[r][rank]) for r in range(world)]
            assert sc == [int(v) for v in send[rank]], "routing counts disagree with the plan"
            backend.import_packed(torch, keep, all_to_all(rows, sc, rc))
        backend.dedup()
        pre_total = int(sizes.sum())  # before dedup: duplicates are thin rows now on one shard
        rows_stats.append([round_no, g_in, g_after_filter, pre_total, g_width if pre_total else 0.0,
                           time.perf_counter() - t0, g_children, g_calls])
        if pre_total == 0:  # dedup never empties a non-empty frontier
            status = NO_REAL_SOLUTION
            break
        if g_width <= target:
            status = WIDTH_REACHED
            break
        if pre_total > cfg.max_boxes:
            g = gather([float(backend.size())])  # exact count after dedup (rare)
            rows_stats[-1][3] = int(g[:, 0].sum())
            if rows_stats[-1][3] > cfg.max_boxes:
                status = BUDGET_EXHAUSTED
                break
        if g2[0, 3]:
            status = BUDGET_EXHAUSTED
            break
    final = gather([float(backend.size())])
    counts = final[:, 0].astype(np.int64)
    rows_stats[-1][3] = int(counts.sum())
    # gather the final frontier on rank 0 and order it there (device radix sort)
    if world > 1:
        mine = backend.export_packed(torch, 0, int(counts[rank]))
        sc = [int(counts[rank]) if d == 0 else 0 for d in range(world)]
        rc = [int(c) for c in counts] if rank == 0 else [0] * world
        got = all_to_all(mine, sc, rc)
        if rank != 0:
            return None
        backend.import_packed(torch, 0, got)
    lo, hi, c, u = backend.finalize()
    out = {"status": status, "lo": lo, "hi": hi, "cert": c, "unsplit": u,
           "stats": [dict(round=r[0], boxes_in=r[1], boxes_after_filter=r[2], boxes_after_hs=r[3], width=r[4],
                          elapsed_seconds=r[5], children=r[6], hs_calls=r[7]) for r in rows_stats]}
    return out if arrays else _result(s, out)


def _result(s, out):
    """SolveResult from engine arrays: the reference's own classes for a reference
    PolySystem, else this package's (lazy boxes above bnb.LAZY_THRESHOLD)."""
    types = _reference_types(s)
    if types is None:
        return _own_result(out)
    from .bnb import RootBoxes, _stats_tuples, LAZY_THRESHOLD
    SR, RB, RS, BX, IV = types
    lo, hi, cert, uns = out["lo"], out["hi"], out["cert"], out["unsplit"]
    if lo.shape[0] > LAZY_THRESHOLD:
        boxes = RootBoxes(lo, hi, cert, uns, (RB, BX, IV))
    else:
        boxes = tuple(RB(BX(tuple(IV(a, b) for a, b in zip(lo[r].tolist(), hi[r].tolist()))), bool(cert[r]),
                         bool(uns[r])) for r in range(lo.shape[0]))
    stats = tuple(RS(round=r, boxes_in=bi, boxes_after_filter=af, boxes_after_hs=ah, width=w, elapsed_seconds=el)
                  for r, bi, af, ah, w, el in _stats_tuples(out))
    return SR(out["status"], boxes, stats)

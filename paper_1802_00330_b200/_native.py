"""ctypes binding of the in-tree C-ABI library librootbox_b200.so (include/rootbox_b200.h).

There is no CPU fallback: if the library is missing or no sm_100 device is
visible, every entry point raises.  ctypes releases the GIL for the duration
of each call, so concurrent solves on different handles run in parallel.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RB_LIB_PATH") or os.path.join(PKG, "librootbox_b200.so")  # override: A/B builds

RB_NO_REAL_SOLUTION, RB_WIDTH_REACHED, RB_BUDGET_EXHAUSTED = 0, 1, 2
STATUS_NAMES = {0: "no_real_solution", 1: "width_reached", 2: "budget_exhausted"}
RB_ERR_ARG, RB_ERR_CUDA, RB_ERR_NOMEM, RB_ERR_LIMIT, RB_ERR_STATE = -1, -2, -3, -4, -5


class RbSystem(C.Structure):
    _fields_ = [
        ("n", C.c_int32), ("n_polys", C.c_int32),
        ("poly_off", C.c_void_p), ("coeff", C.c_void_p), ("fac_off", C.c_void_p),
        ("fac_var", C.c_void_p), ("fac_exp", C.c_void_p),
        ("init_lo", C.c_void_p), ("init_hi", C.c_void_p),
    ]


class RbConfig(C.Structure):
    _fields_ = [
        ("target_width", C.c_double), ("hs_enable_round", C.c_int32), ("hs_contract", C.c_int32),
        ("hs_enable_width", C.c_double), ("max_rounds", C.c_int32), ("exact_round_dedup", C.c_int32),
        ("max_boxes", C.c_int64), ("max_seconds", C.c_double),
    ]


class RbRoundStats(C.Structure):
    _fields_ = [
        ("round", C.c_int32), ("hs_on", C.c_int32),
        ("boxes_in", C.c_int64), ("boxes_after_filter", C.c_int64), ("boxes_after_hs", C.c_int64),
        ("width", C.c_double), ("elapsed_seconds", C.c_double),
        ("children", C.c_int64), ("hs_calls", C.c_int64), ("filter_ops", C.c_int64), ("hs_ops", C.c_int64),
        ("dups", C.c_int64), ("exact_boxes", C.c_int64),
        ("filter_ms", C.c_double), ("hs_ms", C.c_double), ("classify_ms", C.c_double),
        ("classify_bytes", C.c_int64), ("attempts", C.c_int64),
    ]


class RbResultInfo(C.Structure):
    _fields_ = [("status", C.c_int32), ("nrounds", C.c_int32), ("nboxes", C.c_int64),
                ("solve_seconds", C.c_double), ("device_ms", C.c_double), ("kernel_launches", C.c_int64)]


STATS_FIELDS = [f for f, _ in RbRoundStats._fields_]
# numpy view of an rb_round_stats array (same layout as the ctypes structure)
_STATS_DTYPE = np.dtype({"names": STATS_FIELDS,
                         "formats": [np.dtype(t) for _, t in RbRoundStats._fields_],
                         "offsets": [getattr(RbRoundStats, f).offset for f in STATS_FIELDS],
                         "itemsize": C.sizeof(RbRoundStats)})

_lib = None


class NativeError(RuntimeError):
    pass


def lib():
    """Load the engine library; raises ImportError when it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_1802_00330_b200/csrc).  There is no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    P, i64, i32 = C.c_void_p, C.c_int64, C.c_int
    L.rb_version.restype = C.c_char_p
    L.rb_device_count.restype = i32
    L.rb_create.argtypes = [C.POINTER(RbSystem), i32, C.POINTER(P)]
    L.rb_create.restype = i32
    L.rb_solve.argtypes = [P, C.POINTER(RbConfig), C.POINTER(RbResultInfo)]
    L.rb_solve.restype = i32
    L.rb_fetch.argtypes = [P, P, P, P, P, P]
    L.rb_fetch.restype = i32
    L.rb_filter.argtypes = [P, P, P, i64, P, P, i64, C.POINTER(i64)]
    L.rb_filter.restype = i32
    L.rb_hs.argtypes = [P, P, P, i64, i32, P, P, P, i64, C.POINTER(i64)]
    L.rb_hs.restype = i32
    L.rb_krawczyk.argtypes = [P, P, P, i64, P, P, P]
    L.rb_krawczyk.restype = i32
    L.rb_last_error.argtypes = [P]
    L.rb_last_error.restype = C.c_char_p
    L.rb_destroy.argtypes = [P]
    L.rb_shard_load.argtypes = [P, P, P, P, P, i64, C.c_double]
    L.rb_shard_load.restype = i32
    L.rb_round_filter.argtypes = [P, i32, C.POINTER(i64), C.POINTER(i64), C.POINTER(C.c_double),
                                  C.POINTER(i64)]
    L.rb_round_filter.restype = i32
    L.rb_round_hs.argtypes = [P, i32, i32, C.POINTER(i64), C.POINTER(C.c_double), C.POINTER(i64)]
    L.rb_round_hs.restype = i32
    L.rb_shard_export.argtypes = [P, i64, i64, P, P, P, P]
    L.rb_shard_export.restype = i32
    L.rb_shard_import.argtypes = [P, i64, P, P, P, P, i64]
    L.rb_shard_import.restype = i32
    L.rb_shard_size.argtypes = [P]
    L.rb_shard_size.restype = i64
    L.rb_shard_partition.argtypes = [P, i32, P]
    L.rb_shard_partition.restype = i32
    L.rb_shard_dedup.argtypes = [P, C.POINTER(i64), C.POINTER(C.c_double)]
    L.rb_shard_dedup.restype = i32
    L.rb_shard_export_device.argtypes = [P, i64, i64, P, P, P, P]
    L.rb_shard_export_device.restype = i32
    L.rb_shard_import_device.argtypes = [P, i64, P, P, P, P, i64]
    L.rb_shard_import_device.restype = i32
    L.rb_merge.argtypes = [i32, P, P, P, P, P, i64, C.c_double, i32, P, P, P, i64, C.POINTER(i64), P, i64,
                           C.POINTER(i64), C.c_char_p, i64]
    L.rb_merge.restype = i32
    L.rb_set_option.argtypes = [P, C.c_char_p, i64]
    L.rb_set_option.restype = i32
    L.rb_fp64_peak.argtypes = [i32, C.POINTER(C.c_double)]
    L.rb_fp64_peak.restype = i32
    L.rb_codegen_prepare.argtypes = [C.POINTER(RbSystem), C.c_char_p, i64]
    L.rb_codegen_prepare.restype = i32
    L.rb_codegen_active.argtypes = [P, C.c_char_p, i64]
    L.rb_codegen_active.restype = i32
    L.rb_shard_route_count.argtypes = [P, i32, P, C.POINTER(i64)]
    L.rb_shard_route_count.restype = i32
    L.rb_shard_route.argtypes = [P, i32, i32, P, P]
    L.rb_shard_route.restype = i32
    L.rb_shard_finalize.argtypes = [P, C.POINTER(i64)]
    L.rb_shard_finalize.restype = i32
    L.rb_kernel_launches.argtypes = [P]
    L.rb_kernel_launches.restype = i64
    L.rb_merge_device.argtypes = [i32] + L.rb_merge.argtypes
    L.rb_merge_device.restype = i32
    L.rb_format_boxes.argtypes = [i32, P, P, P, i64, i32, P, i64, C.POINTER(i64)]
    L.rb_format_boxes.restype = i32
    L.rb_interval_kat.argtypes = [i32, i32, i32, i64, P, P, P, P, P, P, P, P, P]
    L.rb_interval_kat.restype = i32
    _lib = L
    return L


EXPORTED = ["rb_version", "rb_device_count", "rb_create", "rb_solve", "rb_fetch", "rb_filter", "rb_hs",
            "rb_last_error", "rb_destroy", "rb_shard_load", "rb_round_filter", "rb_round_hs",
            "rb_shard_export", "rb_shard_import", "rb_shard_size", "rb_fp64_peak", "rb_set_option",
            "rb_shard_partition", "rb_shard_dedup", "rb_shard_export_device", "rb_shard_import_device",
            "rb_merge", "rb_krawczyk", "rb_codegen_prepare", "rb_codegen_active", "rb_interval_kat",
            "rb_shard_route_count", "rb_shard_route", "rb_shard_finalize", "rb_format_boxes", "rb_merge_device",
            "rb_kernel_launches"]


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _check(rc, h, what):
    if rc != 0:
        msg = lib().rb_last_error(h)
        msg = msg.decode() if msg else ""
        if rc == RB_ERR_NOMEM:
            raise MemoryError(f"{what}: {msg}")
        if rc in (RB_ERR_ARG, RB_ERR_LIMIT):
            raise ValueError(f"{what}: {msg}")
        raise NativeError(f"{what} failed ({rc}): {msg}")


def _rb_system(tables):
    keep = (tables.poly_off, tables.coeff, tables.fac_off,
            tables.fac_var if tables.fac_var.size else np.zeros(1, np.uint8),
            tables.fac_exp if tables.fac_exp.size else np.zeros(1, np.uint8), tables.init_lo, tables.init_hi)
    sysd = RbSystem(
        n=tables.n, n_polys=len(tables.poly_off) - 1,
        poly_off=_p(keep[0]), coeff=_p(keep[1]), fac_off=_p(keep[2]), fac_var=_p(keep[3]), fac_exp=_p(keep[4]),
        init_lo=_p(keep[5]), init_hi=_p(keep[6]))
    return sysd, keep


def codegen_prepare(tables) -> str:
    """Compile the system-specialised kernels into the on-disk cache (no device
    needed); returns the cache key."""
    sysd, keep = _rb_system(tables)
    err = C.create_string_buffer(4096)
    rc = lib().rb_codegen_prepare(C.byref(sysd), err, len(err))
    if rc != 0:
        raise NativeError(f"rb_codegen_prepare failed ({rc}): {err.value.decode(errors='replace')}")
    return err.value.decode()


class Engine:
    """One device-resident engine for one compiled system (rb_handle)."""

    def __init__(self, tables, device: int = 0):
        L = lib()
        self.n = tables.n
        self.device = device
        sysd, self._keep = _rb_system(tables)
        h = C.c_void_p()
        rc = L.rb_create(C.byref(sysd), int(device), C.byref(h))
        _check(rc, None, "rb_create")
        self.h = h
        self._device_timing = True
        # rb_solve + rb_fetch (and the other multi-call sequences below) run as one
        # unit per engine: ctypes releases the GIL, and the engine cache hands the
        # same Engine to every thread solving the same system.
        self._lock = threading.RLock()
        self._info = RbResultInfo()  # reused under the lock
        self._info_ref = C.byref(self._info)
        self._cfg_cache = (None, None)

    def _cfg_ref(self, cfg):
        if self._cfg_cache[0] is not cfg:
            self._cfg_cache = (cfg, C.byref(cfg))
        return self._cfg_cache[1]

    def codegen_active(self):
        """(True, '') when the system-specialised kernels run, else (False, reason)."""
        why = C.create_string_buffer(2048)
        on = lib().rb_codegen_active(self.h, why, len(why))
        return on == 1, why.value.decode(errors="replace")

    def set_option(self, key: str, value: int):
        with self._lock:
            self._live()
            _check(lib().rb_set_option(self.h, key.encode(), int(value)), self.h, "rb_set_option")
            if key == "device_timing":
                self._device_timing = bool(value)

    def _live(self):
        if not self.h:
            raise NativeError("engine is closed")

    def close(self):
        lock = getattr(self, "_lock", None)
        if lock is None:
            return
        with lock:  # waits for a solve in flight on another thread
            if getattr(self, "h", None):
                lib().rb_destroy(self.h)
                self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def solve(self, cfg: RbConfig, stats_rows: bool = False, device_timing: bool = True):
        """One rb_solve + rb_fetch.  stats_rows: per-round statistics as raw tuples in
        STATS_FIELDS order under "stats_rows" (the public solve() path) instead of
        dicts under "stats".  device_timing=False: a solve the round graph finishes
        returns as soon as its results are visible in mapped host memory, without
        waiting for the stream (device_ms is then -1)."""
        L = lib()
        with self._lock:
            self._live()
            if device_timing != self._device_timing:
                self.set_option("device_timing", 1 if device_timing else 0)
                self._device_timing = device_timing
            info = self._info
            _check(L.rb_solve(self.h, self._cfg_ref(cfg), self._info_ref), self.h, "rb_solve")
            N, n, nr = int(info.nboxes), self.n, int(info.nrounds)
            # one host buffer for rows, flags and statistics: a single address lookup
            # (ndarray.ctypes costs ~1 us per access on this per-solve path)
            sb = _STATS_DTYPE.itemsize * max(1, nr)
            rb = 8 * N * n
            buf = np.empty(2 * rb + 2 * N + sb + 8, np.uint8)
            a0 = buf.ctypes.data
            a_st = (a0 + 2 * rb + 2 * N + 7) & ~7
            _check(L.rb_fetch(self.h, a0, a0 + rb, a0 + 2 * rb, a0 + 2 * rb + N, a_st), self.h, "rb_fetch")
            lo = buf[:rb].view(np.float64).reshape(N, n)
            hi = buf[rb:2 * rb].view(np.float64).reshape(N, n)
            flags = buf[2 * rb:2 * rb + 2 * N].reshape(2, N)
            o = a_st - a0
            stats = buf[o:o + sb].view(_STATS_DTYPE)
        rows = stats[:nr].tolist()
        fb = flags.view(np.bool_)
        return {"status": STATUS_NAMES[info.status], "lo": lo, "hi": hi, "cert": fb[0], "unsplit": fb[1],
                **({"stats_rows": rows} if stats_rows else {"stats": [dict(zip(STATS_FIELDS, r)) for r in rows]}),
                "solve_seconds": info.solve_seconds,
                "device_ms": info.device_ms, "kernel_launches": int(info.kernel_launches)}

    def filter(self, plo, phi):
        plo = np.ascontiguousarray(plo, np.float64); phi = np.ascontiguousarray(phi, np.float64)
        P = plo.shape[0]
        cap = max(1, P * 64)
        for _ in range(2):
            olo = np.empty((cap, self.n)); ohi = np.empty((cap, self.n))
            M = C.c_int64()
            with self._lock:
                self._live()
                rc = lib().rb_filter(self.h, _p(plo), _p(phi), P, _p(olo), _p(ohi), cap, C.byref(M))
                _check(rc, self.h, "rb_filter")
            if M.value <= cap:
                return olo[:M.value].copy(), ohi[:M.value].copy()
            cap = M.value
        raise NativeError("rb_filter: capacity retry failed")

    def hs(self, lo, hi, contract_output=True):
        lo = np.ascontiguousarray(lo, np.float64); hi = np.ascontiguousarray(hi, np.float64)
        M = lo.shape[0]
        cap = max(1, 2 * M)
        olo = np.empty((cap, self.n)); ohi = np.empty((cap, self.n)); oc = np.empty(cap, np.uint8)
        M2 = C.c_int64()
        with self._lock:
            self._live()
            _check(lib().rb_hs(self.h, _p(lo), _p(hi), M, int(bool(contract_output)), _p(olo), _p(ohi), _p(oc),
                               cap, C.byref(M2)), self.h, "rb_hs")
        m = M2.value
        return olo[:m].copy(), ohi[:m].copy(), oc[:m].astype(bool)

    def krawczyk(self, lo, hi):
        lo = np.ascontiguousarray(lo, np.float64); hi = np.ascontiguousarray(hi, np.float64)
        M = lo.shape[0]
        olo = np.empty((M, self.n)); ohi = np.empty((M, self.n)); ok = np.empty(M, np.uint8)
        with self._lock:
            self._live()
            _check(lib().rb_krawczyk(self.h, _p(lo), _p(hi), M, _p(olo), _p(ohi), _p(ok)), self.h, "rb_krawczyk")
        return ok.astype(bool), olo, ohi


KAT_OPS = {"_add_rd": 0, "_add_ru": 1, "_mul_rd": 2, "_mul_ru": 3, "_div_rd": 4, "_div_ru": 5,
           "mul": 10, "recip": 11, "mid": 12, "div_extended": 40}
KAT_POLICY = {"fast": 0, "exact": 1, "guarded": 2}


def interval_kat(op, policy, xl, xh, yl=None, yh=None, device: int = 0):
    """One interval.cuh operation on the device over arrays (rb_interval_kat): op is a
    name of KAT_OPS or ("pow", k); returns (o0, o1, o2, o3, kind)."""
    code = 20 + int(op[1]) if isinstance(op, tuple) else KAT_OPS[op]
    arr = [np.ascontiguousarray(v, np.float64) for v in (xl, xh, xl if yl is None else yl, xh if yh is None else yh)]
    m = arr[0].size
    outs = [np.empty(m) for _ in range(4)]
    kind = np.empty(m, np.int8)
    _check(lib().rb_interval_kat(int(device), code, KAT_POLICY[policy], m, *[_p(a) for a in arr],
                                 *[_p(o) for o in outs], _p(kind)), None, "rb_interval_kat")
    return (*outs, kind)


def device_count() -> int:
    return int(lib().rb_device_count())


def fp64_peak(device: int = 0) -> float:
    """Measured directed-rounding FP64 op throughput (ops/s) of the device."""
    v = C.c_double()
    _check(lib().rb_fp64_peak(int(device), C.byref(v)), None, "rb_fp64_peak")
    return v.value


def version() -> str:
    return lib().rb_version().decode()

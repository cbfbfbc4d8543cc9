"""Drop-in ``solve`` for the reference solver entry point, on the B200 engine.

Mirrors rootbox.bnb (bnb.py:40-114, 224-361): same names, same fields, same
argument meaning, same ``ValueError`` from ``SolverConfig.validate``, same
statuses and the same canonically ordered ``SolveResult.boxes``.  The round
loop runs inside librootbox_b200.so (one rb_solve call); this module only
converts types.

If the system passed in is a reference ``rootbox.poly.PolySystem`` (and the
reference package is importable), the result is built from the reference's
own classes (``rootbox.bnb.SolveResult``/``RootBox``/``RoundStats``,
``rootbox.poly.Box``, ``rootbox.interval.Interval``) so downstream reference
code (backtrack.snap_to_grid, cli.RunReport) consumes it unchanged.
Otherwise the lightweight mirror types below are returned.
"""
from __future__ import annotations

import math
import os
import threading
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .system import SystemSpec, as_spec, compile_tables

__all__ = ["SolverConfig", "RoundStats", "RootBox", "RootBoxes", "SolveResult", "Interval", "Box", "solve",
           "solve_arrays", "NO_REAL_SOLUTION", "WIDTH_REACHED", "BUDGET_EXHAUSTED"]

NO_REAL_SOLUTION = "no_real_solution"
WIDTH_REACHED = "width_reached"
BUDGET_EXHAUSTED = "budget_exhausted"


class Interval:
    """Closed interval container (the arithmetic runs on the device)."""

    __slots__ = ("lo", "hi")

    def __init__(self, lo, hi):
        lo = float(lo)
        hi = float(hi)
        if lo != lo or hi != hi:
            raise ValueError(f"NaN bound in [{lo}, {hi}]")
        if lo > hi:
            raise ValueError(f"lower bound {lo!r} exceeds upper bound {hi!r}")
        object.__setattr__(self, "lo", lo)
        object.__setattr__(self, "hi", hi)

    def __setattr__(self, name, value):
        raise AttributeError("Interval is immutable")

    def __repr__(self):
        f = lambda v: "inf" if v == math.inf else ("-inf" if v == -math.inf else repr(v))  # noqa: E731
        return f"[{f(self.lo)},{f(self.hi)}]"

    def __eq__(self, other):
        return isinstance(other, Interval) and self.lo == other.lo and self.hi == other.hi

    def __hash__(self):
        return hash((self.lo, self.hi))


@dataclass(frozen=True)
class Box:
    intervals: tuple

    @classmethod
    def from_bounds(cls, los, his):
        return cls(tuple(Interval(lo, hi) for lo, hi in zip(los, his)))

    def __len__(self):
        return len(self.intervals)

    def __iter__(self):
        return iter(self.intervals)

    def __getitem__(self, i):
        return self.intervals[i]

    @property
    def dimension(self):
        return len(self.intervals)

    def sort_key(self):
        return tuple(iv.lo for iv in self.intervals) + tuple(iv.hi for iv in self.intervals)

    def contains_point(self, point):
        return all(iv.lo <= float(v) <= iv.hi for iv, v in zip(self.intervals, point))

    def __str__(self):
        return " x ".join(str(iv) for iv in self.intervals)


@dataclass(frozen=True)
class SolverConfig:
    """bnb.py:49-86.  worker_count / batch_size / engine are accepted and
    validated for drop-in compatibility; results do not depend on them
    (bnb.py:9-11) and the B200 engine ignores them."""

    target_width: float | None = None
    hs_enable_round: int | None = None
    hs_enable_width: float | None = 1.0
    max_rounds: int = 24
    max_boxes: int = 200_000_000
    max_seconds: float | None = None
    worker_count: int = 1
    batch_size: int = 4096
    hs_contract: bool = True
    engine: str = "batch"

    def validate(self) -> None:
        validate_config(self)


def validate_config(cfg) -> None:
    """SolverConfig.validate (bnb.py:72-86), for our config or the reference's."""
    if cfg.target_width is not None and not cfg.target_width > 0:
        raise ValueError("target_width must be positive")
    if cfg.max_boxes < 1:
        raise ValueError("max_boxes must be at least 1")
    if cfg.max_rounds < 1:
        raise ValueError("max_rounds must be at least 1")
    if cfg.worker_count < 1:
        raise ValueError("worker_count must be at least 1")
    if cfg.batch_size < 1:
        raise ValueError("batch_size must be at least 1")
    if cfg.hs_enable_round is not None and cfg.hs_enable_round < 0:
        raise ValueError("hs_enable_round must be >= 0")
    if cfg.engine not in ("batch", "scalar"):
        raise ValueError(f"unknown engine {cfg.engine!r}")


@dataclass(frozen=True)
class RoundStats:
    round: int
    boxes_in: int
    boxes_after_filter: int
    boxes_after_hs: int
    width: float
    elapsed_seconds: float


@dataclass(frozen=True)
class RootBox:
    box: Box
    certified: bool = False
    unsplittable: bool = False


@dataclass(frozen=True)
class SolveResult:
    status: str
    boxes: tuple = ()
    stats: tuple = field(default=())

    @property
    def reached_width(self) -> bool:
        return self.status == WIDTH_REACHED


# ---------------------------------------------------------------- engine cache

_ENGINES: dict = {}
_LOCK = threading.Lock()
_MAX_ENGINES = 8


_DEFAULT_DEVICE = None


def default_device() -> int:
    """RB_DEVICE, else LOCAL_RANK, else 0 -- read once per process (os.environ
    lookups cost microseconds on the per-solve path)."""
    global _DEFAULT_DEVICE
    if _DEFAULT_DEVICE is None:
        _DEFAULT_DEVICE = _env_device()
    return _DEFAULT_DEVICE


def _env_device() -> int:
    for k in ("RB_DEVICE", "LOCAL_RANK"):
        v = os.environ.get(k)
        if v is not None and v.strip().isdigit():
            return int(v)
    return 0


def _key(spec: SystemSpec):
    t = compile_tables(spec)
    h = t.__dict__.get("_key")
    if h is None:
        h = (t.n, t.poly_off.tobytes(), t.coeff.tobytes(), t.fac_off.tobytes(), t.fac_var.tobytes(),
             t.fac_exp.tobytes(), t.init_lo.tobytes(), t.init_hi.tobytes())
        t.__dict__["_key"] = h
    return h, t


def engine_for(spec: SystemSpec, device: int | None = None) -> _native.Engine:
    """Cached device engine for a system (device buffers persist across solves)."""
    device = default_device() if device is None else device
    key, tables = _key(spec)
    with _LOCK:
        e = _ENGINES.get((key, device))
        if e is None:
            if len(_ENGINES) >= _MAX_ENGINES:
                # dropped, not closed: a thread still solving on it holds a reference,
                # and the engine is destroyed with its last reference (Engine.__del__)
                _ENGINES.pop(next(iter(_ENGINES)))
            e = _native.Engine(tables, device)
            _ENGINES[(key, device)] = e
        return e


_NCFG: dict = {}


def native_config(cfg, exact_round_dedup: bool = True) -> _native.RbConfig:
    """rb_config of a (frozen) SolverConfig, cached per config value."""
    try:
        key = (cfg, exact_round_dedup)
        hit = _NCFG.get(key)
    except TypeError:  # an unhashable config-like object
        key, hit = None, None
    if hit is not None:
        return hit
    out = _native_config(cfg, exact_round_dedup)
    if key is not None and len(_NCFG) < 256:
        _NCFG[key] = out
    return out


def _native_config(cfg, exact_round_dedup: bool) -> _native.RbConfig:
    return _native.RbConfig(
        target_width=-1.0 if cfg.target_width is None else float(cfg.target_width),
        hs_enable_round=-1 if cfg.hs_enable_round is None else int(cfg.hs_enable_round),
        hs_contract=1 if cfg.hs_contract else 0,
        hs_enable_width=math.nan if cfg.hs_enable_width is None else float(cfg.hs_enable_width),
        max_rounds=int(cfg.max_rounds),
        exact_round_dedup=1 if exact_round_dedup else 0,
        max_boxes=int(cfg.max_boxes),
        max_seconds=-1.0 if cfg.max_seconds is None else float(cfg.max_seconds),
    )


def solve_arrays(s, cfg=None, device: int | None = None) -> dict:
    """solve() without Python object materialisation: returns the canonical
    row-major arrays (lo, hi, cert, unsplit), status and per-round stats
    (including device kernel times and algorithmic op counts)."""
    cfg = cfg or SolverConfig()
    validate_config(cfg)
    spec = as_spec(s)
    eng = engine_for(spec, device)
    return eng.solve(native_config(cfg))


def _reference_types(s):
    mod = type(s).__module__
    if not mod.startswith("rootbox"):
        return None
    try:
        from rootbox import bnb as rbnb  # type: ignore
        from rootbox import poly as rpoly  # type: ignore
        from rootbox.interval import Interval as RInterval  # type: ignore
    except Exception:
        return None
    return rbnb.SolveResult, rbnb.RootBox, rbnb.RoundStats, rpoly.Box, RInterval


# Results above this many boxes come back as a lazy RootBoxes sequence.
LAZY_THRESHOLD = 16384


class RootBoxes(Sequence):
    """``SolveResult.boxes`` for large results: RootBox objects are built on
    access instead of up front (the reference materialises every box,
    ``_to_rootboxes`` bnb.py:357-361, ~30 us each).  Indexing, slicing,
    iteration, ``len`` and equality with a tuple behave like the tuple the
    reference returns; ``.lo/.hi/.cert/.unsplit`` expose the arrays."""

    __slots__ = ("lo", "hi", "cert", "unsplit", "_types", "_hash")

    def __init__(self, lo, hi, cert, unsplit, types):
        self.lo, self.hi, self.cert, self.unsplit, self._types = lo, hi, cert, unsplit, types
        self._hash = None

    def __len__(self):
        return self.lo.shape[0]

    def _make(self, r):
        RB, BX, IV = self._types
        return RB(BX(tuple(IV(a, b) for a, b in zip(self.lo[r].tolist(), self.hi[r].tolist()))),
                  bool(self.cert[r]), bool(self.unsplit[r]))

    def __getitem__(self, i):
        if isinstance(i, slice):
            return tuple(self._make(r) for r in range(*i.indices(len(self))))
        n = len(self)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError("RootBoxes index out of range")
        return self._make(i)

    def __iter__(self):
        for r in range(len(self)):
            yield self._make(r)

    def __eq__(self, other):
        if isinstance(other, RootBoxes):
            return (np.array_equal(self.lo, other.lo) and np.array_equal(self.hi, other.hi)
                    and np.array_equal(self.cert, other.cert) and np.array_equal(self.unsplit, other.unsplit))
        if isinstance(other, (tuple, list)):
            return len(other) == len(self) and all(a == b for a, b in zip(self, other))
        return NotImplemented

    def __hash__(self):
        # equal to a tuple of the same RootBox objects, so hash like that tuple (the
        # reference's frozen SolveResult hashes its boxes tuple)
        if self._hash is None:
            self._hash = hash(tuple(self))
        return self._hash

    def __add__(self, other):
        return tuple(self) + tuple(other)

    def __radd__(self, other):
        return tuple(other) + tuple(self)

    def __repr__(self):
        return f"RootBoxes({len(self)} boxes)"


def _made(cls, **fields):
    """Instance of one of this module's frozen dataclasses without the per-field
    frozen __setattr__ of its __init__ (results are built per solve, on the
    end-to-end path); same object as cls(**fields)."""
    obj = object.__new__(cls)
    obj.__dict__.update(fields)
    return obj


def _iv(lo, hi):
    """Interval of finite engine endpoints (already valid: lo <= hi, no NaN)."""
    iv = object.__new__(Interval)
    object.__setattr__(iv, "lo", lo)
    object.__setattr__(iv, "hi", hi)
    return iv


# RoundStats fields in an rb_round_stats row (_native.STATS_FIELDS order)
_RS_IDX = tuple(_native.STATS_FIELDS.index(f) for f in
                ("round", "boxes_in", "boxes_after_filter", "boxes_after_hs", "width", "elapsed_seconds"))


def _stats_tuples(out):
    """(round, boxes_in, after_filter, after_hs, width, elapsed) per round, from the
    raw rows of Engine.solve(stats_rows=True) or from the dicts of solve_arrays."""
    if "stats_rows" in out:
        a, b, c, d, e, f = _RS_IDX
        return [(r[a], r[b], r[c], r[d], r[e], r[f]) for r in out["stats_rows"]]
    return [(int(st["round"]), int(st["boxes_in"]), int(st["boxes_after_filter"]), int(st["boxes_after_hs"]),
             float(st["width"]), float(st["elapsed_seconds"])) for st in out["stats"]]


def _own_result(out):
    lo, hi, cert, uns = out["lo"], out["hi"], out["cert"], out["unsplit"]
    if lo.shape[0] > LAZY_THRESHOLD:
        boxes = RootBoxes(lo, hi, cert, uns, (RootBox, Box, Interval))
    else:
        cl, ul = cert.tolist(), uns.tolist()
        boxes = tuple(
            _made(RootBox, box=_made(Box, intervals=tuple(map(_iv, a, b))), certified=c, unsplittable=u)
            for a, b, c, u in zip(lo.tolist(), hi.tolist(), cl, ul))
    stats = tuple(_made(RoundStats, round=r, boxes_in=bi, boxes_after_filter=af, boxes_after_hs=ah, width=w,
                        elapsed_seconds=el) for r, bi, af, ah, w, el in _stats_tuples(out))
    return _made(SolveResult, status=out["status"], boxes=boxes, stats=stats)


def solve(s, cfg=None) -> SolveResult:
    """Isolate all real roots of the system inside its initial box (bnb.py:224)."""
    cfg = cfg or SolverConfig()
    validate_config(cfg)
    spec = as_spec(s)
    out = engine_for(spec).solve(native_config(cfg), stats_rows=True, device_timing=False)
    types = _reference_types(s)
    if types is None:
        return _own_result(out)
    SR, RB, RS, BX, IV = types
    lo, hi, cert, uns = out["lo"], out["hi"], out["cert"], out["unsplit"]
    if lo.shape[0] > LAZY_THRESHOLD:
        boxes = RootBoxes(lo, hi, cert, uns, (RB, BX, IV))
    else:
        boxes = tuple(
            RB(BX(tuple(IV(a, b) for a, b in zip(lo[r].tolist(), hi[r].tolist()))), bool(cert[r]), bool(uns[r]))
            for r in range(lo.shape[0]))
    stats = tuple(RS(round=r, boxes_in=bi, boxes_after_filter=af, boxes_after_hs=ah, width=w, elapsed_seconds=el)
                  for r, bi, af, ah, w, el in _stats_tuples(out))
    return SR(out["status"], boxes, stats)

"""Solve + backtracking merge + report: the native counterpart of
``rootbox.cli.run_pipeline`` (cli.py:172-205).

The merge (snap_to_grid + merge_to_width, backtrack.py:118-242) runs in exact
integer arithmetic in librootbox_b200.so (``rb_merge``); the report has the
reference's JSON / CSV / text formats (cli.py:42-123).  When the reference
package is importable and the system is a reference ``PolySystem``, the
reference's own ``RunReport`` class is returned.
"""
from __future__ import annotations

import ctypes as C
import json
import math
import time
from dataclasses import dataclass

import numpy as np

from . import __version__, _native
from .bnb import BUDGET_EXHAUSTED, Box, Interval, RootBox, RootBoxes, SolverConfig, _reference_types, solve
from .system import as_spec

SCHEMA_VERSION = 1


DEVICE_MERGE_MIN = 20000  # result sets at least this large merge on the device when it applies


def merge_arrays(init_lo, init_hi, lo, hi, cert, stop_width=None, stop_on_plateau=True, device=None):
    """rb_merge / rb_merge_device: merged boxes (canonical order), certified flags and
    the merge levels [(width, count), ...] of merge_to_width(snap_to_grid(boxes)).
    device: run on that GPU when the set is on its fast path (power-of-two initial
    widths, levels <= 53), else on the host; None = the host."""
    L = _native.lib()
    ilo = np.ascontiguousarray(init_lo, np.float64)
    ihi = np.ascontiguousarray(init_hi, np.float64)
    n = ilo.size
    lo = np.ascontiguousarray(lo, np.float64).reshape(-1, n)
    hi = np.ascontiguousarray(hi, np.float64).reshape(-1, n)
    c = np.ascontiguousarray(cert, np.uint8).reshape(-1)
    N = lo.shape[0]
    cap, cap_lv = max(1, N), 64
    err = C.create_string_buffer(512)
    for _ in range(2):
        olo = np.empty((cap, n)); ohi = np.empty((cap, n)); oc = np.empty(cap, np.uint8)
        lv = np.empty((cap_lv, 2))
        M = C.c_int64(); K = C.c_int64()
        p = _native._p
        args = (n, p(ilo), p(ihi), p(lo), p(hi), p(c), N, -1.0 if stop_width is None else float(stop_width),
                int(bool(stop_on_plateau)), p(olo), p(ohi), p(oc), cap, C.byref(M), p(lv), cap_lv, C.byref(K),
                err, 512)
        rc = -1
        if device is not None:
            rc = L.rb_merge_device(int(device), *args)
            if rc == _native.RB_ERR_LIMIT:  # not on the device fast path: the host merge decides
                device = None
            elif rc != 0:
                raise _native.NativeError(f"rb_merge_device: {err.value.decode()}")
        if device is None:
            rc = L.rb_merge(*args)
        if rc != 0:
            raise ValueError(f"rb_merge: {err.value.decode()}")
        if M.value <= cap and K.value <= cap_lv:
            break
        cap, cap_lv = max(cap, M.value), max(cap_lv, K.value)
    m, k = M.value, K.value
    levels = tuple((float(lv[i, 0]), int(lv[i, 1])) for i in range(k))
    return olo[:m].copy(), ohi[:m].copy(), oc[:m].astype(bool), levels


@dataclass
class RunReport:
    """Mirror of rootbox.cli.RunReport (cli.py:42-123), same output formats."""

    system: str
    config: dict
    status: str
    result: object
    roots: tuple
    merge_levels: tuple
    wall_seconds: float

    def to_json_dict(self) -> dict:
        return {
            "schema_version": SCHEMA_VERSION,
            "solver_version": "0.1.0",  # the reference's version: the report format is its
            "system": self.system,
            "config": self.config,
            "status": self.status,
            "rounds": [{"round": st.round, "boxes_in": st.boxes_in, "boxes_after_filter": st.boxes_after_filter,
                        "boxes_after_hs": st.boxes_after_hs, "width": st.width,
                        "elapsed_seconds": st.elapsed_seconds} for st in self.result.stats],
            "roots": [{"intervals": [[iv.lo, iv.hi] for iv in rb.box], "certified": rb.certified}
                      for rb in self.roots],
            "merge_levels": [{"width": w, "count": c} for w, c in self.merge_levels],
            "wall_seconds": self.wall_seconds,
        }

    def to_json(self) -> str:
        return report_to_json(self)

    def to_csv(self, var_names) -> str:
        return report_to_csv(self, var_names)


def format_boxes(lo, hi, cert, fmt: str) -> str:
    """rb_format_boxes: the "roots" elements of RunReport.to_json (fmt "json") or the
    rows of RunReport.to_csv (fmt "csv") for row-major boxes, written natively with
    Python's float repr (cli.py:54-100)."""
    L = _native.lib()
    lo = np.ascontiguousarray(lo, np.float64)
    hi = np.ascontiguousarray(hi, np.float64)
    N = lo.shape[0]
    n = lo.shape[1] if lo.ndim == 2 else 1
    c = np.ascontiguousarray(cert, np.uint8).reshape(-1)
    code = {"json": 0, "csv": 1}[fmt]
    ln = C.c_int64()
    p = _native._p
    rc = L.rb_format_boxes(n, p(lo), p(hi), p(c), N, code, None, 0, C.byref(ln))
    if rc != 0:
        raise ValueError("rb_format_boxes: bad arguments")
    buf = C.create_string_buffer(max(1, ln.value))
    rc = L.rb_format_boxes(n, p(lo), p(hi), p(c), N, code, buf, ln.value, C.byref(ln))
    if rc != 0:
        raise ValueError("rb_format_boxes: bad arguments")
    return buf.raw[:ln.value].decode("ascii")


def _root_arrays(roots):
    if isinstance(roots, RootBoxes):
        return roots.lo, roots.hi, roots.cert
    n = len(roots[0].box) if roots else 1
    lo = np.array([[iv.lo for iv in rb.box] for rb in roots], np.float64).reshape(-1, n)
    hi = np.array([[iv.hi for iv in rb.box] for rb in roots], np.float64).reshape(-1, n)
    return lo, hi, np.array([rb.certified for rb in roots], bool)


_ROOTS_MARK = "\x00roots\x00"


def report_to_json(rep) -> str:
    """RunReport.to_json() (cli.py:54-86) with the roots section from rb_format_boxes:
    byte-identical, for this package's RunReport or the reference's."""
    d = {
        "schema_version": SCHEMA_VERSION,
        "solver_version": "0.1.0",
        "system": rep.system,
        "config": rep.config,
        "status": rep.status,
        "rounds": [{"round": st.round, "boxes_in": st.boxes_in, "boxes_after_filter": st.boxes_after_filter,
                    "boxes_after_hs": st.boxes_after_hs, "width": st.width,
                    "elapsed_seconds": st.elapsed_seconds} for st in rep.result.stats],
        "roots": _ROOTS_MARK,
        "merge_levels": [{"width": w, "count": c} for w, c in rep.merge_levels],
        "wall_seconds": rep.wall_seconds,
    }
    text = json.dumps(d, indent=2)
    if len(rep.roots) == 0:
        body = "[]"
    else:
        lo, hi, cert = _root_arrays(rep.roots)
        body = "[\n" + format_boxes(lo, hi, cert, "json") + "\n  ]"
    return text.replace(json.dumps(_ROOTS_MARK), body, 1)


def report_to_csv(rep, var_names) -> str:
    """RunReport.to_csv (cli.py:88-100) with the rows from rb_format_boxes."""
    header = []
    for nm in var_names:
        header += [f"{nm}_lo", f"{nm}_hi"]
    header.append("certified")
    if len(rep.roots) == 0:
        return ",".join(header) + "\n"
    lo, hi, cert = _root_arrays(rep.roots)
    return ",".join(header) + "\n" + format_boxes(lo, hi, cert, "csv")


def config_echo(cfg, merge: bool) -> dict:
    """cli._config_echo (cli.py:156-169)."""
    return {"target_width": cfg.target_width, "hs_enable_round": cfg.hs_enable_round,
            "hs_enable_width": cfg.hs_enable_width, "max_rounds": cfg.max_rounds, "max_boxes": cfg.max_boxes,
            "max_seconds": cfg.max_seconds, "worker_count": cfg.worker_count, "batch_size": cfg.batch_size,
            "hs_contract": cfg.hs_contract, "engine": cfg.engine, "backtrack": merge}


def run_pipeline(s, cfg=None, merge: bool = True, merge_width=None):
    """solve + grid normalisation + backtracking merge, as one report (cli.py:172-205)."""
    cfg = cfg or SolverConfig()
    t0 = time.perf_counter()
    result = solve(s, cfg)
    spec = as_spec(s)
    types = _reference_types(s)
    if types is None:
        RB, BX, IV, Report = RootBox, Box, Interval, RunReport
    else:
        from rootbox import cli as rcli  # type: ignore
        _, RB, _, BX, IV = types
        Report = rcli.RunReport
    if result.status == BUDGET_EXHAUSTED or not merge:
        roots, levels = result.boxes, ()
    elif not result.boxes:
        roots, levels = (), ()
    else:
        n = spec.n
        if isinstance(result.boxes, RootBoxes):  # large result: arrays, no per-box objects
            lo, hi, cert = result.boxes.lo, result.boxes.hi, result.boxes.cert
        else:
            lo = np.array([[iv.lo for iv in rb.box] for rb in result.boxes]).reshape(-1, n)
            hi = np.array([[iv.hi for iv in rb.box] for rb in result.boxes]).reshape(-1, n)
            cert = np.array([rb.certified for rb in result.boxes], bool)
        from .bnb import default_device
        dev = default_device() if lo.shape[0] >= DEVICE_MERGE_MIN else None
        mlo, mhi, mc, levels = merge_arrays(spec.init_lo, spec.init_hi, lo, hi, cert, stop_width=merge_width,
                                            device=dev)
        roots = tuple(RB(BX(tuple(IV(a, b) for a, b in zip(mlo[r].tolist(), mhi[r].tolist()))), bool(mc[r]))
                      for r in range(mlo.shape[0]))
    wall = time.perf_counter() - t0
    return Report(system=getattr(s, "name", "") or spec.name or "?", config=config_echo(cfg, merge),
                  status=result.status, result=result, roots=roots, merge_levels=levels, wall_seconds=wall)

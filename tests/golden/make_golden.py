"""Generate the golden fixtures that pin the oracle and the CUDA engine.

TEST INFRASTRUCTURE ONLY.  This script imports the *unmodified* reference
package (``rootbox`` 0.1.0, read-only at /root/reference/pkg/src) and records
its outputs as exact float64 bit patterns.  It runs in the build container
only; the fixtures it writes travel with the repo, the reference does not.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--part NAME ...]

Parts:
  systems   tests/golden/systems.json     every corpus system + the BASELINE configs,
                                          parsed by rootbox.poly.parse_system (poly.py:451-533),
                                          canonical monomials and PolySystem.jacobian (poly.py:284-291)
  interval  tests/golden/kat_interval.npz directed scalar ops interval.py:66-205, Interval.__mul__/
                                          __pow__/recip/mid (interval.py:269-351), div_extended (:394-432)
  poly      tests/golden/kat_poly.npz     Polynomial.eval_interval (poly.py:187-203) of F and J on random boxes
  gj        tests/golden/kat_gj.npz       linalg.gauss_jordan_inverse (linalg.py:137-172)
  hs        tests/golden/kat_hs.npz       hansen.contract (hansen.py:77-138) on random boxes
  solve     tests/golden/solve_*.json     bnb.solve (bnb.py:224-354) end to end, with per-round
                                          _chunk_batch / _hs_pass captures in rounds_*.npz
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import struct
import sys
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import rootbox  # noqa: E402
from rootbox import bnb, corpus, hansen, interval, linalg, poly  # noqa: E402
from rootbox.interval import Interval  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


# ---------------------------------------------------------------- systems


def circle_line_text():
    return "vars: x y\ninit: x in [-2,2]; y in [-2,2]\neq: x^2 + y^2 - 1\neq: x - y\n"


def broyden_tri_text(n, lo, hi):
    v = [f"x{i}" for i in range(1, n + 1)]
    L = ["vars: " + " ".join(v), "init: " + "; ".join(f"{x} in [{lo},{hi}]" for x in v)]
    for i in range(n):
        t = f"(3 - 2*{v[i]})*{v[i]}" + (f" - {v[i-1]}" if i > 0 else "") + \
            (f" - 2*{v[i+1]}" if i < n - 1 else "") + " + 1"
        L.append("eq: " + t)
    return "\n".join(L) + "\n"


def broyden_banded_text(n, lo, hi, ml=5, mu=1):
    v = [f"x{i}" for i in range(1, n + 1)]
    L = ["vars: " + " ".join(v), "init: " + "; ".join(f"{x} in [{lo},{hi}]" for x in v)]
    for i in range(n):
        t = f"{v[i]}*(2 + 5*{v[i]}^2) + 1" + "".join(
            f" - {v[j]}*(1 + {v[j]})"
            for j in range(max(0, i - ml), min(n - 1, i + mu) + 1) if j != i)
        L.append("eq: " + t)
    return "\n".join(L) + "\n"


def brown_text(n, lo, hi):
    v = [f"x{i}" for i in range(1, n + 1)]
    s = " + ".join(v)
    L = ["vars: " + " ".join(v), "init: " + "; ".join(f"{x} in [{lo},{hi}]" for x in v)]
    L += [f"eq: {v[i]} + {s} - {n + 1}" for i in range(n - 1)] + ["eq: " + "*".join(v) + " - 1"]
    return "\n".join(L) + "\n"


def quirk17b_text():
    # SURVEY Appendix A #17b: unsplittable boxes idle until max_rounds
    return "vars: x y\ninit: x in [0,2]; y in [-2,2]\neq: x - 1\neq: y^3 - y - 1\n"


def wide_circle_text():
    # coefficients 2^1000 > 2^995: every product with them is in the reference's
    # "untrusted" band (interval.py:38-39, 98-136), so the engine's exponent guards
    # must route the filter, HS preconditioning and sweep to the Exact policy
    return ("vars: x y\ninit: x in [-2,2]; y in [-2,2]\n"
            "eq: 2^1000*x^2 + 2^1000*y^2 - 2^1000\neq: x - y\n")


def synthetic_texts():
    return {
        "wide_circle": wide_circle_text(),
        "circle_line": circle_line_text(),
        "broyden_tri4": broyden_tri_text(4, -2, 2),
        "broyden_tri6": broyden_tri_text(6, -2, 2),
        "broyden_banded12": broyden_banded_text(12, -1, 1),
        "broyden_banded6": broyden_banded_text(6, -1, 1),
        "brown8": brown_text(8, -2, 2),
        "brown5": brown_text(5, -2, 2),
        "quirk17b": quirk17b_text(),
    }


def load_system(name):
    syn = synthetic_texts()
    if name in syn:
        return poly.parse_system(syn[name], name=name)
    return corpus.load(name)


def all_system_names():
    return list(synthetic_texts()) + corpus.names()


def poly_to_json(p):
    return [[m.coeff.hex(), list(m.exps)] for m in p.monomials]


def system_to_json(s):
    return {
        "n": s.dimension,
        "var_names": list(s.var_names),
        "init_lo": [iv.lo.hex() for iv in s.initial_box],
        "init_hi": [iv.hi.hex() for iv in s.initial_box],
        "eqs": [poly_to_json(p) for p in s.polynomials],
        "jac": [[poly_to_json(q) for q in row] for row in s.jacobian()],
        "source": s.source_equations and list(s.source_equations) or [],
    }


def part_systems():
    out = {}
    for name in all_system_names():
        out[name] = system_to_json(load_system(name))
    texts = synthetic_texts()
    meta = {"generated_by": "tests/golden/make_golden.py", "rootbox_version": rootbox.__version__,
            "synthetic_texts": texts}
    with open(os.path.join(HERE, "systems.json"), "w") as f:
        json.dump({"meta": meta, "systems": out}, f, indent=1, sort_keys=True)
    print(f"systems: {len(out)}")


# ---------------------------------------------------------------- interval KATs


def _rand_doubles(rng, m, kind):
    if kind == "solver":
        # dyadic-ish values of moderate magnitude, like box endpoints/midpoints
        v = rng.uniform(-16, 16, m)
        k = rng.integers(0, 40, m)
        v = np.where(rng.random(m) < 0.5, np.round(v * 2.0 ** k) / 2.0 ** k, v)
        return v
    if kind == "wide":
        mant = rng.uniform(1.0, 2.0, m)
        ex = rng.integers(-1074, 1023, m)
        sgn = np.where(rng.random(m) < 0.5, -1.0, 1.0)
        return sgn * np.ldexp(mant, ex)
    if kind == "edge":
        pool = np.array([0.0, -0.0, 1.0, -1.0, 0.5, 2.0 ** -970, 2.0 ** -969, 2.0 ** 995, 2.0 ** 996,
                         -(2.0 ** 995), 5e-324, -5e-324, sys.float_info.max, -sys.float_info.max,
                         math.inf, -math.inf, 3.0, 1e-300, 1e300, 0.1, 2.0 ** -1022,
                         1.0 + 2.0 ** -52, 134217729.0])
        return pool[rng.integers(0, pool.size, m)]
    raise ValueError(kind)


def part_interval():
    rng = np.random.default_rng(20261018)
    m = 4000
    a_parts, b_parts = [], []
    for ka in ("solver", "wide", "edge"):
        for kb in ("solver", "wide", "edge"):
            a_parts.append(_rand_doubles(rng, m, ka))
            b_parts.append(_rand_doubles(rng, m, kb))
    a = np.concatenate(a_parts)
    b = np.concatenate(b_parts)
    fin = np.isfinite(a) & np.isfinite(b)
    res = {"a": a, "b": b}
    for nm in ("_add_rd", "_add_ru", "_mul_rd", "_mul_ru"):
        fn = getattr(interval, nm)
        res[nm] = np.array([fn(float(x), float(y)) for x, y in zip(a, b)])
    for nm in ("_div_rd", "_div_ru"):
        fn = getattr(interval, nm)
        out = []
        for x, y in zip(a, b):
            if y == 0.0:
                out.append(np.nan)  # never called with a zero divisor on the path
            else:
                out.append(fn(float(x), float(y)))
        res[nm] = np.array(out)
    # array twins (_batch.py:31-87) on finite operands
    from rootbox import _batch
    res["fin"] = fin
    with np.errstate(all="ignore"):
        for nm in ("_add_rd", "_add_ru", "_mul_rd", "_mul_ru"):
            res["batch" + nm] = getattr(_batch, nm)(a, b)

    # interval-level ops on random intervals (solver + wide magnitudes)
    def rand_iv(kind, m):
        x = _rand_doubles(rng, m, kind)
        y = _rand_doubles(rng, m, kind)
        lo = np.minimum(x, y)
        hi = np.maximum(x, y)
        # some degenerate and sign-definite ones
        d = rng.random(m)
        hi = np.where(d < 0.05, lo, hi)
        lo = np.where((d > 0.05) & (d < 0.10), 0.0, lo)
        hi = np.where((d > 0.10) & (d < 0.15), np.maximum(lo, 0.0), hi)
        return np.minimum(lo, hi), np.maximum(lo, hi)

    xl, xh, yl, yh = [], [], [], []
    for kind in ("solver", "wide", "edge"):
        a1, a2 = rand_iv(kind, 6000)
        b1, b2 = rand_iv(kind, 6000)
        xl.append(a1); xh.append(a2); yl.append(b1); yh.append(b2)
    xl = np.concatenate(xl); xh = np.concatenate(xh); yl = np.concatenate(yl); yh = np.concatenate(yh)
    keep = np.isfinite(xl) & np.isfinite(xh) & np.isfinite(yl) & np.isfinite(yh)
    xl, xh, yl, yh = xl[keep], xh[keep], yl[keep], yh[keep]
    res.update(xl=xl, xh=xh, yl=yl, yh=yh)
    mlo, mhi, rlo, rhi = [], [], [], []
    powlo = {k: [] for k in range(0, 7)}
    powhi = {k: [] for k in range(0, 7)}
    mid = []
    dk, dp0l, dp0h, dp1l, dp1h = [], [], [], [], []
    kinds = {"empty": 0, "single": 1, "split": 2, "whole": 3}
    for i in range(xl.size):
        X = Interval(xl[i], xh[i])
        Y = Interval(yl[i], yh[i])
        P = X * Y
        mlo.append(P.lo); mhi.append(P.hi)
        for k in range(0, 7):
            Q = X ** k
            powlo[k].append(Q.lo); powhi[k].append(Q.hi)
        mid.append(X.mid)
        if Y.contains_zero():
            rlo.append(np.nan); rhi.append(np.nan)
        else:
            R = Y.recip()
            rlo.append(R.lo); rhi.append(R.hi)
        D = interval.div_extended(X, Y)
        dk.append(kinds[D.kind])
        parts = list(D.parts) + [None, None]
        dp0l.append(parts[0].lo if parts[0] else np.nan)
        dp0h.append(parts[0].hi if parts[0] else np.nan)
        dp1l.append(parts[1].lo if parts[1] else np.nan)
        dp1h.append(parts[1].hi if parts[1] else np.nan)
    res.update(mul_lo=np.array(mlo), mul_hi=np.array(mhi), recip_lo=np.array(rlo),
               recip_hi=np.array(rhi), mid=np.array(mid), div_kind=np.array(dk, dtype=np.int8),
               div_p0_lo=np.array(dp0l), div_p0_hi=np.array(dp0h),
               div_p1_lo=np.array(dp1l), div_p1_hi=np.array(dp1h))
    for k in range(0, 7):
        res[f"pow{k}_lo"] = np.array(powlo[k])
        res[f"pow{k}_hi"] = np.array(powhi[k])
    np.savez_compressed(os.path.join(HERE, "kat_interval.npz"), **res)
    print(f"interval: {a.size} scalar pairs, {xl.size} interval pairs")


# ---------------------------------------------------------------- poly / gj / hs KATs


def random_cells(rng, s, P, depth):
    n = s.dimension
    L = np.array([iv.lo for iv in s.initial_box])
    H = np.array([iv.hi for iv in s.initial_box])
    k = rng.integers(0, 2 ** depth, (P, n))
    lo = L + k * (H - L) / 2 ** depth
    hi = L + (k + 1) * (H - L) / 2 ** depth
    return lo, hi


POLY_SYSTEMS = ["circle_line", "broyden_tri6", "katsura6", "eco8", "brown8", "broyden_banded12",
                "cyclic5", "reimer5", "noon5", "kinema", "caprasse", "mickey"]


def part_poly():
    rng = np.random.default_rng(7)
    res = {}
    for name in POLY_SYSTEMS:
        s = load_system(name)
        n = s.dimension
        jac = s.jacobian()
        los, his = [], []
        for depth in (1, 3, 6, 20):
            lo, hi = random_cells(rng, s, 48, depth)
            los.append(lo); his.append(hi)
        lo = np.concatenate(los); hi = np.concatenate(his)
        F = np.zeros((lo.shape[0], n, 2))
        J = np.zeros((lo.shape[0], n * n, 2))
        for r in range(lo.shape[0]):
            b = poly.Box.from_bounds(lo[r], hi[r])
            for i, p in enumerate(s.polynomials):
                v = p.eval_interval(b)
                F[r, i] = (v.lo, v.hi)
            for i in range(n):
                for j in range(n):
                    v = jac[i][j].eval_interval(b)
                    J[r, i * n + j] = (v.lo, v.hi)
        res[f"{name}_lo"] = lo
        res[f"{name}_hi"] = hi
        res[f"{name}_F"] = F
        res[f"{name}_J"] = J
    np.savez_compressed(os.path.join(HERE, "kat_poly.npz"), **res)
    print(f"poly: {len(POLY_SYSTEMS)} systems")


def part_gj():
    rng = np.random.default_rng(11)
    mats, invs, sing = [], [], []
    for n in (1, 2, 3, 6, 8, 12):
        for t in range(60):
            a = rng.normal(size=(n, n))
            if t % 10 == 0:
                a[:, 0] = a[:, -1] * 2.0 if n > 1 else 0.0  # exactly singular
            if t % 10 == 1:
                a = a * 1e-8
            if t % 10 == 2:
                a[rng.random((n, n)) < 0.4] = 0.0
            if t % 10 == 3:
                a = np.round(a * 4) / 4  # ties in pivot magnitude
            pm = linalg.PointMatrix(n, n, tuple(float(v) for v in a.ravel()))
            try:
                inv = linalg.gauss_jordan_inverse(pm)
                out = np.array(inv.entries).reshape(n, n)
                s_ = False
            except linalg.Singular:
                out = np.full((n, n), np.nan)
                s_ = True
            pad = np.full((12, 12), np.nan)
            pad[:n, :n] = a
            mats.append(pad)
            padi = np.full((12, 12), np.nan)
            padi[:n, :n] = out
            invs.append(padi)
            sing.append((n, s_))
    np.savez_compressed(os.path.join(HERE, "kat_gj.npz"), a=np.array(mats), inv=np.array(invs),
                        n=np.array([x[0] for x in sing]), singular=np.array([x[1] for x in sing]))
    print(f"gj: {len(mats)} matrices")


HS_SYSTEMS = ["circle_line", "broyden_tri6", "katsura6", "brown8", "eco8", "mickey", "noon3",
              "rediff3", "broyden_banded6", "quirk17b"]


def part_hs():
    rng = np.random.default_rng(13)
    res = {}
    for name in HS_SYSTEMS:
        s = load_system(name)
        jac = s.jacobian()
        los, his = [], []
        for depth in (2, 4, 8, 16, 26):
            lo, hi = random_cells(rng, s, 40, depth)
            los.append(lo); his.append(hi)
        lo = np.concatenate(los); hi = np.concatenate(his)
        kind = []
        olo, ohi = [], []
        cert = []
        for r in range(lo.shape[0]):
            b = poly.Box.from_bounds(lo[r], hi[r])
            oc = hansen.contract(s, jac, b)
            kind.append({"empty": 0, "skipped": 3}.get(oc.kind, len(oc.boxes)))
            cert.append(oc.existence_certified)
            bx = list(oc.boxes) + [None, None]
            for k in range(2):
                if bx[k] is None:
                    olo.append([np.nan] * s.dimension); ohi.append([np.nan] * s.dimension)
                else:
                    olo.append([iv.lo for iv in bx[k]]); ohi.append([iv.hi for iv in bx[k]])
        res[f"{name}_lo"] = lo
        res[f"{name}_hi"] = hi
        res[f"{name}_kind"] = np.array(kind, dtype=np.int8)
        res[f"{name}_cert"] = np.array(cert)
        res[f"{name}_olo"] = np.array(olo).reshape(lo.shape[0], 2, s.dimension)
        res[f"{name}_ohi"] = np.array(ohi).reshape(lo.shape[0], 2, s.dimension)
    np.savez_compressed(os.path.join(HERE, "kat_hs.npz"), **res)
    print(f"hs: {len(HS_SYSTEMS)} systems")


# ---------------------------------------------------------------- solves


def box_digest(lo, hi, cert, unsplit):
    h = hashlib.sha256()
    lo = np.where(lo == 0.0, 0.0, lo)  # canonical +0
    hi = np.where(hi == 0.0, 0.0, hi)
    h.update(np.ascontiguousarray(lo, dtype="<f8").tobytes())
    h.update(np.ascontiguousarray(hi, dtype="<f8").tobytes())
    h.update(np.ascontiguousarray(cert, dtype=np.uint8).tobytes())
    h.update(np.ascontiguousarray(unsplit, dtype=np.uint8).tobytes())
    return h.hexdigest()


# (case name, system, config kwargs, capture per-round operator I/O, keep_rows)
SOLVE_CASES = [
    ("circle_line", "circle_line", dict(target_width=1e-6), True),
    ("broyden_tri6", "broyden_tri6", dict(target_width=1e-8), True),
    ("broyden_tri4", "broyden_tri4", dict(target_width=1e-8), True),
    ("mickey", "mickey", dict(), True),
    ("conform1", "conform1", dict(), False),
    ("noon3", "noon3", dict(), True),
    ("rediff3", "rediff3", dict(), True),
    ("gaukwa2", "gaukwa2", dict(), False),
    ("katsura3", "katsura3", dict(), True),
    ("noon4", "noon4", dict(), False),
    ("quirk17b", "quirk17b", dict(target_width=1e-12), False),
    ("circle_line_nohs", "circle_line", dict(target_width=1e-6, hs_enable_width=None), False),
    ("broyden_tri4_nocontract", "broyden_tri4", dict(target_width=1e-8, hs_contract=False), False),
    ("broyden_tri4_hsround0", "broyden_tri4", dict(target_width=1e-8, hs_enable_round=0,
                                                   hs_enable_width=None), False),
    ("mickey_maxboxes", "mickey", dict(max_boxes=3), False),
    ("rediff3_rounds3", "rediff3", dict(max_rounds=3), False),
    ("brown5", "brown5", dict(target_width=1e-8), False),
    ("wide_circle", "wide_circle", dict(target_width=1e-6), True),
    ("wide_circle_r8", "wide_circle", dict(target_width=1e-6, max_rounds=8, hs_enable_round=1,
                                          hs_enable_width=None), False),
    ("broyden_banded6", "broyden_banded6", dict(target_width=1e-8), False),
    # slow (tens of seconds to minutes on one core)
    ("trinks1", "trinks1", dict(), False),
    ("boon", "boon", dict(), False),
    ("eco6", "eco6", dict(), False),
    ("katsura6_r3", "katsura6", dict(max_rounds=3), True),
    ("brown8_r2", "brown8", dict(target_width=1e-8, max_rounds=2), True),
    ("eco8_r2", "eco8", dict(max_rounds=2), True),
    ("broyden_banded12_r1", "broyden_banded12", dict(target_width=1e-8, max_rounds=1), True),
]
SLOW = {"trinks1", "boon", "eco6", "katsura6_r3", "brown8_r2", "eco8_r2", "broyden_banded12_r1"}
CAP_ROWS = 4096  # rows of operator I/O kept per round


def run_solve_case(case):
    cname, sname, kw, capture = case
    s = load_system(sname)
    cfg = bnb.SolverConfig(**kw)
    state = {"round": 1}
    caps = {}
    orig_chunk, orig_hs, orig_rs = bnb._chunk_batch, bnb._hs_pass, bnb.RoundStats

    def chunk_hook(args):
        out = orig_chunk(args)
        r = state["round"]
        ent = caps.setdefault(("f", r), [])
        if sum(a[1].shape[0] for a in ent) < CAP_ROWS:
            ent.append((args[1].copy(), args[2].copy(), out[0].copy(), out[1].copy()))
        return out

    def hs_hook(s_, jac, lo, hi, contract_output):
        out = orig_hs(s_, jac, lo, hi, contract_output)
        r = state["round"]
        ent = caps.setdefault(("h", r), [])
        if sum(a[0].shape[0] for a in ent) < CAP_ROWS:
            ent.append((lo.copy(), hi.copy(), out[0].copy(), out[1].copy(), out[2].copy()))
        return out

    def rs_hook(**k):
        state["round"] += 1
        return orig_rs(**k)

    if capture:
        bnb._chunk_batch, bnb._hs_pass, bnb.RoundStats = chunk_hook, hs_hook, rs_hook
    try:
        t0 = time.perf_counter()
        res = bnb.solve(s, cfg)
        wall = time.perf_counter() - t0
    finally:
        bnb._chunk_batch, bnb._hs_pass, bnb.RoundStats = orig_chunk, orig_hs, orig_rs
    n = s.dimension
    N = len(res.boxes)
    lo = np.array([[iv.lo for iv in rb.box] for rb in res.boxes]).reshape(N, n)
    hi = np.array([[iv.hi for iv in rb.box] for rb in res.boxes]).reshape(N, n)
    cert = np.array([rb.certified for rb in res.boxes], dtype=bool)
    uns = np.array([rb.unsplittable for rb in res.boxes], dtype=bool)
    out = {
        "case": cname, "system": sname, "config": kw, "status": res.status,
        "wall_seconds_reference": wall,
        "stats": [[st.round, st.boxes_in, st.boxes_after_filter, st.boxes_after_hs, st.width.hex()]
                  for st in res.stats],
        "nboxes": N, "ncert": int(cert.sum()), "nunsplit": int(uns.sum()),
        "digest": box_digest(lo, hi, cert, uns),
    }
    if N <= 2000:
        out["lo"] = [[v.hex() for v in row] for row in lo]
        out["hi"] = [[v.hex() for v in row] for row in hi]
        out["cert"] = cert.astype(int).tolist()
        out["unsplit"] = uns.astype(int).tolist()
    # merged report (cli.run_pipeline) for the JSON-equality check
    if N <= 2000:
        from rootbox import cli
        rep = cli.run_pipeline(s, cfg)
        d = rep.to_json_dict()
        for st in d["rounds"]:
            st["elapsed_seconds"] = 0.0
        d["wall_seconds"] = 0.0
        out["report"] = d
    with open(os.path.join(HERE, f"solve_{cname}.json"), "w") as f:
        json.dump(out, f, indent=1)
    if capture and caps:
        arrs = {}
        for (kind, r), ent in sorted(caps.items()):
            if kind == "f":
                arrs[f"f{r}_plo"] = np.concatenate([e[0] for e in ent])
                arrs[f"f{r}_phi"] = np.concatenate([e[1] for e in ent])
                arrs[f"f{r}_olo"] = np.concatenate([e[2] for e in ent])
                arrs[f"f{r}_ohi"] = np.concatenate([e[3] for e in ent])
                arrs[f"f{r}_ocount"] = np.array([e[2].shape[0] for e in ent])
                arrs[f"f{r}_pcount"] = np.array([e[0].shape[0] for e in ent])
            else:
                arrs[f"h{r}_lo"] = np.concatenate([e[0] for e in ent])
                arrs[f"h{r}_hi"] = np.concatenate([e[1] for e in ent])
                arrs[f"h{r}_olo"] = np.concatenate([e[2] for e in ent])
                arrs[f"h{r}_ohi"] = np.concatenate([e[3] for e in ent])
                arrs[f"h{r}_ocert"] = np.concatenate([e[4] for e in ent])
                arrs[f"h{r}_icount"] = np.array([e[0].shape[0] for e in ent])
                arrs[f"h{r}_ocount"] = np.array([e[2].shape[0] for e in ent])
        arrs["contract"] = np.array(cfg.hs_contract)
        np.savez_compressed(os.path.join(HERE, f"rounds_{cname}.npz"), **arrs)
    return cname, res.status, N, wall


def part_solve(which, only=None):
    cases = [c for c in SOLVE_CASES if (c[0] in SLOW) == (which == "slow")]
    if only:
        cases = [c for c in SOLVE_CASES if c[0] in only]
    with ProcessPoolExecutor(max_workers=min(8, len(cases))) as ex:
        for cname, status, N, wall in ex.map(run_solve_case, cases):
            print(f"solve {cname}: {status} boxes={N} wall={wall:.1f}s", flush=True)


# ---------------------------------------------------------------- merge (backtrack.py)


def _merge_case(init_lo, init_hi, lo, hi, cert, stop_width):
    from rootbox import backtrack
    g = backtrack.GridContext.from_box(poly.Box.from_bounds(init_lo, init_hi))
    try:
        snapped = [backtrack.snap_to_grid(poly.Box.from_bounds(lo[r], hi[r]), g) for r in range(lo.shape[0])]
        m = backtrack.merge_to_width(snapped, g, stop_width=stop_width, certified=list(cert))
    except ValueError as exc:
        return {"error": type(exc).__name__}
    return {"levels": [[w.hex(), c] for w, c in m.levels],
            "lo": [[iv.lo.hex() for iv in b] for b in m.boxes],
            "hi": [[iv.hi.hex() for iv in b] for b in m.boxes],
            "cert": [int(f) for f in m.certified]}


def part_merge():
    rng = np.random.default_rng(17)
    cases = []
    # solve outputs (the pipeline's real inputs), with and without a stop width
    for fn in sorted(os.listdir(HERE)):
        if not (fn.startswith("solve_") and fn.endswith(".json")):
            continue
        d = json.load(open(os.path.join(HERE, fn)))
        if "lo" not in d or not d["lo"] or d["status"] == "budget_exhausted":
            continue
        sysd = json.load(open(os.path.join(HERE, "systems.json")))["systems"][d["system"]]
        ilo = np.array([float.fromhex(v) for v in sysd["init_lo"]]); ihi = np.array([float.fromhex(v) for v in sysd["init_hi"]])
        lo = np.array([[float.fromhex(v) for v in r] for r in d["lo"]]); hi = np.array([[float.fromhex(v) for v in r] for r in d["hi"]])
        cert = np.array(d["cert"], bool)
        for sw in (None, 0.01):
            cases.append({"name": f"{d['case']}_sw{sw}", "init_lo": ilo, "init_hi": ihi, "lo": lo, "hi": hi,
                          "cert": cert, "stop_width": sw})
    # synthetic sets: aligned cells, contracted sub-boxes, boundary-straddling boxes, point boxes
    for t, (L0, H0) in enumerate([(-2.0, 2.0), (-8.0, 8.0), (0.0, 1.0), (-1.0, 3.0), (-0.75, 0.25), (0.0, 3.0)]):
        n = 3
        ilo = np.full(n, L0); ihi = np.full(n, H0)
        W = H0 - L0
        m = 300
        lev = rng.integers(3, 30, m)
        k = (rng.random((m, n)) * (2.0 ** lev[:, None])).astype(np.int64)
        cl = L0 + k * (W / 2.0 ** lev[:, None]); ch = L0 + (k + 1) * (W / 2.0 ** lev[:, None])
        f = rng.random((m, 1))
        sub_lo = cl + (ch - cl) * rng.random((m, n)) * 0.3
        sub_hi = ch - (ch - cl) * rng.random((m, n)) * 0.3
        straddle = rng.random(m) < 0.2
        sub_hi[straddle] = np.minimum(ch[straddle] + (ch - cl)[straddle] * 0.5, H0)
        pt = rng.random(m) < 0.05
        sub_hi[pt] = sub_lo[pt]
        lo = np.where(f < 0.5, cl, sub_lo); hi = np.where(f < 0.5, ch, sub_hi)
        cert = rng.random(m) < 0.3
        for sw in (None, 0.5):
            cases.append({"name": f"synthetic{t}_sw{sw}", "init_lo": ilo, "init_hi": ihi, "lo": lo, "hi": hi,
                          "cert": cert, "stop_width": sw})
    # deep levels: boxes far narrower than 2^-120 of the initial width (an HS-contracted box
    # around a root at the origin) -- snap_to_grid has no level limit (backtrack.py:118-158)
    ilo = np.array([-2.0, -2.0]); ihi = np.array([2.0, 2.0])
    deep = [([0.0, -1e-300], [1e-40, 0.0]), ([1.0, 1.0], [1.0 + 2.0 ** -30, 1.0 + 2.0 ** -30]),
            ([2.0 ** -200, -2.0 ** -180], [2.0 ** -199, -2.0 ** -181]), ([0.25, 0.25], [0.25, 0.25]),
            ([-1.0, 0.5], [-0.5, 1.0]), ([-0.75, 0.5], [-0.75 + 2.0 ** -300, 0.5 + 2.0 ** -300])]
    lo = np.array([d[0] for d in deep]); hi = np.array([d[1] for d in deep])
    for sw in (None, 0.5):
        cases.append({"name": f"deep_levels_sw{sw}", "init_lo": ilo, "init_hi": ihi, "lo": lo, "hi": hi,
                      "cert": np.array([1, 0, 1, 0, 0, 1], bool), "stop_width": sw})
        cases.append({"name": f"deep_levels_advice_sw{sw}", "init_lo": ilo, "init_hi": ihi, "lo": lo[:2],
                      "hi": hi[:2], "cert": np.array([0, 1], bool), "stop_width": sw})
    # a deep cell whose other component (a point at -0.5) cannot be materialised exactly
    # at that level: locate() then gives per-component levels (rb_merge: uniform levels only)
    cases.append({"name": "deep_levels_mixed_swNone", "init_lo": ilo, "init_hi": ihi,
                  "lo": np.array([[2.0 ** -200, -0.5]]), "hi": np.array([[2.0 ** -199, -0.5]]),
                  "cert": np.array([1], bool), "stop_width": None})
    out = []
    for c in cases:
        r = _merge_case(c["init_lo"], c["init_hi"], c["lo"], c["hi"], c["cert"], c["stop_width"])
        out.append({"name": c["name"], "init_lo": [v.hex() for v in c["init_lo"]],
                    "init_hi": [v.hex() for v in c["init_hi"]],
                    "lo": [[float(v).hex() for v in r_] for r_ in c["lo"]],
                    "hi": [[float(v).hex() for v in r_] for r_ in c["hi"]],
                    "cert": [int(v) for v in c["cert"]], "stop_width": c["stop_width"], "result": r})
    with open(os.path.join(HERE, "merge_cases.json"), "w") as f:
        json.dump(out, f)
    print(f"merge: {len(out)} cases, {sum('error' in o['result'] for o in out)} raise")


def part_krawczyk():
    rng = np.random.default_rng(19)
    res = {}
    for name in ["circle_line", "broyden_tri6", "katsura6", "brown8", "mickey", "noon3", "broyden_banded6",
                 "quirk17b", "eco8"]:
        s = load_system(name)
        jac = s.jacobian()
        los, his = [], []
        for depth in (2, 6, 12, 24, 40):
            lo, hi = random_cells(rng, s, 40, depth)
            los.append(lo); his.append(hi)
        lo = np.concatenate(los); hi = np.concatenate(his)
        ok, olo, ohi = [], [], []
        for r in range(lo.shape[0]):
            k = hansen.krawczyk(s, jac, poly.Box.from_bounds(lo[r], hi[r]))
            ok.append(k is not None)
            olo.append([iv.lo for iv in k] if k is not None else [np.nan] * s.dimension)
            ohi.append([iv.hi for iv in k] if k is not None else [np.nan] * s.dimension)
        res[f"{name}_lo"] = lo; res[f"{name}_hi"] = hi
        res[f"{name}_ok"] = np.array(ok); res[f"{name}_olo"] = np.array(olo); res[f"{name}_ohi"] = np.array(ohi)
    np.savez_compressed(os.path.join(HERE, "kat_krawczyk.npz"), **res)
    print("krawczyk:", {k[:-3]: int(v.sum()) for k, v in res.items() if k.endswith("_ok")})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--part", nargs="*", default=["systems", "interval", "poly", "gj", "hs", "solve"])
    ap.add_argument("--case", nargs="*", default=None, help="solve only these SOLVE_CASES")
    a = ap.parse_args()
    for p in a.part:
        t0 = time.time()
        if p == "systems":
            part_systems()
        elif p == "interval":
            part_interval()
        elif p == "poly":
            part_poly()
        elif p == "gj":
            part_gj()
        elif p == "hs":
            part_hs()
        elif p == "solve":
            part_solve("fast", a.case)
        elif p == "solve_slow":
            part_solve("slow")
        elif p == "merge":
            part_merge()
        elif p == "krawczyk":
            part_krawczyk()
        print(f"[{p}] {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()

"""Known real roots of the benchmark and golden systems, for the enclosure checks.

TEST INFRASTRUCTURE ONLY (never imported by the product package).

The reference's own soundness / completeness oracles (acceptance
criteria 4-5) are damped Newton from random starts, refined in high precision;
north_star asks that both runs "enclose every known real root".  This script
computes those roots independently of any interval code:

  1. 10^4 random starts in the initial box (numpy.random.default_rng(seed)), damped
     Newton in float64 on F and its Jacobian (the exact canonical polynomials of
     tests/golden/systems.json, i.e. rootbox.poly.PolySystem / jacobian);
  2. converged points (max|f| < 1e-10) are clustered and each cluster is refined by
     Newton in 256-bit arithmetic (mpmath) until the step is < 2^-200;
  3. a root is kept when it lies in the closed initial box and max|f| < 1e-30 at
     the refined point.

Each root is written as its two neighbouring doubles RD(r) <= r <= RU(r): for a
box with double endpoints, lo <= r <= hi  <=>  lo <= RD(r) and RU(r) <= hi, so the
tests check enclosure exactly with float64 compares.  Known closed forms are
added and cross-checked: circle-line (+-sqrt(1/2), +-sqrt(1/2)), Brown's
(1, ..., 1).

    python tests/golden/make_roots.py          ->  tests/golden/roots.json
"""
from __future__ import annotations

import json
import os
import sys
import time

import mpmath
import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

SYSTEMS = ["circle_line", "broyden_tri6", "broyden_tri4", "katsura6", "eco8", "brown8", "broyden_banded12",
           "mickey", "noon3", "noon4", "rediff3", "gaukwa2", "katsura3", "brown5", "broyden_banded6",
           "trinks1", "boon", "eco6", "conform1", "quirk17b"]
STARTS = 10_000
mpmath.mp.prec = 256


def load(name):
    with open(os.path.join(HERE, "systems.json")) as f:
        d = json.load(f)["systems"][name]
    eqs = [[(float.fromhex(c), tuple(e)) for c, e in p] for p in d["eqs"]]
    jac = [[[(float.fromhex(c), tuple(e)) for c, e in q] for q in row] for row in d["jac"]]
    lo = np.array([float.fromhex(v) if isinstance(v, str) else float(v) for v in d["init_lo"]])
    hi = np.array([float.fromhex(v) if isinstance(v, str) else float(v) for v in d["init_hi"]])
    return d["n"], eqs, jac, lo, hi


def _np_poly(terms, X):
    """sum_t c_t prod_j x_j^e_tj over rows of X (M, n)."""
    out = np.zeros(X.shape[0])
    for c, e in terms:
        t = np.full(X.shape[0], c)
        for j, k in enumerate(e):
            if k:
                t = t * X[:, j] ** k
        out += t
    return out


def _mp_poly(terms, x):
    s = mpmath.mpf(0)
    for c, e in terms:
        t = mpmath.mpf(c)
        for j, k in enumerate(e):
            if k:
                t *= x[j] ** k
        s += t
    return s


def newton_float(n, eqs, jac, lo, hi, seed):
    rng = np.random.default_rng(seed)
    X = lo + (hi - lo) * rng.random((STARTS, n))
    span = np.max(hi - lo)
    for _ in range(80):
        F = np.stack([_np_poly(p, X) for p in eqs], axis=1)
        J = np.stack([np.stack([_np_poly(q, X) for q in row], axis=1) for row in jac], axis=1)
        ok = np.all(np.isfinite(F), axis=1) & np.all(np.isfinite(J.reshape(len(X), -1)), axis=1)
        step = np.zeros_like(X)
        good = ok & (np.abs(np.linalg.det(np.where(ok[:, None, None], J, np.eye(n)))) > 1e-300)
        if good.any():
            try:
                step[good] = np.linalg.solve(J[good], F[good][..., None])[..., 0]
            except np.linalg.LinAlgError:
                pass
        # damping: cap the step at half the box span
        nrm = np.max(np.abs(step), axis=1, keepdims=True)
        step = np.where(nrm > 0.5 * span, step * (0.5 * span / np.maximum(nrm, 1e-300)), step)
        X = X - step
        X = np.where(np.isfinite(X), X, lo + (hi - lo) * rng.random(X.shape))
    F = np.stack([_np_poly(p, X) for p in eqs], axis=1)
    conv = np.all(np.isfinite(F), axis=1) & (np.max(np.abs(F), axis=1) < 1e-10)
    return X[conv]


def refine(n, eqs, jac, x0):
    x = [mpmath.mpf(float(v)) for v in x0]
    for _ in range(40):
        F = mpmath.matrix([_mp_poly(p, x) for p in eqs])
        J = mpmath.matrix([[_mp_poly(q, x) for q in row] for row in jac])
        try:
            d = mpmath.lu_solve(J, F)
        except ZeroDivisionError:
            return None
        x = [x[i] - d[i] for i in range(n)]
        if max(abs(d[i]) for i in range(n)) < mpmath.mpf(2) ** -200:
            break
    fmax = max(abs(_mp_poly(p, x)) for p in eqs)
    if not fmax < mpmath.mpf(10) ** -30:
        return None
    return x


def neighbours(v):
    """(RD(v), RU(v)) as doubles for an mpf v."""
    f = float(v)  # round to nearest
    if mpmath.mpf(f) > v:
        return float(np.nextafter(f, -np.inf)), f
    if mpmath.mpf(f) < v:
        return f, float(np.nextafter(f, np.inf))
    return f, f


def roots_of(name, seed=0):
    n, eqs, jac, lo, hi = load(name)
    X = newton_float(n, eqs, jac, lo, hi, seed)
    extra = []
    if name == "circle_line":
        s = float(mpmath.sqrt(mpmath.mpf(1) / 2))
        extra = [[s, s], [-s, -s]]
    if name.startswith("brown"):
        extra = [[1.0] * n]
    cand = np.concatenate([X, np.array(extra).reshape(-1, n)]) if len(extra) else X
    found = []
    for x0 in cand:
        if any(np.max(np.abs(x0 - np.array([float(v) for v in r]))) < 1e-7 for r in found):
            continue
        r = refine(n, eqs, jac, x0)
        if r is None:
            continue
        if not all(mpmath.mpf(lo[i]) <= r[i] <= mpmath.mpf(hi[i]) for i in range(n)):
            continue
        if any(max(abs(r[i] - q[i]) for i in range(n)) < mpmath.mpf(2) ** -100 for q in found):
            continue
        found.append(r)
    for e in extra:  # closed forms must be among the roots
        assert any(max(abs(float(q[i]) - e[i]) for i in range(n)) < 1e-12 for q in found), (name, e)
    found.sort(key=lambda r: [float(v) for v in r])
    return {
        "n": n, "starts": STARTS, "seed": seed, "converged_starts": int(X.shape[0]),
        "roots_rd": [[neighbours(v)[0].hex() for v in r] for r in found],
        "roots_ru": [[neighbours(v)[1].hex() for v in r] for r in found],
        "roots_dec": [[mpmath.nstr(v, 40) for v in r] for r in found],
    }


def main():
    names = sys.argv[1:] or SYSTEMS
    path = os.path.join(HERE, "roots.json")
    out = {}
    if os.path.exists(path):
        with open(path) as f:
            out = json.load(f).get("systems", {})
    for name in names:
        t0 = time.time()
        out[name] = roots_of(name)
        print(f"{name}: {len(out[name]['roots_rd'])} real roots ({out[name]['converged_starts']} of {STARTS} "
              f"starts converged) {time.time() - t0:.1f} s", flush=True)
    with open(path, "w") as f:
        json.dump({"generator": "tests/golden/make_roots.py", "systems": out}, f, indent=1)


if __name__ == "__main__":
    main()

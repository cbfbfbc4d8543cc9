"""ctypes binding of the CPU oracle (rootbox_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs.  The product package
(paper_1802_00330_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")

_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(HERE, "rootbox_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        i64 = C.c_int64
        L.o_system_new.restype = P
        L.o_system_new.argtypes = [C.c_int, C.c_int, P, P, P]
        L.o_system_free.argtypes = [P]
        L.o_vec_scalar.argtypes = [C.c_int, i64, P, P, P]
        L.o_vec_interval.argtypes = [C.c_int, i64, P, P, P, P, P, P]
        L.o_vec_divx.argtypes = [i64, P, P, P, P, P, P]
        L.o_eval_F.argtypes = [P, i64, P, P, P]
        L.o_eval_J.argtypes = [P, i64, P, P, P]
        L.o_gj_inverse.argtypes = [C.c_int, P, P]
        L.o_gj_inverse.restype = C.c_int
        L.o_contract_vec.argtypes = [P, i64, P, P, P, P, P, P]
        L.o_krawczyk_vec.argtypes = [P, i64, P, P, P, P, P]
        L.o_chunk_filter.argtypes = [P, i64, P, P, i64, P, P]
        L.o_chunk_filter.restype = i64
        L.o_hs_pass.argtypes = [P, i64, P, P, C.c_int, i64, P, P, P]
        L.o_hs_pass.restype = i64
        L.o_solve.argtypes = [P, P, P, P]
        L.o_solve.restype = P
        L.o_result_status.argtypes = [P]
        L.o_result_nrounds.argtypes = [P]
        L.o_result_nboxes.argtypes = [P]
        L.o_result_nboxes.restype = i64
        L.o_result_wall.argtypes = [P]
        L.o_result_wall.restype = C.c_double
        L.o_result_boxes.argtypes = [P, P, P, P, P]
        L.o_result_stats.argtypes = [P, P]
        L.o_result_free.argtypes = [P]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


class OConfig(C.Structure):
    _fields_ = [
        ("target_width", C.c_double),
        ("hs_enable_round", C.c_int32),
        ("hs_enable_width", C.c_double),
        ("max_rounds", C.c_int32),
        ("max_boxes", C.c_int64),
        ("max_seconds", C.c_double),
        ("hs_contract", C.c_int32),
        ("threads", C.c_int32),
    ]


STATUS = {0: "no_real_solution", 1: "width_reached", 2: "budget_exhausted"}


def _flatten_polys(n, polys):
    off = [0]
    coeff = []
    exps = []
    for p in polys:
        for c, e in p:
            coeff.append(float(c))
            exps.append(list(e))
        off.append(len(coeff))
    return (np.array(off, dtype=np.int32), np.array(coeff, dtype=np.float64),
            np.array(exps, dtype=np.uint8).reshape(-1, n) if exps else np.zeros((0, n), np.uint8))


class OSystem:
    """Oracle view of a polynomial system: F polys then the n*n Jacobian polys,
    each a list of (coeff, exps) in canonical order (poly.py:159)."""

    def __init__(self, n, eqs, jac):
        self.n = n
        polys = list(eqs) + [jac[i][j] for i in range(n) for j in range(n)]
        self._arrs = _flatten_polys(n, polys)
        off, coeff, exps = self._arrs
        self.h = lib().o_system_new(n, len(polys), _p(off), _p(coeff), _p(np.ascontiguousarray(exps)))

    def __del__(self):
        try:
            if self.h:
                lib().o_system_free(self.h)
        except Exception:
            pass

    # -- operators
    def eval_F(self, lo, hi):
        lo = np.ascontiguousarray(lo, np.float64); hi = np.ascontiguousarray(hi, np.float64)
        out = np.empty((lo.shape[0], self.n, 2))
        lib().o_eval_F(self.h, lo.shape[0], _p(lo), _p(hi), _p(out))
        return out

    def eval_J(self, lo, hi):
        lo = np.ascontiguousarray(lo, np.float64); hi = np.ascontiguousarray(hi, np.float64)
        out = np.empty((lo.shape[0], self.n * self.n, 2))
        lib().o_eval_J(self.h, lo.shape[0], _p(lo), _p(hi), _p(out))
        return out

    def contract(self, lo, hi):
        lo = np.ascontiguousarray(lo, np.float64); hi = np.ascontiguousarray(hi, np.float64)
        m = lo.shape[0]
        kind = np.empty(m, np.int8)
        olo = np.empty((m, 2, self.n)); ohi = np.empty((m, 2, self.n))
        cert = np.empty(m, np.uint8)
        lib().o_contract_vec(self.h, m, _p(lo), _p(hi), _p(kind), _p(olo), _p(ohi), _p(cert))
        return kind, olo, ohi, cert.astype(bool)

    def krawczyk(self, lo, hi):
        lo = np.ascontiguousarray(lo, np.float64); hi = np.ascontiguousarray(hi, np.float64)
        m = lo.shape[0]
        ok = np.empty(m, np.uint8); olo = np.empty((m, self.n)); ohi = np.empty((m, self.n))
        lib().o_krawczyk_vec(self.h, m, _p(lo), _p(hi), _p(ok), _p(olo), _p(ohi))
        return ok.astype(bool), olo, ohi

    def chunk_filter(self, plo, phi):
        plo = np.ascontiguousarray(plo, np.float64); phi = np.ascontiguousarray(phi, np.float64)
        P = plo.shape[0]
        cap = max(1, P << self.n)
        olo = np.empty((cap, self.n)); ohi = np.empty((cap, self.n))
        M = lib().o_chunk_filter(self.h, P, _p(plo), _p(phi), cap, _p(olo), _p(ohi))
        return olo[:M].copy(), ohi[:M].copy()

    def hs_pass(self, lo, hi, contract_output=True):
        lo = np.ascontiguousarray(lo, np.float64); hi = np.ascontiguousarray(hi, np.float64)
        M = lo.shape[0]
        cap = max(1, 2 * M)
        olo = np.empty((cap, self.n)); ohi = np.empty((cap, self.n)); oc = np.empty(cap, np.uint8)
        M2 = lib().o_hs_pass(self.h, M, _p(lo), _p(hi), int(contract_output), cap, _p(olo), _p(ohi), _p(oc))
        return olo[:M2].copy(), ohi[:M2].copy(), oc[:M2].astype(bool)

    def solve(self, init_lo, init_hi, target_width=None, hs_enable_round=None, hs_enable_width=1.0,
              max_rounds=24, max_boxes=200_000_000, max_seconds=None, hs_contract=True, threads=1):
        cfg = OConfig(
            target_width=-1.0 if target_width is None else float(target_width),
            hs_enable_round=-1 if hs_enable_round is None else int(hs_enable_round),
            hs_enable_width=float("nan") if hs_enable_width is None else float(hs_enable_width),
            max_rounds=int(max_rounds), max_boxes=int(max_boxes),
            max_seconds=-1.0 if max_seconds is None else float(max_seconds),
            hs_contract=int(bool(hs_contract)), threads=int(threads))
        ilo = np.ascontiguousarray(init_lo, np.float64); ihi = np.ascontiguousarray(init_hi, np.float64)
        L = lib()
        R = L.o_solve(self.h, _p(ilo), _p(ihi), C.byref(cfg))
        try:
            N = L.o_result_nboxes(R)
            nr = L.o_result_nrounds(R)
            lo = np.empty((N, self.n)); hi = np.empty((N, self.n))
            cert = np.empty(N, np.uint8); uns = np.empty(N, np.uint8)
            L.o_result_boxes(R, _p(lo), _p(hi), _p(cert), _p(uns))
            st = np.empty((nr, 9))
            L.o_result_stats(R, _p(st))
            return {
                "status": STATUS[L.o_result_status(R)], "lo": lo, "hi": hi,
                "cert": cert.astype(bool), "unsplit": uns.astype(bool), "stats": st,
                "wall": L.o_result_wall(R),
            }
        finally:
            L.o_result_free(R)


# -- scalar / interval vector entry points (KAT checks)

SCALAR_OPS = {"_add_rd": 0, "_add_ru": 1, "_mul_rd": 2, "_mul_ru": 3, "_div_rd": 4, "_div_ru": 5}


def vec_scalar(name, a, b):
    a = np.ascontiguousarray(a, np.float64); b = np.ascontiguousarray(b, np.float64)
    out = np.empty_like(a)
    lib().o_vec_scalar(SCALAR_OPS[name], a.size, _p(a), _p(b), _p(out))
    return out


def vec_interval(op, xl, xh, yl=None, yh=None):
    xl = np.ascontiguousarray(xl, np.float64); xh = np.ascontiguousarray(xh, np.float64)
    yl = xl if yl is None else np.ascontiguousarray(yl, np.float64)
    yh = xh if yh is None else np.ascontiguousarray(yh, np.float64)
    olo = np.empty_like(xl); ohi = np.empty_like(xl)
    lib().o_vec_interval(op, xl.size, _p(xl), _p(xh), _p(yl), _p(yh), _p(olo), _p(ohi))
    return olo, ohi


def vec_divx(xl, xh, yl, yh):
    arrs = [np.ascontiguousarray(v, np.float64) for v in (xl, xh, yl, yh)]
    m = arrs[0].size
    kind = np.empty(m, np.int8)
    parts = np.empty((m, 4))
    lib().o_vec_divx(m, *[_p(v) for v in arrs], _p(kind), _p(parts))
    return kind, parts


def gj_inverse(a):
    a = np.ascontiguousarray(a, np.float64)
    n = a.shape[0]
    out = np.empty((n, n))
    sing = lib().o_gj_inverse(n, _p(a), _p(out))
    return (None if sing else out)

"""Pin the CPU oracle (oracle/rootbox_oracle.c) against the reference's own
outputs recorded in tests/golden/ (tests/golden/make_golden.py).

Bit-exact: every float64 compared as a bit pattern (signed zero canonicalised,
which only the printing layer can observe)."""
import os

import numpy as np
import pytest

from conftest import (GOLDEN, assert_bits_equal, bits, canonical_sort, golden_jac, golden_spec,
                      golden_systems, load_solve, solve_cases)
from oracle import oracle as O


def osys(name):
    spec = golden_spec(name)
    return O.OSystem(spec.n, spec.eqs, golden_jac(name)), spec


@pytest.fixture(scope="module")
def kat():
    return np.load(os.path.join(GOLDEN, "kat_interval.npz"))


@pytest.mark.parametrize("op", ["_add_rd", "_add_ru", "_mul_rd", "_mul_ru", "_div_rd", "_div_ru"])
def test_scalar_directed_ops(kat, op):
    # interval.py:66-190, including the _TINY/_BIG untrusted band and infinities;
    # raw bits: the scalar reference's signed zeros are reproduced exactly
    got = O.vec_scalar(op, kat["a"], kat["b"])
    ref = kat[op]
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(got[~nan].view(np.uint64), ref[~nan].view(np.uint64)), op


@pytest.mark.parametrize("op", ["_add_rd", "_add_ru", "_mul_rd", "_mul_ru"])
def test_batch_twins_equal_on_finite(kat, op):
    # _batch.py:31-87 agree with the scalar code on finite operands (what the filter sees)
    fin = kat["fin"]
    got = O.vec_scalar(op, kat["a"][fin], kat["b"][fin])
    ref = kat["batch" + op][fin]
    ok = np.isfinite(ref) & np.isfinite(got)
    assert_bits_equal(got[ok], ref[ok], op)


def test_interval_mul_pow_recip_mid(kat):
    xl, xh, yl, yh = kat["xl"], kat["xh"], kat["yl"], kat["yh"]
    lo, hi = O.vec_interval(0, xl, xh, yl, yh)
    assert_bits_equal(lo, kat["mul_lo"], "mul lo")
    assert_bits_equal(hi, kat["mul_hi"], "mul hi")
    for k in range(7):
        lo, hi = O.vec_interval(2 + k, xl, xh)
        assert_bits_equal(lo, kat[f"pow{k}_lo"], f"pow{k} lo")
        assert_bits_equal(hi, kat[f"pow{k}_hi"], f"pow{k} hi")
    lo, hi = O.vec_interval(1, xl, xh, yl, yh)
    assert_bits_equal(lo, kat["recip_lo"], "recip lo")
    assert_bits_equal(hi, kat["recip_hi"], "recip hi")
    lo, _ = O.vec_interval(9, xl, xh)
    ok = np.isfinite(kat["mid"])
    assert_bits_equal(lo[ok], kat["mid"][ok], "mid")


def test_div_extended(kat):
    kind, parts = O.vec_divx(kat["xl"], kat["xh"], kat["yl"], kat["yh"])
    assert np.array_equal(kind, kat["div_kind"])
    assert_bits_equal(parts[:, 0], kat["div_p0_lo"], "p0 lo")
    assert_bits_equal(parts[:, 1], kat["div_p0_hi"], "p0 hi")
    two = kind == 2
    assert_bits_equal(parts[two, 2], kat["div_p1_lo"][two], "p1 lo")
    assert_bits_equal(parts[two, 3], kat["div_p1_hi"][two], "p1 hi")


def test_jacobian_matches_reference(systems):
    # package-side symbolic Jacobian (system.differentiate) == PolySystem.jacobian
    for name in systems:
        spec = golden_spec(name)
        ref = golden_jac(name)
        for i in range(spec.n):
            for j in range(spec.n):
                got = spec.jac[i][j]
                want = ref[i][j]
                assert len(got) == len(want), (name, i, j)
                for (c1, e1), (c2, e2) in zip(got, want):
                    assert e1 == e2 and float(c1).hex() == float(c2).hex(), (name, i, j)


def test_poly_eval():
    d = np.load(os.path.join(GOLDEN, "kat_poly.npz"))
    names = sorted({k.rsplit("_", 1)[0] for k in d.files})
    assert names
    for name in names:
        s, _ = osys(name)
        lo, hi = d[f"{name}_lo"], d[f"{name}_hi"]
        assert_bits_equal(s.eval_F(lo, hi), d[f"{name}_F"], f"{name} F")
        assert_bits_equal(s.eval_J(lo, hi), d[f"{name}_J"], f"{name} J")


def test_gauss_jordan():
    d = np.load(os.path.join(GOLDEN, "kat_gj.npz"))
    for a, inv, n, sing in zip(d["a"], d["inv"], d["n"], d["singular"]):
        got = O.gj_inverse(a[:n, :n])
        if sing:
            assert got is None
        else:
            assert got is not None
            assert_bits_equal(got, inv[:n, :n], f"gj n={n}")


def test_hansen_contract():
    d = np.load(os.path.join(GOLDEN, "kat_hs.npz"))
    names = sorted({k.rsplit("_", 1)[0] for k in d.files if k.endswith("_kind")})
    seen = set()
    for name in names:
        s, _ = osys(name)
        kind, olo, ohi, cert = s.contract(d[f"{name}_lo"], d[f"{name}_hi"])
        assert np.array_equal(kind, d[f"{name}_kind"]), name
        assert np.array_equal(cert, d[f"{name}_cert"]), name
        assert_bits_equal(olo, d[f"{name}_olo"], f"{name} olo")
        assert_bits_equal(ohi, d[f"{name}_ohi"], f"{name} ohi")
        seen.update(kind.tolist())
    assert {0, 1, 2}.issubset(seen)  # empty, single and fork outcomes all covered


def _round_files():
    return sorted(f for f in os.listdir(GOLDEN) if f.startswith("rounds_"))


@pytest.mark.parametrize("fn", _round_files())
def test_round_operators(fn):
    """Per-round _chunk_batch / _hs_pass captures (bnb.py:161-218), same order."""
    case = fn[len("rounds_"):-4]
    meta = load_solve(case)
    s, _ = osys(meta["system"])
    d = np.load(os.path.join(GOLDEN, fn))
    nf = nh = 0
    for k in d.files:
        if k.endswith("_plo"):
            r = k[:-4]
            plo, phi = d[f"{r}_plo"], d[f"{r}_phi"]
            # chunks were recorded back to back; filter each chunk separately
            off_p = np.concatenate([[0], np.cumsum(d[f"{r}_pcount"])])
            off_o = np.concatenate([[0], np.cumsum(d[f"{r}_ocount"])])
            for c in range(len(off_p) - 1):
                glo, ghi = s.chunk_filter(plo[off_p[c]:off_p[c + 1]], phi[off_p[c]:off_p[c + 1]])
                assert_bits_equal(glo, d[f"{r}_olo"][off_o[c]:off_o[c + 1]], f"{case} {r} lo")
                assert_bits_equal(ghi, d[f"{r}_ohi"][off_o[c]:off_o[c + 1]], f"{case} {r} hi")
                nf += 1
        if k.endswith("_ocert"):
            r = k[:-6]
            lo, hi = d[f"{r}_lo"], d[f"{r}_hi"]
            olo, ohi, oc = s.hs_pass(lo, hi, bool(d["contract"]))
            assert_bits_equal(olo, d[f"{r}_olo"], f"{case} {r} hs lo")
            assert_bits_equal(ohi, d[f"{r}_ohi"], f"{case} {r} hs hi")
            assert np.array_equal(oc, d[f"{r}_ocert"])
            nh += 1
    assert nf + nh > 0


def check_solution(case, res, meta):
    """Compare a solve result dict (status/lo/hi/cert/unsplit/stats) with a golden case."""
    assert res["status"] == meta["status"], case
    st = res["stats"]
    assert len(st) == len(meta["stats"]), case
    for got, want in zip(st, meta["stats"]):
        assert [int(got[0]), int(got[1]), int(got[2]), int(got[3])] == want[:4], (case, got, want)
        assert bits(got[4]) == bits(float.fromhex(want[4])), (case, got[4], want[4])
    lo, hi = res["lo"], res["hi"]
    order = canonical_sort(lo, hi)
    lo, hi = lo[order], hi[order]
    cert, uns = res["cert"][order], res["unsplit"][order]
    assert lo.shape[0] == meta["nboxes"]
    assert int(cert.sum()) == meta["ncert"] and int(uns.sum()) == meta["nunsplit"]
    if "lo" in meta:
        assert_bits_equal(lo, np.array([[float.fromhex(v) for v in r] for r in meta["lo"]]).reshape(lo.shape),
                          f"{case} lo")
        assert_bits_equal(hi, np.array([[float.fromhex(v) for v in r] for r in meta["hi"]]).reshape(hi.shape),
                          f"{case} hi")
        assert cert.astype(int).tolist() == meta["cert"]
        assert uns.astype(int).tolist() == meta["unsplit"]
    from conftest import bits as _b  # noqa
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(np.where(lo == 0.0, 0.0, lo), "<f8").tobytes())
    h.update(np.ascontiguousarray(np.where(hi == 0.0, 0.0, hi), "<f8").tobytes())
    h.update(cert.astype(np.uint8).tobytes())
    h.update(uns.astype(np.uint8).tobytes())
    assert h.hexdigest() == meta["digest"], case


FAST_CASES = [c for c in solve_cases() if load_solve(c)["wall_seconds_reference"] < 25]


@pytest.mark.parametrize("case", FAST_CASES)
def test_oracle_solve(case):
    meta = load_solve(case)
    s, spec = osys(meta["system"])
    res = s.solve(spec.init_lo, spec.init_hi, threads=2, **meta["config"])
    check_solution(case, res, meta)


def test_krawczyk():
    """hansen.krawczyk (hansen.py:141-170): K(X) intersected with X, None when singular or empty."""
    d = np.load(os.path.join(GOLDEN, "kat_krawczyk.npz"))
    names = sorted({k.rsplit("_", 1)[0] for k in d.files if k.endswith("_ok")})
    for name in names:
        s, _ = osys(name)
        ok, olo, ohi = s.krawczyk(d[f"{name}_lo"], d[f"{name}_hi"])
        assert np.array_equal(ok, d[f"{name}_ok"]), name
        assert_bits_equal(olo[ok], d[f"{name}_olo"][ok], f"{name} lo")
        assert_bits_equal(ohi[ok], d[f"{name}_ohi"][ok], f"{name} hi")

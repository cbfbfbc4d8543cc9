"""The device Exact policy (interval.cuh) against the reference's known answers.

The engine runs IEEE directed rounding (Fast) only where its exponent guards
prove it equal to the reference's error-free-transformation rounding
(rootbox/interval.py:66-205, with the "untrusted" band |a|,|b| > 2^995 or
|a*b| < 2^-970 where the reference always steps one ulp outward); everything
else runs Exact.  These tests exercise that second path on the device:

* rb_interval_kat: every device operation, per policy, on the 36k scalar and
  16k interval operand pairs of kat_interval.npz (reference outputs, including
  2^-970 / 2^995 / subnormal / infinite operands).  Exact and guarded must equal
  the reference everywhere; Fast must differ somewhere in the untrusted band
  (otherwise the guard would be pointless) and agree everywhere else.
* rb_set_option("force_exact", 1): whole solves, filter and HS with every guard
  failing, bit-identical to the reference goldens and the oracle, with
  exact_boxes > 0 in the round statistics.
* wide_circle (coefficients 2^1000, tests/golden/make_golden.py) trips the
  guards on its own; it is one of the golden solve cases of test_gpu_parity.py.
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN, assert_bits_equal, bits, golden_jac, golden_spec, load_solve
from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kat():
    return np.load(os.path.join(GOLDEN, "kat_interval.npz"))


@pytest.fixture(scope="module")
def nat():
    from paper_1802_00330_b200 import _native
    assert _native.device_count() >= 1
    return _native


def _untrusted(a, b):
    with np.errstate(all="ignore"):
        p = a * b
    return (np.abs(a) > 2.0 ** 995) | (np.abs(b) > 2.0 ** 995) | ((np.abs(p) < 2.0 ** -970) & (a != 0) & (b != 0))


@pytest.mark.parametrize("op", ["_add_rd", "_add_ru", "_mul_rd", "_mul_ru", "_div_rd", "_div_ru"])
def test_scalar_exact_policy_equals_reference(kat, nat, op):
    a, b = kat["a"], kat["b"]
    if op.startswith("_div"):
        # the reference raises ZeroDivisionError for b == 0 (recorded as NaN); div_extended
        # never divides by an interval containing zero, so the device need not mimic it
        keep = b != 0.0
        a, b = a[keep], b[keep]
        ref = kat[op][keep]
    else:
        ref = kat[op]
    got = nat.interval_kat(op, "exact", a, a, b, b)[0]
    nan = np.isnan(ref)
    assert np.array_equal(np.isnan(got), nan), op
    # raw bits, signed zeros included: the device Exact policy is the scalar reference
    assert np.array_equal(got[~nan].view(np.uint64), ref[~nan].view(np.uint64)), op


@pytest.mark.parametrize("op", ["_mul_rd", "_mul_ru"])
def test_scalar_guarded_product_equals_reference(kat, nat, op):
    """gmul (the sweep's per-product guard) == _mul_rd/_mul_ru on every operand pair."""
    a, b = kat["a"], kat["b"]
    fin = np.isfinite(a) & np.isfinite(b)
    got = nat.interval_kat(op, "guarded", a[fin], a[fin], b[fin], b[fin])[0]
    assert_bits_equal(got, kat[op][fin], op)


@pytest.mark.parametrize("op", ["_mul_rd", "_mul_ru"])
def test_scalar_fast_differs_only_in_untrusted_band(kat, nat, op):
    a, b = kat["a"], kat["b"]
    fin = np.isfinite(a) & np.isfinite(b)
    with np.errstate(all="ignore"):
        fin &= np.isfinite(a * b)
    got = nat.interval_kat(op, "fast", a[fin], a[fin], b[fin], b[fin])[0]
    ref = kat[op][fin]
    diff = bits(got) != bits(ref)
    unt = _untrusted(a[fin], b[fin])
    assert not np.any(diff & ~unt), f"{op}: Fast differs from the reference inside the trusted band"
    assert np.any(diff & unt), f"{op}: the untrusted band never mattered (guards untested)"


def test_interval_mul_pow_recip_mid_exact(kat, nat):
    xl, xh, yl, yh = kat["xl"], kat["xh"], kat["yl"], kat["yh"]
    for pol in ("exact", "guarded"):
        lo, hi = nat.interval_kat("mul", pol, xl, xh, yl, yh)[:2]
        assert_bits_equal(lo, kat["mul_lo"], f"mul lo {pol}")
        assert_bits_equal(hi, kat["mul_hi"], f"mul hi {pol}")
    for k in range(7):
        lo, hi = nat.interval_kat(("pow", k), "exact", xl, xh)[:2]
        assert_bits_equal(lo, kat[f"pow{k}_lo"], f"pow{k} lo")
        assert_bits_equal(hi, kat[f"pow{k}_hi"], f"pow{k} hi")
    lo, hi = nat.interval_kat("recip", "exact", yl, yh)[:2]
    ok = ~np.isnan(kat["recip_lo"])
    assert_bits_equal(lo[ok], kat["recip_lo"][ok], "recip lo")
    assert_bits_equal(hi[ok], kat["recip_hi"][ok], "recip hi")
    mid = nat.interval_kat("mid", "fast", xl, xh)[0]
    ok = np.isfinite(kat["mid"])
    assert_bits_equal(mid[ok], kat["mid"][ok], "mid")


def test_fast_recip_inside_band(kat, nat):
    """The drcp-based reciprocal of the HS sweep (recip_dir) equals _div_rd/_div_ru(1, y)
    wherever the sweep uses it (2^-990 < |y| < 2^990)."""
    yl, yh = kat["yl"], kat["yh"]
    band = (~((yl <= 0) & (yh >= 0)) & np.isfinite(yl) & np.isfinite(yh) &
            (np.minimum(np.abs(yl), np.abs(yh)) > 2.0 ** -990) & (np.maximum(np.abs(yl), np.abs(yh)) < 2.0 ** 990))
    assert band.sum() > 1000
    lo, hi = nat.interval_kat("recip", "fast", yl[band], yh[band])[:2]
    assert_bits_equal(lo, kat["recip_lo"][band], "recip_dir lo")
    assert_bits_equal(hi, kat["recip_hi"][band], "recip_dir hi")


@pytest.mark.parametrize("policy", ["fast", "exact", "guarded"])
def test_div_extended_all_policies(kat, nat, policy):
    o0, o1, o2, o3, kind = nat.interval_kat("div_extended", policy, kat["xl"], kat["xh"], kat["yl"], kat["yh"])
    assert np.array_equal(kind, kat["div_kind"]), policy
    single = kind != 0
    assert_bits_equal(o0[single], kat["div_p0_lo"][single], f"p0 lo {policy}")
    assert_bits_equal(o1[single], kat["div_p0_hi"][single], f"p0 hi {policy}")
    two = kind == 2
    assert_bits_equal(o2[two], kat["div_p1_lo"][two], f"p1 lo {policy}")
    assert_bits_equal(o3[two], kat["div_p1_hi"][two], f"p1 hi {policy}")


# ------------------------------------------------------------------ force_exact: whole engine on Exact


FORCE_CASES = ["circle_line", "broyden_tri6", "katsura3", "noon3", "wide_circle", "broyden_tri4_nocontract"]


@pytest.mark.parametrize("graph", [1, 0], ids=["device_loop", "host_loop"])
@pytest.mark.parametrize("case", FORCE_CASES)
def test_force_exact_solve_vs_reference(nat, case, graph):
    from paper_1802_00330_b200 import bnb
    from test_gpu_parity import check_against_golden
    meta = load_solve(case)
    spec = golden_spec(meta["system"])
    eng = bnb.engine_for(spec)
    eng.set_option("force_exact", 1)
    eng.set_option("graph", graph)
    try:
        out = eng.solve(bnb.native_config(bnb.SolverConfig(**meta["config"])))
    finally:
        eng.set_option("force_exact", 0)
        eng.set_option("graph", 1)
    check_against_golden(case, out, meta)
    assert sum(st["exact_boxes"] for st in out["stats"]) > 0, "force_exact ran no Exact box"


@pytest.mark.parametrize("fused", [2, 0], ids=["fused_hs", "three_kernel_hs"])
@pytest.mark.parametrize("name", ["broyden_tri6", "katsura6", "brown8"])
def test_force_exact_filter_and_hs_vs_oracle(nat, name, fused):
    """rb_filter / rb_hs with every guard failing == the oracle on random cells."""
    from paper_1802_00330_b200 import bnb
    spec = golden_spec(name)
    osys = O.OSystem(spec.n, spec.eqs, golden_jac(name))
    eng = bnb.engine_for(spec)
    rng = np.random.default_rng(7)
    depth = 6
    k = rng.integers(0, 2 ** depth, (300, spec.n))
    w = (spec.init_hi - spec.init_lo) / 2 ** depth
    plo = spec.init_lo + k * w
    phi = plo + w
    eng.set_option("force_exact", 1)
    eng.set_option("hs_fused", fused)
    try:
        flo, fhi = eng.filter(plo, phi)
        hlo, hhi, hc = eng.hs(plo, phi)
    finally:
        eng.set_option("force_exact", 0)
        eng.set_option("hs_fused", 1)
    olo, ohi = osys.chunk_filter(plo, phi)
    assert_bits_equal(flo, olo, f"{name} filter lo")
    assert_bits_equal(fhi, ohi, f"{name} filter hi")
    rlo, rhi, rc = osys.hs_pass(plo, phi)
    assert_bits_equal(hlo, rlo, f"{name} hs lo")
    assert_bits_equal(hhi, rhi, f"{name} hs hi")
    assert np.array_equal(hc, rc)


def test_wide_circle_trips_the_guards(nat):
    """Coefficients of 2^1000 put every product in the untrusted band: the engine must
    take the Exact path on its own (exact_boxes > 0) and match the reference."""
    from paper_1802_00330_b200 import bnb
    from test_gpu_parity import check_against_golden
    meta = load_solve("wide_circle")
    spec = golden_spec("wide_circle")
    for graph in (1, 0):
        eng = bnb.engine_for(spec)
        eng.set_option("graph", graph)
        try:
            out = eng.solve(bnb.native_config(bnb.SolverConfig(**meta["config"])))
        finally:
            eng.set_option("graph", 1)
        check_against_golden("wide_circle", out, meta)
        assert sum(st["exact_boxes"] for st in out["stats"]) > 0

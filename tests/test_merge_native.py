"""Native backtracking merge (rb_merge, host C++) against the reference's
snap_to_grid + merge_to_width (backtrack.py:118-242), recorded in
tests/golden/merge_cases.json and in the run_pipeline reports of the solve
goldens.  Host code: runs in the CPU suite."""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, assert_bits_equal, golden_spec, load_solve, solve_cases

with open(os.path.join(GOLDEN, "merge_cases.json")) as f:
    CASES = json.load(f)


def _arr(rows, n):
    return np.array([[float.fromhex(v) for v in r] for r in rows]).reshape(-1, n)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_merge_matches_reference(case):
    from paper_1802_00330_b200.pipeline import merge_arrays
    ilo = np.array([float.fromhex(v) for v in case["init_lo"]])
    ihi = np.array([float.fromhex(v) for v in case["init_hi"]])
    n = ilo.size
    lo, hi = _arr(case["lo"], n), _arr(case["hi"], n)
    ref = case["result"]
    if "mixed" in case["name"]:  # per-component levels after locate(): documented rb_merge limit
        with pytest.raises(ValueError, match="per-component levels"):
            merge_arrays(ilo, ihi, lo, hi, np.array(case["cert"], bool), stop_width=case["stop_width"])
        return
    if "error" in ref:
        with pytest.raises(ValueError):
            merge_arrays(ilo, ihi, lo, hi, np.array(case["cert"], bool), stop_width=case["stop_width"])
        return
    mlo, mhi, mc, levels = merge_arrays(ilo, ihi, lo, hi, np.array(case["cert"], bool),
                                        stop_width=case["stop_width"])
    assert [(w.hex(), c) for w, c in levels] == [tuple(x) for x in ref["levels"]]
    assert_bits_equal(mlo, _arr(ref["lo"], n), "lo")
    assert_bits_equal(mhi, _arr(ref["hi"], n), "hi")
    assert mc.astype(int).tolist() == ref["cert"]


REPORT_CASES = [c for c in solve_cases() if "report" in load_solve(c)]


@pytest.mark.parametrize("case", REPORT_CASES)
def test_merge_reproduces_run_pipeline_reports(case):
    """roots + merge_levels of the reference's JSON report (cli.py:54-83) from the
    golden solve result, through the native merge."""
    from paper_1802_00330_b200.pipeline import merge_arrays
    meta = load_solve(case)
    rep = meta["report"]
    spec = golden_spec(meta["system"])
    n = spec.n
    if meta["status"] == "budget_exhausted" or not meta.get("lo"):
        pytest.skip("no merge in the reference pipeline for this status / empty result")
    lo, hi = _arr(meta["lo"], n), _arr(meta["hi"], n)
    mlo, mhi, mc, levels = merge_arrays(spec.init_lo, spec.init_hi, lo, hi, np.array(meta["cert"], bool))
    assert [{"width": w, "count": c} for w, c in levels] == rep["merge_levels"]
    assert [{"intervals": [[a, b] for a, b in zip(mlo[r], mhi[r])], "certified": bool(mc[r])}
            for r in range(mlo.shape[0])] == rep["roots"]


# ------------------------------------------------------------------ rb_merge_device (GPU)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_device_merge_matches_reference(case):
    """rb_merge_device == the reference's snap_to_grid + merge_to_width wherever it takes
    the device path; elsewhere it declines (RB_ERR_LIMIT) and the host merge runs."""
    from paper_1802_00330_b200.pipeline import merge_arrays
    ilo = np.array([float.fromhex(v) for v in case["init_lo"]])
    ihi = np.array([float.fromhex(v) for v in case["init_hi"]])
    n = ilo.size
    lo, hi = _arr(case["lo"], n), _arr(case["hi"], n)
    ref = case["result"]
    if "error" in ref or "mixed" in case["name"]:
        with pytest.raises(ValueError):
            merge_arrays(ilo, ihi, lo, hi, np.array(case["cert"], bool), stop_width=case["stop_width"], device=0)
        return
    mlo, mhi, mc, levels = merge_arrays(ilo, ihi, lo, hi, np.array(case["cert"], bool),
                                        stop_width=case["stop_width"], device=0)
    assert [(w.hex(), c) for w, c in levels] == [tuple(x) for x in ref["levels"]]
    assert_bits_equal(mlo, _arr(ref["lo"], n), "lo")
    assert_bits_equal(mhi, _arr(ref["hi"], n), "hi")
    assert mc.astype(int).tolist() == ref["cert"]


@pytest.mark.gpu
def test_device_merge_takes_the_fast_path_on_baseline_results():
    """Large result sets (katsura6: 263,971 boxes; brown8) merge on the device, identically
    to the host merge (pinned to the reference above)."""
    import ctypes as C
    from paper_1802_00330_b200 import SolverConfig, _native, solve_arrays
    for name, kw in (("katsura6", {}), ("brown8", {"target_width": 1e-8}), ("eco8", {})):
        spec = golden_spec(name)
        out = solve_arrays(spec, SolverConfig(**kw))
        lo, hi, cert = out["lo"], out["hi"], out["cert"]
        n, N = spec.n, lo.shape[0]
        L = _native.lib()
        olo = np.empty((N, n)); ohi = np.empty((N, n)); oc = np.empty(N, np.uint8); lv = np.empty((128, 2))
        M = C.c_int64(); K = C.c_int64(); err = C.create_string_buffer(512)
        p = _native._p
        c8 = np.ascontiguousarray(cert, np.uint8)
        rc = L.rb_merge_device(0, n, p(spec.init_lo), p(spec.init_hi), p(lo), p(hi), p(c8), N, -1.0, 1, p(olo),
                               p(ohi), p(oc), N, C.byref(M), p(lv), 128, C.byref(K), err, 512)
        assert rc == 0, (name, err.value)
        from paper_1802_00330_b200.pipeline import merge_arrays
        hlo, hhi, hc, hlev = merge_arrays(spec.init_lo, spec.init_hi, lo, hi, cert)
        assert M.value == hlo.shape[0], name
        assert_bits_equal(olo[:M.value], hlo, f"{name} lo")
        assert_bits_equal(ohi[:M.value], hhi, f"{name} hi")
        assert np.array_equal(oc[:M.value].astype(bool), hc)
        assert [(float(lv[i, 0]), int(lv[i, 1])) for i in range(K.value)] == list(hlev)

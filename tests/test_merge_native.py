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

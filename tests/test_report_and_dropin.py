"""Report writers and the drop-in path, on the CPU.

* rb_format_boxes (csrc/report.cpp) writes the raw-box sections of the
  reference's reports -- RunReport.to_json's "roots" (json.dumps(indent=2),
  cli.py:54-86) and RunReport.to_csv's rows (cli.py:88-100) -- with Python's
  float repr: checked against json.dumps / repr on adversarial doubles and on
  every golden result set.
* With the reference importable (this container only; skipped on the GPU box):
  SystemSpec.from a reference PolySystem equals the golden tables, cli.install()
  rebinds the reference's entry points, and the reference's own RunReport objects
  serialise byte-identically through the native writer.
"""
import json
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, golden_spec, golden_systems, load_solve, solve_cases

REF = "/root/reference/pkg/src"


def _adversarial(rng, m):
    v = np.concatenate([
        rng.standard_normal(m) * 10.0 ** rng.integers(-30, 30, m),
        rng.uniform(-2, 2, m),
        np.array([0.0, -0.0, 1.0, -1.0, 0.1, 1e15, 1e16, 9999999999999998.0, 1e16 - 2, 1e-4, 1e-5, 0.00011,
                  123456789012345678.0, 5e-324, -5e-324, 2.2250738585072014e-308, 1.7976931348623157e308,
                  0.5, 2.0 ** -30, 1 + 2.0 ** -52, 100.0, 1e22, 1e-7, 12345.678]),
        (rng.random(m) * 2.0 ** rng.integers(-1074, 1023, m)),
    ])
    return v[np.isfinite(v)]


def test_format_boxes_matches_python_json_and_repr():
    from paper_1802_00330_b200.pipeline import format_boxes
    rng = np.random.default_rng(5)
    v = _adversarial(rng, 2000)
    n = 3
    N = v.size // (2 * n)
    lo = v[:N * n].reshape(N, n)
    hi = v[N * n:2 * N * n].reshape(N, n)
    cert = rng.random(N) < 0.5
    got = format_boxes(lo, hi, cert, "json")
    want = json.dumps({"roots": [{"intervals": [[a, b] for a, b in zip(lo[r].tolist(), hi[r].tolist())],
                                  "certified": bool(cert[r])} for r in range(N)]}, indent=2)
    want = want[want.index("[") + 2:want.rindex("]") - 3]  # the list elements, as inside the report
    assert got == want
    csv = format_boxes(lo, hi, cert, "csv")
    want_csv = "".join(",".join([x for a, b in zip(lo[r].tolist(), hi[r].tolist()) for x in (repr(a), repr(b))]
                                + ["true" if cert[r] else "false"]) + "\n" for r in range(N))
    assert csv == want_csv


@pytest.mark.parametrize("case", [c for c in solve_cases() if "report" in load_solve(c)])
def test_native_report_json_equals_reference_report(case):
    """report_to_json on the golden result == the reference's run_pipeline JSON (cli.py),
    here for the raw (no-merge) boxes of every golden set through the native writer."""
    from paper_1802_00330_b200.bnb import Box, Interval, RootBox, RoundStats, SolveResult
    from paper_1802_00330_b200.pipeline import RunReport, config_echo, merge_arrays, report_to_csv, report_to_json
    meta = load_solve(case)
    rep = meta["report"]
    spec = golden_spec(meta["system"])
    n = spec.n
    roots = tuple(RootBox(Box(tuple(Interval(a, b) for a, b in iv)), c)
                  for iv, c in ((r["intervals"], r["certified"]) for r in rep["roots"]))
    stats = tuple(RoundStats(**st) for st in rep["rounds"])
    r = RunReport(system=rep["system"], config=rep["config"], status=rep["status"],
                  result=SolveResult(rep["status"], (), stats), roots=roots,
                  merge_levels=tuple((m["width"], m["count"]) for m in rep["merge_levels"]),
                  wall_seconds=rep["wall_seconds"])
    assert report_to_json(r) == json.dumps(rep, indent=2)
    names = golden_systems()[meta["system"]]["var_names"]
    csv = report_to_csv(r, names)
    lines = csv.split("\n")
    assert lines[0] == ",".join([f"{nm}_{s}" for nm in names for s in ("lo", "hi")] + ["certified"])
    assert len(lines) == len(roots) + 2 and lines[-1] == ""


@pytest.fixture(scope="module")
def rootbox():
    if not os.path.isdir(REF):
        pytest.skip("the reference package is not present (GPU box)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import rootbox  # noqa: F401
    return rootbox


def test_spec_from_reference_polysystem(rootbox):
    """as_spec(rootbox PolySystem) == the golden tables (PolySystem.jacobian, poly.py:284-291)."""
    from rootbox import corpus
    from paper_1802_00330_b200.system import as_spec
    for name in ("katsura6", "eco8", "noon3", "boon", "cyclic5"):
        s = corpus.load(name)
        spec = as_spec(s)
        ref = golden_spec(name)
        assert spec.n == ref.n and spec.eqs == ref.eqs and spec.jac == ref.jac, name
        assert np.array_equal(spec.init_lo, ref.init_lo) and np.array_equal(spec.init_hi, ref.init_hi)


def test_cli_install_rebinds_the_reference(rootbox):
    import rootbox.bnb
    import rootbox.cli
    from paper_1802_00330_b200 import cli, pipeline, solve
    saved = (rootbox.bnb.solve, rootbox.cli.solve, rootbox.solve, rootbox.cli.run_pipeline,
             rootbox.cli.RunReport.to_json, rootbox.cli.RunReport.to_csv)
    try:
        cli.install()
        assert rootbox.bnb.solve is solve and rootbox.cli.solve is solve and rootbox.solve is solve
        assert rootbox.cli.run_pipeline is pipeline.run_pipeline
        assert rootbox.cli.RunReport.to_json is pipeline.report_to_json
    finally:
        (rootbox.bnb.solve, rootbox.cli.solve, rootbox.solve, rootbox.cli.run_pipeline,
         rootbox.cli.RunReport.to_json, rootbox.cli.RunReport.to_csv) = saved


def test_reference_runreport_through_native_writer(rootbox):
    """The reference's own RunReport (reference Box/Interval/RootBox objects) serialises
    byte-identically with the native JSON / CSV writers."""
    from rootbox import bnb as rbnb, cli as rcli, corpus
    from rootbox.interval import Interval as RI
    from rootbox.poly import Box as RB
    from paper_1802_00330_b200.pipeline import report_to_csv, report_to_json
    meta = load_solve("noon3")
    roots = tuple(rbnb.RootBox(RB(tuple(RI(float.fromhex(a), float.fromhex(b)) for a, b in zip(lo, hi))), bool(c))
                  for lo, hi, c in zip(meta["lo"], meta["hi"], meta["cert"]))
    stats = (rbnb.RoundStats(1, 1, 8, 8, 8.0, 0.25),)
    rep = rcli.RunReport(system="noon3", config={"target_width": None}, status=meta["status"],
                         result=rbnb.SolveResult(meta["status"], roots, stats), roots=roots,
                         merge_levels=((0.5, 7),), wall_seconds=1.5)
    assert report_to_json(rep) == rep.to_json()
    s = corpus.load("noon3")
    assert report_to_csv(rep, s.var_names) == rep.to_csv(s.var_names)

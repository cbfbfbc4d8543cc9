"""Capacity-bounded rounds: parents streamed in chunks (run_round_streamed).

The reference processes a round's parents in batch_size chunks (bnb.py:271-313);
the engine does the same when a round's survivors would not fit its survivor
buffer, so a round is bounded by the frontier (max_boxes) rather than by all of
its survivors.  Forced tiny chunks (rb_set_option "stream_parents") and a small
memory budget ("mem_budget_mb", which makes the engine switch on its own) must
give bit-identical solves: the 27 reference goldens and the oracle's complete
solves of the BASELINE configs.  Also here: the max_seconds budget
(bnb.py:348-350), which no other test reaches."""
import numpy as np
import pytest

from conftest import golden_jac, golden_spec, load_solve, solve_cases
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _solve(meta_config, spec, **opts):
    from paper_1802_00330_b200 import bnb
    eng = bnb.engine_for(spec)
    for k, v in opts.items():
        eng.set_option(k, v)
    try:
        return eng.solve(bnb.native_config(bnb.SolverConfig(**meta_config)))
    finally:
        eng.set_option("stream_parents", 0)
        eng.set_option("graph", 1)
        if "mem_budget_mb" in opts:
            eng.set_option("mem_budget_mb", 0)


@pytest.mark.parametrize("chunk", [1, 3])
@pytest.mark.parametrize("case", solve_cases())
def test_streamed_rounds_vs_reference_golden(case, chunk):
    from test_gpu_parity import check_against_golden
    meta = load_solve(case)
    spec = golden_spec(meta["system"])
    out = _solve(meta["config"], spec, graph=0, stream_parents=chunk)
    check_against_golden(case, out, meta)


@pytest.mark.parametrize("name", ["katsura6", "brown8", "broyden_banded12", "eco8"])
def test_streamed_full_solves_vs_oracle(name):
    """Chunks of 4096 parents: 16M-child rounds run as thousands of chunks."""
    from test_full_solves import check_full, load_full
    meta = load_full(name)
    spec = golden_spec(meta["system"])
    out = _solve(meta["config"], spec, graph=0, stream_parents=4096)
    check_full(name, out, meta)


@pytest.mark.parametrize("name", ["katsura6", "brown8"])
def test_small_memory_budget_streams_on_its_own(name):
    """A 64 MB budget caps the survivor buffer far below katsura6 round 5's 1.28M
    survivors: the engine must stream those rounds by itself, with identical results."""
    from test_full_solves import check_full, load_full
    meta = load_full(name)
    spec = golden_spec(meta["system"])
    out = _solve(meta["config"], spec, graph=0, mem_budget_mb=64)
    check_full(name, out, meta)


def test_max_seconds_budget():
    """max_seconds (bnb.py:348-350): an elapsed-time budget below one round stops the
    solve after round 1 as budget_exhausted with round 1's frontier."""
    from paper_1802_00330_b200 import SolverConfig, solve_arrays
    spec = golden_spec("katsura6")
    out = solve_arrays(spec, SolverConfig(max_seconds=1e-9))
    ref = O.OSystem(spec.n, spec.eqs, golden_jac("katsura6")).solve(spec.init_lo, spec.init_hi, max_rounds=1)
    assert out["status"] == "budget_exhausted" == ref["status"]
    assert len(out["stats"]) == 1
    assert out["lo"].shape[0] == ref["lo"].shape[0] == int(ref["stats"][0, 3])
    keys = tuple(ref["hi"][:, i] for i in reversed(range(spec.n))) + tuple(ref["lo"][:, i] for i in reversed(range(spec.n)))
    o = np.lexsort(keys)
    assert np.array_equal(out["lo"], ref["lo"][o]) and np.array_equal(out["hi"], ref["hi"][o])
    # a generous budget changes nothing
    full = solve_arrays(spec, SolverConfig(max_seconds=3600.0, max_rounds=3))
    meta = load_solve("katsura6_r3")
    assert full["status"] == meta["status"] and [s["boxes_after_hs"] for s in full["stats"]] == \
        [w[3] for w in meta["stats"]]

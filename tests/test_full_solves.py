"""BASELINE configs 3-5 solved to completion on the device, against the oracle.

The Python reference cannot finish katsura6 / eco8 / brown8 / broyden-banded-12
(BASELINE.md §2), so their complete solves are pinned by the oracle
(oracle/rootbox_oracle.c, itself pinned bit-exact against the reference by
tests/golden/make_golden.py, including the first rounds of these same configs).
tests/golden/make_oracle_full.py recorded per-round statistics and a SHA-256 of
the canonical final set (rows + flags) in tests/golden/full_<config>.json.

Each config is solved with the device round loop (CUDA graph) and with
host-driven rounds (which run the throughput kernels k_filter and
k_hs_eval/lin/sweep at full scale, e.g. katsura6 round 5: 1.28M HS boxes,
eco8 round 5: 513M children), and checked for identical per-round
statistics, identical final rows and flags, and enclosure of every known real
root (tests/golden/roots.json)."""
import hashlib
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, bits, canonical_sort, golden_spec

pytestmark = pytest.mark.gpu

FULL = sorted(fn[5:-5] for fn in os.listdir(GOLDEN) if fn.startswith("full_") and fn.endswith(".json"))


def load_full(name):
    with open(os.path.join(GOLDEN, f"full_{name}.json")) as f:
        return json.load(f)


def digest(lo, hi, cert, uns):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(np.where(lo == 0.0, 0.0, lo), "<f8").tobytes())
    h.update(np.ascontiguousarray(np.where(hi == 0.0, 0.0, hi), "<f8").tobytes())
    h.update(np.ascontiguousarray(cert, np.uint8).tobytes())
    h.update(np.ascontiguousarray(uns, np.uint8).tobytes())
    return h.hexdigest()


def check_full(name, out, meta):
    assert out["status"] == meta["status"], name
    assert len(out["stats"]) == len(meta["rounds"]), (name, len(out["stats"]))
    for st, want in zip(out["stats"], meta["rounds"]):
        got = [st["round"], st["boxes_in"], st["boxes_after_filter"], st["boxes_after_hs"]]
        assert got == want[:4], (name, got, want)
        assert bits(st["width"]) == bits(float.fromhex(want[4])), (name, st["round"])
        assert st["children"] == want[5] and st["hs_calls"] == want[6], (name, st["round"])
        assert st["dups"] == want[7], (name, st["round"])
    lo, hi = out["lo"], out["hi"]
    assert lo.shape[0] == meta["nboxes"]
    assert int(out["cert"].sum()) == meta["ncert"] and int(out["unsplit"].sum()) == meta["nunsplit"]
    assert np.array_equal(canonical_sort(lo, hi), np.arange(lo.shape[0]))
    if "lo" in meta:
        want = np.array([[float.fromhex(v) for v in r] for r in meta["lo"]]).reshape(lo.shape)
        assert np.array_equal(bits(lo), bits(want)), name
    else:
        for i, r in enumerate(meta["sample_rows"]):
            assert [v.hex() for v in lo[r]] == meta["sample_lo"][i], (name, r)
            assert [v.hex() for v in hi[r]] == meta["sample_hi"][i], (name, r)
    assert digest(lo, hi, out["cert"], out["unsplit"]) == meta["digest"], name
    assert not np.any(np.signbit(lo) & (lo == 0)) and not np.any(np.signbit(hi) & (hi == 0))


def roots_of(system):
    with open(os.path.join(GOLDEN, "roots.json")) as f:
        r = json.load(f)["systems"].get(system)
    if r is None:
        return None
    rd = np.array([[float.fromhex(v) for v in row] for row in r["roots_rd"]]).reshape(-1, r["n"])
    ru = np.array([[float.fromhex(v) for v in row] for row in r["roots_ru"]]).reshape(-1, r["n"])
    return rd, ru


def enclosing(lo, hi, rd, ru):
    """boxes (row indices) containing the root r with RD(r) = rd, RU(r) = ru:
    lo <= r <= hi  <=>  lo <= rd and ru <= hi for double endpoints."""
    return np.nonzero(np.all(lo <= rd, axis=1) & np.all(ru <= hi, axis=1))[0]


def check_enclosure(system, lo, hi):
    roots = roots_of(system)
    assert roots is not None, system
    rd, ru = roots
    for k in range(rd.shape[0]):
        assert enclosing(lo, hi, rd[k], ru[k]).size >= 1, f"{system}: known root {k} not enclosed"
    return rd.shape[0]


@pytest.mark.parametrize("graph", [1, 0], ids=["device_loop", "host_loop"])
@pytest.mark.parametrize("name", FULL)
def test_full_solve_vs_oracle(name, graph):
    from paper_1802_00330_b200 import bnb
    meta = load_full(name)
    spec = golden_spec(meta["system"])
    eng = bnb.engine_for(spec)
    eng.set_option("graph", graph)
    try:
        out = eng.solve(bnb.native_config(bnb.SolverConfig(**meta["config"])))
    finally:
        eng.set_option("graph", 1)
    check_full(name, out, meta)
    check_enclosure(meta["system"], out["lo"], out["hi"])


@pytest.mark.parametrize("name", FULL)
def test_full_solve_three_kernel_hs_tables(name):
    """The table (non-specialised) kernels and the three-kernel HS for every batch."""
    from paper_1802_00330_b200 import bnb
    meta = load_full(name)
    spec = golden_spec(meta["system"])
    eng = bnb.engine_for(spec)
    eng.set_option("codegen", 0)
    eng.set_option("hs_fused", 0)
    eng.set_option("graph", 0)
    try:
        out = eng.solve(bnb.native_config(bnb.SolverConfig(**meta["config"])))
    finally:
        eng.set_option("codegen", 1)
        eng.set_option("hs_fused", 1)
        eng.set_option("graph", 1)
    check_full(name, out, meta)

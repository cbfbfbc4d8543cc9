"""Known-root enclosure (north_star: "both runs must enclose every known real root").

tests/golden/roots.json holds the real roots of the benchmark and golden systems,
found independently of any interval code (random-start Newton refined to 256 bits,
tests/golden/make_roots.py; the reference's own soundness/completeness oracles,
SPEC.md:616-617).  Each root r is stored as the doubles RD(r) <= r <= RU(r), so
"box contains r" is an exact float64 test.

CPU part (this file): the reference's recorded result sets (solve_*.json) and the
oracle's complete solves of BASELINE configs 3-5 (full_*.json, rows stored up to
4096) enclose every known root, and every certified box contains exactly one.  The
engine's result sets are bit-identical to these (test_gpu_parity.py,
test_full_solves.py), and test_full_solves.py also checks enclosure directly on
the device results, including katsura6 (263,971 boxes, digest-only fixture).
"""
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

with open(os.path.join(GOLDEN, "roots.json")) as f:
    ROOTS = json.load(f)["systems"]


def _rows(meta):
    n = ROOTS[meta["system"]]["n"]
    lo = np.array([[float.fromhex(v) for v in r] for r in meta["lo"]]).reshape(meta["nboxes"], n)
    hi = np.array([[float.fromhex(v) for v in r] for r in meta["hi"]]).reshape(meta["nboxes"], n)
    return lo, hi, np.array(meta["cert"], bool)


def _roots(system):
    r = ROOTS[system]
    rd = np.array([[float.fromhex(v) for v in row] for row in r["roots_rd"]]).reshape(-1, r["n"])
    ru = np.array([[float.fromhex(v) for v in row] for row in r["roots_ru"]]).reshape(-1, r["n"])
    return rd, ru


def _results():
    out = []
    for fn in sorted(os.listdir(GOLDEN)):
        if (fn.startswith("solve_") or fn.startswith("full_")) and fn.endswith(".json"):
            with open(os.path.join(GOLDEN, fn)) as f:
                meta = json.load(f)
            if "lo" in meta and meta["system"] in ROOTS:
                out.append(pytest.param(meta, id=fn[:-5]))
    return out


def test_roots_fixture_is_sane():
    assert ROOTS["circle_line"]["roots_rd"] and len(ROOTS["circle_line"]["roots_rd"]) == 2
    assert len(ROOTS["brown8"]["roots_rd"]) == 2  # (1,...,1) and (0.96769..., 1.25848...)
    assert len(ROOTS["conform1"]["roots_rd"]) == 0  # no real solutions (manifest)
    for name, r in ROOTS.items():
        rd, ru = _roots(name)
        assert np.all(rd <= ru), name
        assert np.all(np.nextafter(rd, np.inf) >= ru), name  # adjacent doubles


@pytest.mark.parametrize("meta", _results())
def test_result_set_encloses_every_known_root(meta):
    """Every solve result (complete or budget-capped) keeps every real root: B&B
    discards only boxes proven root-free."""
    lo, hi, cert = _rows(meta)
    rd, ru = _roots(meta["system"])
    if meta["status"] == "no_real_solution":
        assert rd.shape[0] == 0
        return
    for k in range(rd.shape[0]):
        inside = np.all(lo <= rd[k], axis=1) & np.all(ru[k] <= hi, axis=1)
        assert inside.any(), f"{meta['case']}: root {ROOTS[meta['system']]['roots_dec'][k]} not enclosed"


@pytest.mark.parametrize("meta", _results())
def test_certified_boxes_hold_exactly_one_known_root(meta):
    """HS certification (existence + uniqueness, hansen.py:129-138): a certified box
    contains exactly one root, and the root list must contain it."""
    lo, hi, cert = _rows(meta)
    rd, ru = _roots(meta["system"])
    for b in np.nonzero(cert)[0]:
        inside = np.all(lo[b] <= rd, axis=1) & np.all(ru <= hi[b], axis=1)
        assert inside.sum() == 1, f"{meta['case']}: certified box {b} holds {inside.sum()} known roots"

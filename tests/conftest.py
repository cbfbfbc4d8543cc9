import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


_SYSTEMS = None


def golden_systems():
    global _SYSTEMS
    if _SYSTEMS is None:
        with open(os.path.join(GOLDEN, "systems.json")) as f:
            _SYSTEMS = json.load(f)["systems"]
    return _SYSTEMS


def golden_spec(name):
    from paper_1802_00330_b200.system import SystemSpec
    return SystemSpec.from_json(golden_systems()[name], name=name)


def golden_jac(name):
    d = golden_systems()[name]
    return [[[(float.fromhex(c), tuple(e)) for c, e in q] for q in row] for row in d["jac"]]


def load_solve(case):
    with open(os.path.join(GOLDEN, f"solve_{case}.json")) as f:
        return json.load(f)


def solve_cases():
    return sorted(fn[6:-5] for fn in os.listdir(GOLDEN) if fn.startswith("solve_") and fn.endswith(".json"))


def bits(a):
    """float64 bit patterns with -0.0 canonicalised to +0.0 and NaNs unified."""
    a = np.asarray(a, dtype=np.float64)
    a = np.where(a == 0.0, 0.0, a)
    a = np.where(np.isnan(a), np.nan, a)
    return a.view(np.uint64)


def raw_bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def assert_bits_equal(a, b, what=""):
    ba, bb = bits(a), bits(b)
    if not np.array_equal(ba, bb):
        bad = np.nonzero(ba.ravel() != bb.ravel())[0]
        i = bad[0]
        raise AssertionError(f"{what}: {bad.size} mismatches; first at {i}: "
                             f"{np.asarray(a).ravel()[i]!r} vs {np.asarray(b).ravel()[i]!r}")


def canonical_sort(lo, hi):
    n = lo.shape[1]
    keys = tuple(hi[:, i] for i in reversed(range(n))) + tuple(lo[:, i] for i in reversed(range(n)))
    return np.lexsort(keys) if lo.shape[0] else np.zeros(0, dtype=np.int64)


@pytest.fixture(scope="session")
def systems():
    return golden_systems()

"""Lazy SolveResult.boxes (RootBoxes) behaves like the reference's tuple."""
import numpy as np

from paper_1802_00330_b200.bnb import Box, Interval, RootBox, RootBoxes


def _mk(n=5, d=3):
    rng = np.random.default_rng(1)
    lo = rng.uniform(-1, 0, (n, d)); hi = lo + rng.uniform(0, 1, (n, d))
    c = rng.random(n) < 0.5; u = rng.random(n) < 0.5
    return lo, hi, c, u


def test_rootboxes_sequence_semantics():
    lo, hi, c, u = _mk()
    rb = RootBoxes(lo, hi, c, u, (RootBox, Box, Interval))
    eager = tuple(RootBox(Box(tuple(Interval(a, b) for a, b in zip(lo[r], hi[r]))), bool(c[r]), bool(u[r]))
                  for r in range(len(lo)))
    assert len(rb) == 5 and bool(rb)
    assert rb == eager and list(rb) == list(eager)
    assert rb[0] == eager[0] and rb[-1] == eager[-1] and rb[1:3] == eager[1:3]
    assert rb[2].box[1].lo == lo[2, 1] and rb[2].certified == bool(c[2])
    empty = RootBoxes(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0, bool), np.zeros(0, bool),
                      (RootBox, Box, Interval))
    assert not empty and len(empty) == 0 and empty == ()


def test_rootboxes_hash_and_concat():
    """A frozen SolveResult holding RootBoxes is hashable like the tuple it equals."""
    from paper_1802_00330_b200.bnb import SolveResult
    lo, hi, c, u = _mk()
    rb = RootBoxes(lo, hi, c, u, (RootBox, Box, Interval))
    eager = tuple(rb)
    assert hash(rb) == hash(eager)
    assert hash(SolveResult("width_reached", rb, ())) == hash(SolveResult("width_reached", eager, ()))
    assert rb + () == eager and () + rb == eager and rb + rb == eager + eager

"""Krawczyk operator on the B200 engine (hansen.krawczyk, hansen.py:141-170).

``krawczyk(s, jac, b)`` keeps the reference signature and return convention
(``Box`` or ``None``; ``ValueError`` on an unbounded box).  ``krawczyk_arrays``
is the batched form: M boxes in one call, row-major ``(M, n)`` lo/hi.  Both
run ``rb_krawczyk``: the HS preconditioning kernels (x = mid X, J(X), F(x),
Gauss-Jordan A, M = A J, g = A F(x)) followed by one thread per box for
K(X) intersected with X.

The Jacobian is the engine's own symbolic derivative of ``s``, which is
bit-identical to ``PolySystem.jacobian`` (tests/test_oracle_golden.py); the
``jac`` argument is accepted for signature compatibility.
"""
from __future__ import annotations

import numpy as np

from .bnb import Box, Interval, engine_for
from .system import as_spec

__all__ = ["krawczyk", "krawczyk_arrays"]


def krawczyk_arrays(s, lo, hi, device: int | None = None):
    """Batched Krawczyk: returns (ok[M] bool, olo[M, n], ohi[M, n]); rows with
    ok False (the reference's None) are NaN."""
    spec = as_spec(s)
    lo = np.ascontiguousarray(lo, np.float64).reshape(-1, spec.n)
    hi = np.ascontiguousarray(hi, np.float64).reshape(-1, spec.n)
    return engine_for(spec, device).krawczyk(lo, hi)


def krawczyk(s, jac, b):
    """K(X) intersected with X for one box, or None (hansen.py:141-170)."""
    del jac  # the engine differentiates s itself (bit-identical to PolySystem.jacobian)
    ivs = tuple(b)
    if not all(np.isfinite(iv.lo) and np.isfinite(iv.hi) for iv in ivs):
        raise ValueError("box must be bounded")
    lo = np.array([[iv.lo for iv in ivs]])
    hi = np.array([[iv.hi for iv in ivs]])
    ok, olo, ohi = krawczyk_arrays(s, lo, hi)
    if not ok[0]:
        return None
    if type(b).__module__.startswith("rootbox"):
        BX, IV = type(b), type(ivs[0])
    else:
        BX, IV = Box, Interval
    return BX(tuple(IV(a, c) for a, c in zip(olo[0].tolist(), ohi[0].tolist())))

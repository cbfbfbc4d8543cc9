"""Host-side polynomial-system model and the flat device tables.

This is the B200 engine's view of the reference's ``PolySystem``
(rootbox/poly.py:258-291) and of ``compile_system`` (rootbox/_batch.py:144-164).
A system is accepted from any object shaped like the reference's
``PolySystem`` (duck-typed: ``.polynomials[i].monomials[t].coeff/.exps``,
``.initial_box`` iterable of intervals with ``.lo/.hi``, ``.var_names``,
``.name``), or from the JSON form written by tests/golden/make_golden.py.

Canonical monomial order is the reference's: descending by
``(total degree, exponent tuple)`` (poly.py:72-73, 159).  The Jacobian is the
exact symbolic derivative with coefficient ``float(Fraction(c) * e)``
(poly.py:209-221) -- a single correctly rounded product, i.e. ``c * e`` in
binary64 -- re-sorted canonically, zero polynomials kept as empty term lists
(PolySystem.jacobian, poly.py:284-291).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import weakref

import numpy as np

Term = tuple  # (coeff: float, exps: tuple[int, ...])


def canonical(terms, n):
    """Combine (coeff, exps) pairs into canonical order, dropping zeros (poly.py:147-161)."""
    combined = {}
    for c, e in terms:
        e = tuple(int(v) for v in e)
        if len(e) != n:
            raise ValueError(f"monomial arity {len(e)} != dimension {n}")
        if float(c) == 0.0:
            continue
        if e in combined:
            raise ValueError(f"duplicate exponent vector {e}")
        combined[e] = float(c)
    order = sorted(combined, key=lambda e: (sum(e), e), reverse=True)
    return [(combined[e], e) for e in order]


def differentiate(terms, n, j):
    """d/dx_j of a canonical term list (poly.py:209-221)."""
    out = []
    for c, e in terms:
        k = e[j]
        if k == 0:
            continue
        ee = list(e)
        ee[j] = k - 1
        out.append((c * k, tuple(ee)))  # float(Fraction(c) * k) == RN(c * k)
    return canonical(out, n)


@dataclass
class SystemSpec:
    n: int
    eqs: list            # n canonical term lists
    init_lo: np.ndarray  # (n,) float64
    init_hi: np.ndarray
    var_names: tuple = ()
    name: str = ""
    jac: list = field(default=None)  # n x n canonical term lists

    def __post_init__(self):
        if len(self.eqs) != self.n:
            raise ValueError(f"{len(self.eqs)} equations for {self.n} variables")
        self.init_lo = np.asarray(self.init_lo, dtype=np.float64).reshape(self.n)
        self.init_hi = np.asarray(self.init_hi, dtype=np.float64).reshape(self.n)
        if not np.all(np.isfinite(self.init_lo)) or not np.all(np.isfinite(self.init_hi)):
            raise ValueError("initial box must be bounded")
        if np.any(self.init_lo > self.init_hi):
            raise ValueError("initial box has lo > hi")
        if not self.var_names:
            self.var_names = tuple(f"x{i + 1}" for i in range(self.n))
        if self.jac is None:
            self.jac = [[differentiate(p, self.n, j) for j in range(self.n)] for p in self.eqs]

    # -- constructors --------------------------------------------------------
    @classmethod
    def from_polysystem(cls, s) -> "SystemSpec":
        """Duck-typed adapter for rootbox.poly.PolySystem (poly.py:258-291)."""
        n = len(s.var_names)
        eqs = [[(float(m.coeff), tuple(m.exps)) for m in p.monomials] for p in s.polynomials]
        lo = [float(iv.lo) for iv in s.initial_box]
        hi = [float(iv.hi) for iv in s.initial_box]
        return cls(n=n, eqs=eqs, init_lo=np.array(lo), init_hi=np.array(hi),
                   var_names=tuple(s.var_names), name=getattr(s, "name", "") or "")

    @classmethod
    def from_json(cls, d, name="") -> "SystemSpec":
        n = int(d["n"])
        eqs = [[(float.fromhex(c), tuple(e)) for c, e in p] for p in d["eqs"]]
        return cls(n=n, eqs=eqs,
                   init_lo=np.array([float.fromhex(v) for v in d["init_lo"]]),
                   init_hi=np.array([float.fromhex(v) for v in d["init_hi"]]),
                   var_names=tuple(d.get("var_names", ())), name=name)

    @classmethod
    def from_terms(cls, eqs, init_lo, init_hi, var_names=(), name="") -> "SystemSpec":
        """Build from raw (coeff, exps) lists in any order (canonicalised here)."""
        n = len(eqs)
        return cls(n=n, eqs=[canonical(p, n) for p in eqs], init_lo=np.asarray(init_lo, float),
                   init_hi=np.asarray(init_hi, float), var_names=tuple(var_names), name=name)

    # -- algorithmic work per unit ------------------------------
    def ops_poly(self, terms) -> int:
        """Minimal directed-op count of one interval evaluation: per term
        2*nfac (interval products) + 2(e-1) per power + 2 (the accumulate)."""
        ops = 0
        for _c, e in terms:
            nf = sum(1 for v in e if v)
            ops += 2 * nf + sum(2 * (v - 1) for v in e if v >= 2) + 2
        return ops

    def ops_eqs(self):
        return [self.ops_poly(p) for p in self.eqs]

    def ops_hs(self) -> int:
        """ops_HS = ops_J + 2n^2 + ops_GJ + 2n + ops_F + 4n^2 + 4n^3 + n(6(n-1)+8)."""
        n = self.n
        ops_j = sum(self.ops_poly(q) for row in self.jac for q in row)
        ops_gj = sum((2 * n - k) + 1 + 2 * (n - 1) * (2 * n - k) for k in range(n))
        ops_f = sum(self.ops_eqs())
        return ops_j + 2 * n * n + ops_gj + 2 * n + ops_f + 4 * n * n + 4 * n ** 3 + n * (6 * (n - 1) + 8)


# -- flat tables handed to the C-ABI (rb_system in include/rootbox_b200.h) -------

@dataclass
class FlatTables:
    n: int
    poly_off: np.ndarray   # int32 (n + n*n + 1): term ranges, F polys then J[i][j] row-major
    coeff: np.ndarray      # float64 (T,)
    fac_off: np.ndarray    # int32 (T + 1): factor ranges per term
    fac_var: np.ndarray    # uint8 (Fc,) ascending variable index within a term (_batch.py:161)
    fac_exp: np.ndarray    # uint8 (Fc,) exponent >= 1
    init_lo: np.ndarray
    init_hi: np.ndarray


def compile_tables(spec: SystemSpec) -> FlatTables:
    """compile_system (_batch.py:156-164) for F and J: per term the coefficient
    and its nonzero (var, exp) factors in ascending variable order.  Cached on the
    spec (keyed by the identity of its term lists and the initial box bytes)."""
    fp = (id(spec.eqs), id(spec.jac), spec.init_lo.tobytes(), spec.init_hi.tobytes())
    cached = spec.__dict__.get("_flat_cache")
    if cached is not None and cached[0] == fp:
        return cached[1]
    t = _compile_tables(spec)
    spec.__dict__["_flat_cache"] = (fp, t)
    return t


def _compile_tables(spec: SystemSpec) -> FlatTables:
    n = spec.n
    polys = list(spec.eqs) + [spec.jac[i][j] for i in range(n) for j in range(n)]
    poly_off = [0]
    coeff, fac_off, fac_var, fac_exp = [], [0], [], []
    for p in polys:
        for c, e in p:
            coeff.append(c)
            for j, k in enumerate(e):
                if k:
                    if k > 255:
                        raise ValueError("exponent > 255 not supported")
                    fac_var.append(j)
                    fac_exp.append(k)
            fac_off.append(len(fac_var))
        poly_off.append(len(coeff))
    return FlatTables(
        n=n,
        poly_off=np.array(poly_off, dtype=np.int32),
        coeff=np.array(coeff, dtype=np.float64),
        fac_off=np.array(fac_off, dtype=np.int32),
        fac_var=np.array(fac_var, dtype=np.uint8),
        fac_exp=np.array(fac_exp, dtype=np.uint8),
        init_lo=np.ascontiguousarray(spec.init_lo, dtype=np.float64),
        init_hi=np.ascontiguousarray(spec.init_hi, dtype=np.float64),
    )


_SPEC_CACHE: dict = {}  # id(PolySystem) -> (weakref, SystemSpec): solve() on the same system converts once


def as_spec(s) -> SystemSpec:
    if isinstance(s, SystemSpec):
        return s
    if hasattr(s, "polynomials") and hasattr(s, "initial_box"):
        hit = _SPEC_CACHE.get(id(s))
        if hit is not None and hit[0]() is s:
            return hit[1]
        spec = SystemSpec.from_polysystem(s)
        try:
            ref = weakref.ref(s, lambda _r, k=id(s): _SPEC_CACHE.pop(k, None))
        except TypeError:  # not weak-referenceable: no caching
            return spec
        _SPEC_CACHE[id(s)] = (ref, spec)
        return spec
    raise TypeError(f"cannot interpret {type(s).__name__} as a polynomial system")

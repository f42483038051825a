"""Host-side exact stencil algebra (the part `north_star` keeps on the host).

A Python mirror of the reference's L1 layer so tests, smoke() and bench.py
can produce composed weights without the C++ reference:
  Stencil / scale / add / shift / compose / outer_product / weight_sum
      (stencil.hpp:19-58, stencil.cpp:15-107)
  make / laplacian / solve_rational (generators.cpp:7-108)
Exact `fractions.Fraction` arithmetic; `to_double` truncates toward zero like
GMP's mpq_get_d behind `Rational::to_double` (rational.hpp:32), so the doubles
handed to the device equal the reference's. Offsets are tuples; entries are
kept in lexicographic order (std::map<Offset, Rational> order).
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction
from typing import Dict, Iterable, List, Sequence, Tuple

from .errors import Errc, StencilkitError

Offset = Tuple[int, ...]


def to_double(q: Fraction) -> float:
    """mpq_get_d semantics: the double nearest q in the direction of zero."""
    d = float(q)
    if Fraction(d) != q and abs(Fraction(d)) > abs(q):
        d = math.nextafter(d, 0.0)
    return d


class Stencil:
    """Canonical stencil: offset -> exact coefficient, h exponent (stencil.hpp:19-42)."""

    __slots__ = ("dim", "h_power", "entries")

    def __init__(self, dim: int, h_power: int, entries: Dict[Offset, Fraction]):
        if dim < 1:
            raise StencilkitError(Errc.invalid_argument, "stencil dimension must be >= 1")
        clean: Dict[Offset, Fraction] = {}
        for off, c in entries.items():
            off = tuple(int(o) for o in off)
            if len(off) != dim:
                raise StencilkitError(Errc.dim_mismatch, "offset length does not match stencil dimension")
            c = Fraction(c)
            if c != 0:
                clean[off] = c
        if not clean:
            raise StencilkitError(Errc.empty_stencil,
                                  "all coefficients cancelled; empty stencil is not representable")
        self.dim = dim
        self.h_power = int(h_power)
        self.entries = dict(sorted(clean.items()))

    @staticmethod
    def identity(dim: int) -> "Stencil":
        return Stencil(dim, 0, {(0,) * dim: Fraction(1)})

    def support(self, axis: int) -> Tuple[int, int]:
        if axis < 0 or axis >= self.dim:
            raise StencilkitError(Errc.invalid_argument, "axis out of range")
        vals = [o[axis] for o in self.entries]
        return min(vals), max(vals)

    def __eq__(self, other) -> bool:
        return (isinstance(other, Stencil) and self.dim == other.dim and self.h_power == other.h_power
                and self.entries == other.entries)

    def __repr__(self) -> str:
        return f"Stencil(dim={self.dim}, h_power={self.h_power}, {len(self.entries)} entries)"

    # flat arrays for the C-ABI: offsets (entry-major), to_double coefficients
    def flat(self) -> Tuple[List[int], List[float]]:
        offs: List[int] = []
        coeffs: List[float] = []
        for off, c in self.entries.items():
            offs.extend(off)
            coeffs.append(to_double(c))
        return offs, coeffs


def scale(s: Stencil, c) -> Stencil:
    c = Fraction(c)
    if c == 0:
        raise StencilkitError(Errc.zero_scale, "scaling a stencil by zero")
    return Stencil(s.dim, s.h_power, {o: v * c for o, v in s.entries.items()})


def add(a: Stencil, b: Stencil) -> Stencil:
    if a.dim != b.dim:
        raise StencilkitError(Errc.dim_mismatch, "adding stencils of different dimension")
    if a.h_power != b.h_power:
        raise StencilkitError(Errc.power_mismatch, "adding stencils of different h power")
    out = dict(a.entries)
    for o, v in b.entries.items():
        out[o] = out.get(o, Fraction(0)) + v
    return Stencil(a.dim, a.h_power, out)


def shift(s: Stencil, o: Sequence[int]) -> Stencil:
    if len(o) != s.dim:
        raise StencilkitError(Errc.dim_mismatch, "shift offset length does not match stencil dimension")
    return Stencil(s.dim, s.h_power, {tuple(a + b for a, b in zip(off, o)): v for off, v in s.entries.items()})


def compose(inner: Stencil, outer: Stencil) -> Stencil:
    """Offsets add, coefficients multiply, h exponents add (stencil.cpp:75-87)."""
    if inner.dim != outer.dim:
        raise StencilkitError(Errc.dim_mismatch, "composing stencils of different dimension")
    out: Dict[Offset, Fraction] = {}
    for u, a in inner.entries.items():
        for v, b in outer.entries.items():
            w = tuple(x + y for x, y in zip(u, v))
            out[w] = out.get(w, Fraction(0)) + a * b
    return Stencil(inner.dim, inner.h_power + outer.h_power, out)


def outer_product(sx: Stencil, sy: Stencil) -> Stencil:
    out: Dict[Offset, Fraction] = {}
    for u, a in sx.entries.items():
        for v, b in sy.entries.items():
            w = tuple(u) + tuple(v)
            out[w] = out.get(w, Fraction(0)) + a * b
    return Stencil(sx.dim + sy.dim, sx.h_power + sy.h_power, out)


def weight_sum(s: Stencil) -> Fraction:
    return sum(s.entries.values(), Fraction(0))


def solve_rational(m: List[List[Fraction]], rhs: List[Fraction]) -> List[Fraction]:
    """Exact full-pivot elimination (generators.cpp:7-46)."""
    n = len(m)
    if len(rhs) != n:
        raise StencilkitError(Errc.shape_mismatch, "matrix/rhs size mismatch")
    m = [list(map(Fraction, row)) for row in m]
    rhs = list(map(Fraction, rhs))
    col_of = list(range(n))
    for k in range(n):
        pr = pc = n
        for i in range(k, n):
            for j in range(k, n):
                if m[i][j] != 0:
                    pr, pc = i, j
                    break
            if pr != n:
                break
        if pr == n:
            raise StencilkitError(Errc.singular_system, "exact elimination hit a zero block")
        m[k], m[pr] = m[pr], m[k]
        rhs[k], rhs[pr] = rhs[pr], rhs[k]
        if pc != k:
            for i in range(n):
                m[i][k], m[i][pc] = m[i][pc], m[i][k]
            col_of[k], col_of[pc] = col_of[pc], col_of[k]
        for i in range(k + 1, n):
            if m[i][k] == 0:
                continue
            f = m[i][k] / m[k][k]
            for j in range(k, n):
                m[i][j] -= f * m[k][j]
            rhs[i] -= f * rhs[k]
    y = [Fraction(0)] * n
    for k in range(n - 1, -1, -1):
        s = rhs[k]
        for j in range(k + 1, n):
            s -= m[k][j] * y[j]
        y[k] = s / m[k][k]
    x = [Fraction(0)] * n
    for k in range(n):
        x[col_of[k]] = y[k]
    return x


@dataclass(frozen=True)
class StencilSpec:
    derivative: int = 1
    accuracy: int = 2
    style: str = "centered"  # centered | forward | backward


def make(spec: StencilSpec) -> Stencil:
    """Moment conditions sum_i a_i u_i^alpha / alpha! = delta_{alpha p} (generators.cpp:50-92)."""
    p, q = spec.derivative, spec.accuracy
    if p < 1:
        raise StencilkitError(Errc.invalid_argument, "derivative order must be >= 1")
    if q < 1:
        raise StencilkitError(Errc.invalid_argument, "accuracy must be >= 1")
    if spec.style == "centered":
        q_eff = q + (q % 2)
        m = (p + 1) // 2 + q_eff // 2 - 1
        points = list(range(-m, m + 1))
    elif spec.style == "forward":
        points = list(range(0, p + q))
    elif spec.style == "backward":
        points = list(range(-(p + q - 1), 1))
    else:
        raise StencilkitError(Errc.invalid_argument, f"unknown stencil style '{spec.style}'")
    if len(points) <= p:
        raise StencilkitError(Errc.invalid_argument, "support too small for the requested derivative")
    n = len(points)
    mat = [[Fraction(pt) ** a / math.factorial(a) for pt in points] for a in range(n)]
    rhs = [Fraction(1) if a == p else Fraction(0) for a in range(n)]
    w = solve_rational(mat, rhs)
    return Stencil(1, -p, {(points[i],): w[i] for i in range(n) if w[i] != 0})


def laplacian(dim: int, accuracy: int) -> Stencil:
    """Sum of per-axis second-derivative stencils (generators.cpp:94-108)."""
    if dim < 1 or dim > 3:
        raise StencilkitError(Errc.invalid_argument, "laplacian supports d in {1,2,3}")
    if accuracy < 2 or accuracy % 2 != 0 or accuracy > 8:
        raise StencilkitError(Errc.unsupported_accuracy, "laplacian accuracy must be even, 2..8")
    base = make(StencilSpec(2, accuracy, "centered"))
    out: Dict[Offset, Fraction] = {}
    for axis in range(dim):
        for (o,), c in base.entries.items():
            off = [0] * dim
            off[axis] = o
            t = tuple(off)
            out[t] = out.get(t, Fraction(0)) + c
    return Stencil(dim, -2, out)


def bilaplacian(dim: int, accuracy: int = 2) -> Stencil:
    """compose(laplacian, laplacian): 13-point (2D), 25-point (3D), 73-point (3D, accuracy 4)."""
    lap = laplacian(dim, accuracy)
    return compose(lap, lap)


def builtin_stencil(name: str) -> Stencil:
    """The hot-path subset of io.cpp:139-167."""
    d1 = make(StencilSpec(1, 2))
    table = {
        "d1": lambda: d1,
        "d2": lambda: make(StencilSpec(2, 2)),
        "wide-heat": lambda: compose(d1, d1),
        "dxx-dxx": lambda: compose(make(StencilSpec(2, 2)), make(StencilSpec(2, 2))),
        "laplacian-1d": lambda: laplacian(1, 2),
        "laplacian-2d": lambda: laplacian(2, 2),
        "laplacian-3d": lambda: laplacian(3, 2),
        "bilaplacian-2d": lambda: bilaplacian(2),
        "bilaplacian-3d": lambda: bilaplacian(3),
        "identity-1d": lambda: Stencil.identity(1),
        "identity-2d": lambda: Stencil.identity(2),
    }
    if name not in table:
        raise StencilkitError(Errc.invalid_argument, f"unknown builtin stencil '{name}'")
    return table[name]()


def from_entries(dim: int, h_power: int, items: Iterable[Tuple[Offset, Fraction]]) -> Stencil:
    out: Dict[Offset, Fraction] = {}
    for o, c in items:
        out[tuple(o)] = out.get(tuple(o), Fraction(0)) + Fraction(c)
    return Stencil(dim, h_power, out)

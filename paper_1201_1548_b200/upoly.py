"""Square-free decomposition with the GPU gcd plugged in.

Restates curvekit.upoly.squarefree_decompose (pkg/src/curvekit/upoly.py:241-299,
Yun's algorithm) for users without curvekit; its ``gcd_fn`` injection point
defaults to the B200 ``int_gcd_uni``.  The rational divisions of Yun's loop
stay on the host exactly as in the reference; every gcd runs on the GPU.
With curvekit installed, ``paper_1201_1548_b200.install()`` makes the
reference's own function use the GPU gcd (its lazy import of
``curvekit.modpoly.int_gcd_uni`` is rebound).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from fractions import Fraction


@dataclass(frozen=True)
class SquareFreeDecomposition:
    factors: tuple  # ((IntPoly-as-tuple, multiplicity), ...) primitive, lc > 0
    content: int

    def reconstruct(self) -> list:
        out = [self.content]
        for f, m in self.factors:
            for _ in range(m):
                out = _mul(out, list(f))
        return out


def _mul(p, q):
    if not p or not q:
        return []
    out = [0] * (len(p) + len(q) - 1)
    for i, a in enumerate(p):
        if a:
            for j, b in enumerate(q):
                out[i + j] += a * b
    while out and out[-1] == 0:
        out.pop()
    return out


def _primitive(p):
    if not p:
        return []
    c = 0
    for a in p:
        c = math.gcd(c, a)
    if p[-1] < 0:
        c = -c
    return [a // c for a in p]


def _derivative(p):
    out = [i * p[i] for i in range(1, len(p))]
    while out and out[-1] == 0:
        out.pop()
    return out


def _divmod_frac(p, d):
    p = [Fraction(a) for a in p]
    d = [Fraction(a) for a in d]
    while d and d[-1] == 0:
        d.pop()
    if not d:
        raise ZeroDivisionError
    q = [Fraction(0)] * max(0, len(p) - len(d) + 1)
    r = list(p)
    while True:
        while r and r[-1] == 0:
            r.pop()
        if len(r) < len(d):
            break
        c = r[-1] / d[-1]
        k = len(r) - len(d)
        q[k] = c
        for j, b in enumerate(d):
            r[k + j] -= c * b
        r.pop()
    return q, r


def _frac_div(p, d):
    q, r = _divmod_frac(p, d)
    if any(r):
        raise ArithmeticError("inexact division in square-free decomposition")
    return q


def _sub_frac(p, q):
    n = max(len(p), len(q))
    out = [(p[i] if i < len(p) else Fraction(0)) - (q[i] if i < len(q) else Fraction(0)) for i in range(n)]
    while out and out[-1] == 0:
        out.pop()
    return out


def _clear_denominators(p):
    lcm = 1
    for a in p:
        a = Fraction(a)
        lcm = lcm * a.denominator // math.gcd(lcm, a.denominator)
    out = [int(Fraction(a) * lcm) for a in p]
    while out and out[-1] == 0:
        out.pop()
    return out


def squarefree_decompose(p, gcd_fn=None) -> SquareFreeDecomposition:
    """Yun's square-free decomposition p = content * prod f_i^i (upoly.py:253-279)."""
    if not p:
        raise ValueError("zero polynomial")
    if gcd_fn is None:
        from .modpoly import int_gcd_uni
        gcd_fn = int_gcd_uni
    p = list(p)
    if len(p) == 1:
        return SquareFreeDecomposition((), p[0])
    w = _primitive(p)
    cont = p[-1] // w[-1] if w[-1] else 0
    dp = _derivative(w)
    g = gcd_fn(w, dp)
    if len(g) - 1 == 0:
        return SquareFreeDecomposition(((tuple(w), 1),), cont)
    factors = []
    v = _frac_div(w, g)
    u = _frac_div(dp, g)
    i = 1
    while len(v) > 1:
        d = _sub_frac(u, [k * v[k] for k in range(1, len(v))])
        h = gcd_fn(_clear_denominators(v), _clear_denominators(d))
        if len(h) - 1 > 0:
            factors.append((tuple(h), i))
        v, u = _frac_div(v, h), _frac_div(d, h)
        i += 1
    return SquareFreeDecomposition(tuple(factors), cont)

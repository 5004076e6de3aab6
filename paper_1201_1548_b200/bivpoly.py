"""Minimal bivariate container with the accessors the hot path consumes.

The drop-in accepts the reference's ``curvekit.bivpoly.BivPoly``
(pkg/src/curvekit/bivpoly.py:18-147) or anything exposing the same accessors;
this class provides them for users without curvekit: sparse ``{(i, j): c}``
for c x^i y^j, ``coeffs_wrt_y`` (:74-81), ``swap`` (:146-147), degrees.
"""

from __future__ import annotations


class BivPoly:
    __slots__ = ("terms",)

    def __init__(self, terms=None):
        self.terms = {}
        if terms:
            for (i, j), c in dict(terms).items():
                if c:
                    self.terms[(int(i), int(j))] = int(c)

    def is_zero(self) -> bool:
        return not self.terms

    def deg_x(self) -> int:
        return max((i for i, _ in self.terms), default=-1)

    def deg_y(self) -> int:
        return max((j for _, j in self.terms), default=-1)

    def total_degree(self) -> int:
        return max((i + j for i, j in self.terms), default=-1)

    def coeffs_wrt_y(self) -> list:
        out = [[] for _ in range(self.deg_y() + 1)]
        for (i, j), c in self.terms.items():
            col = out[j]
            if len(col) < i + 1:
                col.extend([0] * (i + 1 - len(col)))
            col[i] = c
        for col in out:
            while col and col[-1] == 0:
                col.pop()
        return out

    def lead_coeff_y(self) -> list:
        cs = self.coeffs_wrt_y()
        return cs[-1] if cs else []

    def swap(self) -> "BivPoly":
        return BivPoly({(j, i): c for (i, j), c in self.terms.items()})

    def diff(self, var: str) -> "BivPoly":
        terms = {}
        for (i, j), c in self.terms.items():
            if var == "x" and i:
                terms[(i - 1, j)] = terms.get((i - 1, j), 0) + i * c
            elif var == "y" and j:
                terms[(i, j - 1)] = terms.get((i, j - 1), 0) + j * c
        return BivPoly(terms)

    def __eq__(self, other) -> bool:
        return isinstance(other, BivPoly) and self.terms == other.terms

    def __hash__(self):
        return hash(frozenset(self.terms.items()))

    def __repr__(self) -> str:
        return f"BivPoly({self.terms!r})"


def as_biv(obj):
    """Accept a BivPoly-like object or a {(i, j): c} dict."""
    if isinstance(obj, dict):
        return BivPoly(obj)
    if hasattr(obj, "coeffs_wrt_y"):
        return obj
    raise TypeError("expected a BivPoly or a {(i, j): c} dict")

"""Minimal bivariate container with the accessors the hot path consumes.

The drop-in accepts the reference's ``curvekit.bivpoly.BivPoly``
(pkg/src/curvekit/bivpoly.py:18-147) or anything exposing the same accessors;
this class provides them for users without curvekit: sparse ``{(i, j): c}``
for c x^i y^j, ``coeffs_wrt_y`` (:74-81), ``swap`` (:146-147), degrees.
"""

from __future__ import annotations

import numpy as np


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


# ---------------------------------------------------------------------------
# bivariate gcd: drop-in for curvekit.bivpoly.gcd_biv,
# is_squarefree_biv, square_part (pkg/src/curvekit/bivpoly.py:266-320)
# ---------------------------------------------------------------------------

def _maker(like):
    """Constructor of the caller's polynomial type (the reference's BivPoly or ours)."""
    cls = type(like) if hasattr(like, "terms") else BivPoly
    return lambda terms: cls(terms)


def _cols_to_terms(cols) -> dict:
    return {(i, j): a for j, c in enumerate(cols) for i, a in enumerate(c) if a}


def _deg_y(cols) -> int:
    return len(cols) - 1


def content_y(cols, gcd_fn=None) -> list:
    """bivpoly.py:183-197: gcd in Z[x] of the y-coefficients, integer content included."""
    from math import gcd as igcd
    from .modpoly import _primitive, int_gcd_uni
    gcd_fn = gcd_fn or int_gcd_uni
    cs = [c for c in cols if c]
    if not cs:
        return []
    g = _primitive(cs[0])
    for c in cs[1:]:
        if len(g) - 1 == 0:
            break
        g = gcd_fn(g, c)
    if len(g) - 1 == 0:
        g = [1]
    ci = 0
    for c in cs:
        for a in c:
            ci = igcd(ci, a)
    return [a * ci for a in g]


def div_uni_x(cols, d) -> list:
    """bivpoly.py:199-210: exact division of every y-coefficient by d(x)."""
    from .modpoly import _divexact
    out = []
    for c in cols:
        if not c:
            out.append([])
            continue
        q = _divexact(c, d)
        if q is None:
            raise ArithmeticError("inexact division by x-content")
        out.append(q)
    while out and not out[-1]:
        out.pop()
    return out


def _sub_x(p, q):
    n = max(len(p), len(q))
    r = [(p[i] if i < len(p) else 0) - (q[i] if i < len(q) else 0) for i in range(n)]
    while r and r[-1] == 0:
        r.pop()
    return r


def divexact_cols(fc, gc):
    """bivpoly.py:213-240 (divexact_biv) on y-coefficient lists: quotient or None."""
    from .modpoly import _divexact, _mul
    if not gc:
        raise ZeroDivisionError
    if not fc:
        return []
    if len(gc) == 1:
        try:
            return div_uni_x(fc, gc[0])
        except ArithmeticError:
            return None
    qn = len(fc) - len(gc)
    if qn < 0:
        return None
    quot = [[] for _ in range(qn + 1)]
    rem = [list(c) for c in fc]
    glead = gc[-1]
    for k in range(qn, -1, -1):
        top = rem[k + len(gc) - 1]
        while top and top[-1] == 0:
            top.pop()
        if not top:
            continue
        q = _divexact(top, glead)
        if q is None:
            return None
        quot[k] = q
        for j, gcj in enumerate(gc):
            rem[k + j] = _sub_x(rem[k + j], _mul(q, gcj))
    if any(r for r in rem[: len(gc) - 1]):
        return None
    return quot


def _normalize_sign(terms: dict) -> dict:
    """bivpoly.py:298-304: the coefficient of the largest (i, j) is positive."""
    if not terms:
        return terms
    if terms[max(terms)] < 0:
        return {k: -a for k, a in terms.items()}
    return terms


def _modular_gcd_primitive(A, B, table=None):
    """Primitive gcd (up to sign) of primitive A, B in Z[x][y], deg_y A >= deg_y B >= 1.

    Brown's dense modular algorithm: the GPU computes Gamma(x_t) * monic
    gcd(A(x_t, y), B(x_t, y)) mod p for a batch of primes and points
    (ckb_biv_gcd_images), the host keeps the images of minimal y-degree
    (every other image is unlucky: the image degree never falls below
    deg_y gcd where the leading coefficients do not vanish), interpolates
    them in x (ckb_interp_points) and lifts them by CRT (ckb_crt_lift);
    the candidate is verified by exact trial division, as the reference
    verifies its univariate gcds (modpoly.py:337-340).
    """
    from math import gcd as igcd
    from . import _lib
    from .modpoly import _content, crt_lift, int_gcd_uni, zp_interpolate_arrays
    from .planner import ints_to_limbs
    from .primes30 import PRIMES30
    table = table or PRIMES30
    m, n = _deg_y(A), _deg_y(B)
    lcA, lcB = A[-1], B[-1]
    gam = [a * igcd(_content(lcA), _content(lcB)) for a in int_gcd_uni(lcA, lcB)]
    dax = max(len(c) - 1 for c in A)
    dbx = max(len(c) - 1 for c in B)
    dgam = len(gam) - 1
    D = dgam + min(dax, dbx)          # deg_x H <= deg_x Gamma + deg_x gcd
    npts = D + 1
    NP = npts + 8 + npts // 8         # spare points for vanishing leading coefficients / unlucky points
    flat = []
    for cols, dx in ((A, dax), (B, dbx)):
        for c in cols:
            flat.extend(c)
            flat.extend([0] * (dx + 1 - len(c)))
    flat.extend(gam)
    limbs, L = ints_to_limbs(flat)
    C = len(flat)
    degs = np.array([len(c) - 1 for c in A] + [len(c) - 1 for c in B], dtype=np.int16)
    Wo = m + 1
    lib = _lib.lib()
    best = None
    acc_p, acc_r = [], []
    idx, batch = 0, 2
    while True:
        primes = []
        while len(primes) < batch:
            if idx >= len(table):
                raise ArithmeticError("prime table exhausted in gcd computation")
            primes.append(table[idx][0])
            idx += 1
        K = len(primes)
        parr = np.array(primes, dtype=np.uint32)
        out = np.zeros((K, NP, Wo), dtype=np.uint32)
        odeg = np.zeros((K, NP), dtype=np.int32)
        _lib.check(lib.ckb_biv_gcd_images(_lib.ptr(limbs), C, L, _lib.ptr(degs), m, n, dax, dbx, dgam,
                                          _lib.ptr(parr), K, NP, _lib.ptr(out), Wo, _lib.ptr(odeg)),
                   "ckb_biv_gcd_images")
        new = []
        for k, p in enumerate(primes):
            ok = odeg[k] >= 0
            if ok.sum() < npts:
                continue
            e = int(odeg[k][ok].min())
            sel = np.nonzero(odeg[k] == e)[0][:npts]
            if len(sel) < npts:
                continue
            if e == 0:
                return [[1]]
            if best is None or e < best:
                best = e
                acc_p, acc_r = [], []
                new = []
            elif e > best:
                continue
            new.append((k, p, sel))
        if new:
            xs = np.stack([(sel + 1).astype(np.uint32) for _, _, sel in new])        # [k][npts]
            vals = np.stack([out[k, sel, :best + 1].T for k, _, sel in new])         # [k][e+1][npts]
            coeffs = zp_interpolate_arrays(xs, vals, [p for _, p, _ in new])         # [k][e+1][npts]
            for (_, p, _), cf in zip(new, coeffs):
                acc_p.append(p)
                acc_r.append(cf.reshape(-1))
        if acc_p:
            mod_bits = sum(p.bit_length() - 1 for p in acc_p)
            vals = crt_lift(np.stack(acc_r), acc_p)
            hb = max((abs(v).bit_length() for v in vals), default=0)
            if hb + 20 < mod_bits:  # the symmetric lift has settled well inside the modulus
                H = [vals[i * npts:(i + 1) * npts] for i in range(best + 1)]
                for c in H:
                    while c and c[-1] == 0:
                        c.pop()
                if H[-1]:
                    pp = div_uni_x(H, content_y(H))
                    if _deg_y(pp) == best and divexact_cols(A, pp) is not None and \
                            divexact_cols(B, pp) is not None:
                        return pp
        batch = min(2 * batch, 64)


def gcd_biv(f, g):
    """Primitive gcd in Z[x, y] (positive integer content convention) — bivpoly.py:266-295.

    Same contents, primitive parts and sign normalisation as the reference; the
    gcd of the primitive parts is computed modularly on the GPU
    (_modular_gcd_primitive) instead of by the primitive PRS.
    """
    from .modpoly import _mul, int_gcd_uni
    mk = _maker(f)
    F, G = as_biv(f), as_biv(g)
    if F.is_zero():
        return mk(_normalize_sign(dict(G.terms)))
    if G.is_zero():
        return mk(_normalize_sign(dict(F.terms)))
    fc, gc = F.coeffs_wrt_y(), G.coeffs_wrt_y()
    if len(fc) == 1 and len(gc) == 1:
        return mk(_cols_to_terms([int_gcd_uni(fc[0], gc[0])]))
    cf, cg = content_y(fc), content_y(gc)
    cont = int_gcd_uni(cf, cg)
    pf, pg = div_uni_x(fc, cf), div_uni_x(gc, cg)
    if _deg_y(pf) < _deg_y(pg):
        pf, pg = pg, pf
    pp = [[1]] if _deg_y(pg) == 0 else _modular_gcd_primitive(pf, pg)
    return mk(_normalize_sign(_cols_to_terms([_mul(c, cont) for c in pp])))


def is_squarefree_biv(f) -> bool:
    """bivpoly.py:307-314: square-freeness over Q[x, y] via gcds with both partials."""
    F = as_biv(f)
    if F.is_zero():
        return False
    g = gcd_biv(F, F.diff("x"))
    g = gcd_biv(g, F.diff("y"))
    return g.total_degree() == 0


def square_part(f):
    """bivpoly.py:317-320: gcd(f, f_x, f_y)."""
    F = as_biv(f)
    g = gcd_biv(f, F.diff("x"))
    return gcd_biv(g, F.diff("y"))

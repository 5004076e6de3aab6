"""Exact-integer forms of the planner's bounds (TEST INFRASTRUCTURE).

The product planner (paper_1201_1548_b200/planner.py) works in log2 space
(log2_coeff_bound, choose_primes_log2); these big-integer versions exist only
to check it: the reference's own _det_coeff_bound (modpoly.py:397-414),
restated, the Hadamard refinement, and the prime loop of modpoly.py:370-379
with exact products.
"""

from math import isqrt

from paper_1201_1548_b200.planner import _lc_vanishes, _norm1
from paper_1201_1548_b200.primes30 import PRIMES30


def det_coeff_bound_ref(fc, gc) -> int:
    """The reference's bound (modpoly.py:397-414), restated verbatim."""
    m, n = len(fc) - 1, len(gc) - 1
    norm_f = [_norm1(c) for c in fc]
    norm_g = [_norm1(c) for c in gc]
    bound = 1
    for j in range(m + n):
        s = 0
        for r in range(n):
            k = m - j + r
            if 0 <= k <= m:
                s += norm_f[k]
        for r in range(m):
            k = n - j + r
            if 0 <= k <= n:
                s += norm_g[k]
        bound *= max(1, s)
    return bound


def det_coeff_bound(fc, gc) -> int:
    """min(reference bound, row Hadamard, column Hadamard) -- all valid."""
    m, n = len(fc) - 1, len(gc) - 1
    nf = [_norm1(c) for c in fc]
    ng = [_norm1(c) for c in gc]
    ref = det_coeff_bound_ref(fc, gc)
    # rows: n rows carrying f's coefficients, m rows carrying g's
    row2 = sum(a * a for a in nf) ** n * sum(a * a for a in ng) ** m
    col2 = 1
    for j in range(m + n):
        s = 0
        for r in range(n):
            k = m - j + r
            if 0 <= k <= m:
                s += nf[k] * nf[k]
        for r in range(m):
            k = n - j + r
            if 0 <= k <= n:
                s += ng[k] * ng[k]
        col2 *= max(1, s)
    had = isqrt(min(row2, col2)) + 1
    return min(ref, had)


def choose_primes(bound: int, lcf, lcg, start: int = 0, table=PRIMES30):
    """Primes (descending, from ``start``) until prod > 4 * bound.

    The reference stops at prod > 2 * bound (modpoly.py:374-375); one more bit
    of margin keeps |x / M| < 1/4 so the explicit CRT's FP64 rounding of
    sum_i y_i / p_i is always exact (csrc/ckb_crt.cu)."""
    target = 4 * bound
    primes, gens = [], []
    mod = 1
    i = start
    const = len(lcf) == 1 and len(lcg) == 1
    a, b = (lcf[0], lcg[0]) if const else (None, None)
    while mod <= target:
        if i >= len(table):
            raise ArithmeticError("prime table exhausted in resultant computation")
        p, g = table[i]
        i += 1
        if const:
            if a % p == 0 or b % p == 0:
                continue
        elif _lc_vanishes(lcf, p) or _lc_vanishes(lcg, p):
            continue
        primes.append(p)
        gens.append(g)
        mod *= p
    return primes, gens, mod

"""Host planner for the multi-modular resultant: bounds, primes, points, packing.

Reference behaviour being planned (pkg/src/curvekit/modpoly.py:348-394):
  * CRT stops once the modulus exceeds 2 * _det_coeff_bound (:370, :374-375,
    :397-414).  Here the bound is min(reference bound, row Hadamard bound,
    column Hadamard bound) -- all valid bounds on every coefficient of
    det Sylvester(f, g) (a coefficient of det S(x) is at most
    max_{|z|=1} |det S(z)| <= prod_rows ||row||_2 with |S_ij(z)| <= ||S_ij||_1).
  * The number of points is one more than a degree bound of res.  The
    reference uses deg_x f * n + deg_x g * m (:371); the Bezout-type bound
    n * tdeg f + m * tdeg g - m n (sum of row/column degree weights of the
    Sylvester matrix) is also valid; N = 1 + min of both.
  * Primes: the device table (primes30.py) in descending order, skipping
    primes that annihilate a leading y-coefficient polynomial (:378-379).
The result is the unique integer polynomial determined by these bounds, so it
is identical to the reference's for every seed.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .primes30 import PRIMES30


@dataclass
class Packed:
    limbs: np.ndarray   # uint32 [C * L]
    degs: np.ndarray    # int16 [m + n + 2]
    C: int
    L: int
    m: int
    n: int
    dfx: int
    dgx: int
    # filled by pack_terms: per-row 1-norms (doubles), total degrees, leading rows
    norms: list | None = None
    tdf: int = -1
    tdg: int = -1
    lcf: list | None = None
    lcg: list | None = None


@dataclass
class Plan:
    primes: np.ndarray  # uint32 [K]
    gens: np.ndarray    # uint32 [K]
    N: int
    LW: int
    bound_bits: int
    modulus_bits: int


def _trimmed_deg(c) -> int:
    d = len(c) - 1
    while d >= 0 and c[d] == 0:
        d -= 1
    return d


def _norm1(c) -> int:
    return sum(abs(a) for a in c)


def log2_coeff_bound(fc, gc) -> float:
    """log2 of det_coeff_bound(fc, gc), evaluated in floating point.

    Only the number of primes depends on the bound, so the planner works in
    log2 space (no big-integer products): every term is a log2 of an exact
    integer (relative error ~1e-16), the sums have ~(m + n) terms, and the
    planner adds a full bit of margin on top -- far above the rounding error.
    """
    from math import log2
    m, n = len(fc) - 1, len(gc) - 1
    nf = [_norm1(c) for c in fc]
    ng = [_norm1(c) for c in gc]
    # column j of the Sylvester matrix holds f's coefficients k in
    # [max(0, m-j), min(m, m-j+n-1)] and g's in [max(0, n-j), min(n, n-j+m-1)]:
    # contiguous ranges, so prefix sums give every column sum exactly
    pf, pf2, pg, pg2 = [0], [0], [0], [0]
    for a in nf:
        pf.append(pf[-1] + a)
        pf2.append(pf2[-1] + a * a)
    for a in ng:
        pg.append(pg[-1] + a)
        pg2.append(pg2[-1] + a * a)
    ref = 0.0
    col = 0.0
    for j in range(m + n):
        lo, hi = max(0, m - j), min(m, m - j + n - 1)
        s = pf[hi + 1] - pf[lo] if lo <= hi else 0
        s2 = pf2[hi + 1] - pf2[lo] if lo <= hi else 0
        lo, hi = max(0, n - j), min(n, n - j + m - 1)
        if lo <= hi:
            s += pg[hi + 1] - pg[lo]
            s2 += pg2[hi + 1] - pg2[lo]
        ref += log2(max(1, s))
        col += 0.5 * log2(max(1, s2))
    row = 0.5 * (n * log2(max(1, sum(a * a for a in nf))) + m * log2(max(1, sum(a * a for a in ng))))
    return min(ref, row, col)


def log2_bound_from_norms(nf, ng) -> float:
    """log2_coeff_bound from per-row 1-norms given as doubles (pack_terms).

    Same three bounds; the column sums of the Sylvester matrix are windows of
    n (f) and m (g) consecutive rows, i.e. full convolutions with a box, summed
    directly (all terms positive: relative error <= (m + n) eps, no prefix-sum
    cancellation), so the result is within ~1e-12 bits of the exact one, far
    inside the planner's one-bit margin."""
    if _ckb_limbs is not None and hasattr(_ckb_limbs, "norms_log2_bound"):
        return _ckb_limbs.norms_log2_bound(nf, ng)  # the same sums in one C pass
    nf = np.asarray(nf, dtype=np.float64)
    ng = np.asarray(ng, dtype=np.float64)
    m, n = len(nf) - 1, len(ng) - 1
    s = np.convolve(nf, np.ones(n)) + np.convolve(ng, np.ones(m))
    s2 = np.convolve(nf * nf, np.ones(n)) + np.convolve(ng * ng, np.ones(m))
    ref = float(np.log2(np.maximum(s, 1.0)).sum())
    col = 0.5 * float(np.log2(np.maximum(s2, 1.0)).sum())
    row = 0.5 * (n * np.log2(max(1.0, float((nf * nf).sum()))) + m * np.log2(max(1.0, float((ng * ng).sum()))))
    return min(ref, float(row), col)


def choose_primes_log2(bound_log2: float, lcf, lcg, start: int = 0, table=PRIMES30):
    """Primes (descending, from ``start``) until log2(prod) > log2(4 B) + 1.

    A prime annihilates a leading y-coefficient polynomial (modpoly.py:378-379)
    iff it divides the gcd of that polynomial's coefficients, so the scan tests
    two integers per prime (none at all when both gcds are 1, the usual case)."""
    primes, gens, _ = _choose_primes(bound_log2, lcf, lcg, start, table)
    return primes.tolist(), gens.tolist()


def _choose_primes(bound_log2: float, lcf, lcg, start: int = 0, table=PRIMES30):
    """choose_primes_log2 as (uint32 primes, uint32 generators, log2 of their product)."""
    from math import gcd
    target = bound_log2 + 3.0
    gf, gg = gcd(*lcf), gcd(*lcg)
    check = gf != 1 or gg != 1
    logs, cum, parr, garr = _log2_table(table)
    # the count from the running log-sum, valid when no prime of the run is skipped
    import bisect
    k = bisect.bisect_right(cum, cum[start] + target)  # first index whose prefix exceeds the target
    if not check or (k <= len(table) and not ((_mod_many(gf, parr[start:k]) == 0)
                                              | (_mod_many(gg, parr[start:k]) == 0)).any()):
        if k > len(table):
            raise ArithmeticError("prime table exhausted in resultant computation")
        return parr[start:k].astype(np.uint32), garr[start:k].astype(np.uint32), cum[k] - cum[start]
    primes, gens = [], []
    acc = 0.0
    i = start
    while acc <= target:
        if i >= len(table):
            raise ArithmeticError("prime table exhausted in resultant computation")
        p, g = table[i]
        if check and (gf % p == 0 or gg % p == 0):
            i += 1
            continue
        primes.append(p)
        gens.append(g)
        acc += logs[i]
        i += 1
    return np.array(primes, dtype=np.uint32), np.array(gens, dtype=np.uint32), acc


_LOG2 = {}


def _mod_many(x: int, ps: np.ndarray) -> np.ndarray:
    """|x| mod p for every p < 2^31 of ``ps``: Horner over x's 31-bit limbs (int64 lanes)."""
    x = abs(x)
    r = np.zeros(len(ps), dtype=np.int64)
    for sh in range(((x.bit_length() + 30) // 31 - 1) * 31, -1, -31):
        r = ((r << 31) + ((x >> sh) & 0x7FFFFFFF)) % ps
    return r


def _log2_table(table):
    """(log2 p, prefix sums of log2 p from 0, primes, generators) of a prime table."""
    t = _LOG2.get(id(table))
    if t is None or len(t[0]) != len(table):
        from itertools import accumulate
        from math import log2
        logs = [log2(p) for p, _ in table]
        t = (logs, [0.0] + list(accumulate(logs)), np.array([p for p, _ in table], dtype=np.int64),
             np.array([g for _, g in table], dtype=np.int64))
        _LOG2[id(table)] = t
    return t


def point_count(fc, gc, dfx: int, dgx: int, tdf: int, tdg: int) -> int:
    m, n = len(fc) - 1, len(gc) - 1
    ref = dfx * n + dgx * m
    bez = n * tdf + m * tdg - m * n
    return min(ref, bez) + 1


def _lc_vanishes(lc, p: int) -> bool:
    return all(c % p == 0 for c in lc)


def pack_grid(fc, gc) -> Packed:
    """Dense two's-complement limb grid of f's then g's y-coefficients."""
    m, n = len(fc) - 1, len(gc) - 1
    degf = [_trimmed_deg(c) for c in fc]
    degg = [_trimmed_deg(c) for c in gc]
    dfx = max(0, max(degf))
    dgx = max(0, max(degg))
    C = (m + 1) * (dfx + 1) + (n + 1) * (dgx + 1)
    maxbits = 0
    for cs in (fc, gc):
        for c in cs:
            for a in c:
                if a:
                    b = a.bit_length() if a > 0 else (-a).bit_length()
                    if b > maxbits:
                        maxbits = b
    L = max(1, (maxbits + 1 + 31) // 32)
    if L <= 2:
        flat = []
        for cs, dx in ((fc, dfx), (gc, dgx)):
            for c in cs:
                flat.extend(c)
                flat.extend([0] * (dx + 1 - len(c)))
        grid = np.array(flat, dtype=np.int64)
        limbs = grid.view(np.uint32)
        if L == 1:
            limbs = np.ascontiguousarray(limbs.reshape(C, 2)[:, 0])
        L = 1 if L == 1 else 2
    else:
        nb = 4 * L
        zero = bytes(nb)
        parts = []
        for cs, dx in ((fc, dfx), (gc, dgx)):
            for c in cs:
                row = [a.to_bytes(nb, "little", signed=True) if a else zero for a in c]
                row += [zero] * (dx + 1 - len(c))
                parts.extend(row)
        limbs = np.frombuffer(b"".join(parts), dtype=np.uint32)
    degs = np.array(degf + degg, dtype=np.int16)
    return Packed(np.ascontiguousarray(limbs), degs, C, L, m, n, dfx, dgx)


def pack_terms(f, g, swap: bool = False):
    """pack_grid straight from two term dicts ({(i, j): c}, the reference's
    BivPoly.terms, bivpoly.py:18-25) in one C pass (host/ckb_limbs.c
    terms_grid), with what plan_packed needs; None when the C helper is absent
    or the input is not plain ints (the caller takes coeffs_wrt_y + pack_grid)."""
    if _ckb_limbs is None:
        return None
    tf = f if isinstance(f, dict) else getattr(f, "terms", None)
    tg = g if isinstance(g, dict) else getattr(g, "terms", None)
    if type(tf) is not dict or type(tg) is not dict:
        return None
    r = _ckb_limbs.terms_grid(tf, tg, bool(swap))
    if r is None or r[9] is None:
        return None
    limbs, L, m, n, dfx, dgx, tdf, tdg, degs, norms, lcf, lcg = r
    C = (m + 1) * (dfx + 1) + (n + 1) * (dgx + 1)
    return Packed(np.frombuffer(limbs, dtype=np.uint32), np.frombuffer(degs, dtype=np.int16), C, L, m, n, dfx, dgx,
                  norms, tdf, tdg, lcf, lcg)


def plan_resultant(fc, gc, tdf: int, tdg: int, dfx: int, dgx: int, start: int = 0) -> Plan:
    return _plan(log2_coeff_bound(fc, gc), point_count(fc, gc, dfx, dgx, tdf, tdg), fc[-1], gc[-1], start)


def plan_packed(pk: Packed, start: int = 0) -> Plan:
    """plan_resultant for a grid from pack_terms (its norms, degrees and leading rows)."""
    m, n = pk.m, pk.n
    N = min(pk.dfx * n + pk.dgx * m, n * pk.tdf + m * pk.tdg - m * n) + 1  # point_count
    return _plan(log2_bound_from_norms(pk.norms[:m + 1], pk.norms[m + 1:]), N, pk.lcf, pk.lcg, start)


def _plan(blog: float, N: int, lcf, lcg, start: int) -> Plan:
    primes, gens, lsum = _choose_primes(blog, lcf, lcg, start)
    # bit length of the modulus (LW words must hold M): the float sum is within
    # ~1e-12 of log2 M; rounding it up by 1e-6 can only add a spare word
    mbits = int(lsum + 1e-6) + 1
    LW = (mbits + 31) // 32
    return Plan(primes, gens, N, LW, int(blog) + 1, mbits)


def limbs_to_ints(buf: np.ndarray, N: int, LW: int) -> list:
    """[N][LW] two's-complement u32 limbs -> list of Python ints."""
    if _ckb_limbs is not None:
        return _ckb_limbs.limbs_to_ints(memoryview(np.ascontiguousarray(buf, dtype=np.uint32)).cast("B"), N, LW)
    raw = np.ascontiguousarray(buf).tobytes()  # bytes slices beat memoryview slices here
    w = 4 * LW
    fb = int.from_bytes
    return [fb(raw[i * w:(i + 1) * w], "little", signed=True) for i in range(N)]


try:  # the C helper built next to the library (paper_1201_1548_b200/host/ckb_limbs.c)
    from . import ckb_limbs as _ckb_limbs
except ImportError:  # pragma: no cover - pure-Python conversion (same result)
    _ckb_limbs = None


def ints_to_limbs(vals, L: int | None = None) -> tuple:
    """list of ints -> ([len][L] two's-complement u32 limbs, L)."""
    if L is None:
        mb = max((abs(v).bit_length() for v in vals), default=0)
        L = max(1, (mb + 1 + 31) // 32)
    nb = 4 * L
    raw = b"".join(int(v).to_bytes(nb, "little", signed=True) for v in vals)
    return np.frombuffer(raw, dtype=np.uint32).copy(), L

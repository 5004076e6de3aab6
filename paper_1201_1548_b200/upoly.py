"""Real-root isolation pieces of curvekit.upoly on the GPU.

The Descartes sign-variation test (upoly._variations_on, pkg/src/curvekit/
upoly.py:338-346) as one batched GPU call per subdivision level, and the
breadth-first descartes_isolate around it.  Square-free decomposition is the
reference's own function: ``paper_1201_1548_b200.install()`` rebinds its lazy
import of ``curvekit.modpoly.int_gcd_uni`` (upoly.py:258) to the GPU gcd, so
Yun's loop stays the reference's and every gcd runs on the device.
"""

from __future__ import annotations

import math
from fractions import Fraction


# ---------------------------------------------------------------------------
# Descartes test of real-root isolation on the GPU
# ---------------------------------------------------------------------------

class _DescHandles:
    """Per-polynomial device state (residues + plan), keyed by the list object
    descartes_isolate passes to every test of one isolation (upoly.py:387-405)."""

    def __init__(self, size: int = 8):
        import threading
        self.size = size
        self.entries = []  # [poly list, snapshot, handle, K]
        self.lock = threading.Lock()

    def get(self, p, n: int, K: int):
        with self.lock:
            return self._get(p, n, K)

    def _get(self, p, n: int, K: int):
        from . import _lib
        from .planner import ints_to_limbs
        from .primes30 import PRIMES30
        import numpy as np
        snap = tuple(p[:n + 1])  # the full coefficients: an in-place edit of the list re-prepares
        for e in self.entries:
            if e[0] is p and e[1] == snap and e[3] >= K:
                return e[2], e[3]
        # (re)prepare with headroom: deeper subdivisions need more primes
        Kp = min(len(PRIMES30), max(256, 2 * K))
        lib = _lib.lib()
        limbs, L = ints_to_limbs(p[:n + 1])
        primes = np.array([q for q, _ in PRIMES30[:Kp]], dtype=np.uint32)
        gens = np.array([g for _, g in PRIMES30[:Kp]], dtype=np.uint32)
        h = _lib.check(lib.ckb_descartes_prepare(_lib.ptr(limbs), n, L, _lib.ptr(primes), _lib.ptr(gens), Kp),
                       "ckb_descartes_prepare")
        for e in [e for e in self.entries if e[0] is p]:
            lib.ckb_descartes_release(e[2])
            self.entries.remove(e)
        self.entries.insert(0, [p, snap, h, Kp])
        while len(self.entries) > self.size:
            lib.ckb_descartes_release(self.entries.pop()[2])
        return h, Kp


_desc = _DescHandles()
_log2_prefix = None


def _primes_for_bits(bits: float) -> int:
    """Fewest PRIMES30 (in order) whose product exceeds 2^bits, rounded up to 64."""
    global _log2_prefix
    from .primes30 import PRIMES30
    if _log2_prefix is None:
        acc, pre = 0.0, []
        for q, _ in PRIMES30:
            acc += math.log2(q)
            pre.append(acc)
        _log2_prefix = pre
    import bisect
    k = bisect.bisect_right(_log2_prefix, bits) + 1
    # a log-spaced ladder (64, 80, 96, 112, 128, 160, 192, 224, 256, 320, ...: four
    # steps per doubling) so the cached CRT tables are reused across subdivision depths
    j = 0
    while True:
        rung = -(-int(64 * 2 ** (j / 4)) // 16) * 16
        if rung >= k:
            k = rung
            break
        j += 1
    if k > min(len(_log2_prefix), 8192):
        raise NotImplementedError("Descartes test needs more than 8192 primes")
    return k


def variations_on(p, a, b) -> int:
    """Sign-variation bound for the roots of p in (a, b) — upoly._variations_on
    (pkg/src/curvekit/upoly.py:338-346) on the GPU; a, b are dyadics (man, exp).

    Exact: the coefficients of taylor_shift(reversed(compose_linear(p, ...)), 1)
    are computed modulo enough primes for their a-priori bound and lifted by the
    CRT before their signs are counted, so the result is the reference's.
    """
    from . import _lib
    from .planner import ints_to_limbs
    import numpy as np
    e = min(a.exp, b.exp, 0)
    a_num = a.man << (a.exp - e)
    b_num = b.man << (b.exp - e)
    w = b_num - a_num
    ld = -e
    n = len(p) - 1
    while n >= 0 and p[n] == 0:
        n -= 1
    if n < 1:
        return 0  # compose_linear of a constant has one coefficient: no variation
    # |c|_inf <= 2^n |r|_1 <= 2^n sum_i |p_i| 2^(ld (n-i)) (|a| + |w|)^i   (bit-length bounds)
    t = (abs(a_num) + abs(w)).bit_length()
    top = max(abs(p[i]).bit_length() + ld * (n - i) + i * t for i in range(n + 1) if p[i])
    bits = top + math.log2(n + 1) + n + 4  # M > 4 * bound for the explicit CRT
    K = _primes_for_bits(bits)
    h, _ = _desc.get(p, n, K)
    LW = (int(_log2_prefix[K - 1]) + 1 + 1 + 31) // 32 + 1
    aw, AL = ints_to_limbs([a_num, w])
    v = np.zeros(1, dtype=np.int32)
    lib = _lib.lib()
    _lib.check(lib.ckb_descartes_variations(h, _lib.ptr(aw), AL, ld, K, LW, _lib.ptr(v)), "ckb_descartes_variations")
    return int(v[0])


def _variation_bits(pb, n: int, a_num: int, w: int, ld: int) -> float:
    # |c|_inf <= 2^n |r|_1 <= 2^n sum_i |p_i| 2^(ld (n-i)) (|a| + |w|)^i   (bit-length bounds);
    # pb = _coeff_bits(p): the max over i of pb_i + ld (n - i) + i t, evaluated as one numpy max
    import numpy as np
    t = (abs(a_num) + abs(w)).bit_length()
    top = int((pb + np.arange(n + 1, dtype=np.int64) * (t - ld)).max()) + ld * n
    return top + math.log2(n + 1) + n + 4  # M > 4 * bound for the explicit CRT


def _coeff_bits(p, n: int):
    """Bit lengths of |p_0..p_n| (int64; zero coefficients far below any term)."""
    import numpy as np
    return np.array([abs(c).bit_length() if c else -(1 << 60) for c in p[:n + 1]], dtype=np.int64)


_ZQ = (1 << 61) - 1  # prime


def _nonzero_at(p, pmod, x, U) -> bool:
    """U.eval_dyadic(p, x).sign() != 0 (upoly.py:168-179), decided modulo the
    prime q = 2^61 - 1 first: with x = man 2^e, p(x) = 0 iff the integer
    sum_i p_i man^i 2^(k (n - i)) (k = -e > 0; or p(man 2^e) for e >= 0) is 0,
    and a nonzero residue of it proves it nonzero (2 is invertible mod q).  A
    zero residue (probability ~2^-61, or a real root) takes the exact path."""
    q = _ZQ
    xq = x.man % q
    if x.exp >= 0:
        xq = xq * pow(2, x.exp, q) % q
    else:
        xq = xq * pow(pow(2, -x.exp, q), q - 2, q) % q
    acc = 0
    for c in reversed(pmod):
        acc = (acc * xq + c) % q
    if acc:
        return True
    return U.eval_dyadic(p, x).sign() != 0


def variations_batch(p, intervals, pbits=None) -> list:
    """[variations_on(p, a, b) for (a, b) in intervals] with whole batches of
    intervals in one library call (ckb_descartes_variations_batch: every
    interval's Taylor shift for every prime in one launch, one CRT over all
    their coefficients, one sign count per interval)."""
    from . import _lib
    from .planner import ints_to_limbs
    import numpy as np
    intervals = list(intervals)
    n = len(p) - 1
    while n >= 0 and p[n] == 0:
        n -= 1
    if n < 1:
        return [0] * len(intervals)
    pb = pbits if pbits is not None else _coeff_bits(p, n)  # (descartes_isolate passes it once per polynomial)
    params = []
    for a, b in intervals:
        e = min(a.exp, b.exp, 0)
        a_num = a.man << (a.exp - e)
        b_num = b.man << (b.exp - e)
        params.append((a_num, b_num - a_num, -e))
    out = [0] * len(intervals)
    lib = _lib.lib()
    i0 = 0
    while i0 < len(params):
        # chunk so that the CRT input and output stay within ~1 GB of HBM
        bits = max(_variation_bits(pb, n, a_num, w, ld) for a_num, w, ld in params[i0:i0 + 256])
        K = _primes_for_bits(bits)
        LW = (int(_log2_prefix[K - 1]) + 1 + 1 + 31) // 32 + 1
        B = max(1, min(256, len(params) - i0, (1 << 28) // ((n + 1) * (K + 2 * LW))))
        chunk = params[i0:i0 + B]
        h, _ = _desc.get(p, n, K)
        aw, AL = ints_to_limbs([v for a_num, w, _ in chunk for v in (a_num, w)])
        lds = np.array([ld for _, _, ld in chunk], dtype=np.int32)
        v = np.zeros(len(chunk), dtype=np.int32)
        _lib.check(lib.ckb_descartes_variations_batch(h, _lib.ptr(aw), AL, _lib.ptr(lds), len(chunk), K, LW,
                                                      _lib.ptr(v)), "ckb_descartes_variations_batch")
        out[i0:i0 + len(chunk)] = [int(x) for x in v]
        i0 += len(chunk)
    return out


def descartes_isolate(p, check_squarefree: bool = True, multiplicity: int = 1) -> list:
    """curvekit.upoly.descartes_isolate (pkg/src/curvekit/upoly.py:358-408), breadth first.

    The reference pops one interval at a time off a stack and runs one Descartes
    test per pop; the subdivision of an interval depends only on that interval
    (its test and its own split point), so the set of leaves — the isolating
    intervals — does not depend on the traversal order.  Here every interval of
    a subdivision level is tested in ONE batched GPU call (variations_batch);
    split points, the zero root, sorting and _make_disjoint are the reference's
    own code, so the returned brackets are identical.  Needs curvekit (it
    returns the reference's AlgebraicNumber objects).
    """
    import importlib
    U = importlib.import_module("curvekit.upoly")
    if any(isinstance(c, Fraction) for c in p):
        p = U.clear_denominators(p)
    p = U.primitive(U.trim(list(p)))
    if not p:
        raise ValueError("zero polynomial")
    if check_squarefree:
        from .modpoly import int_gcd_uni
        if U.degree(int_gcd_uni(p, U.derivative(p))) > 0:
            raise ValueError("polynomial is not square-free")
    roots = []
    work = list(p)
    if U.degree(work) <= 0:
        return []
    if work[0] == 0:
        i = next(i for i, c in enumerate(work) if c)
        work = work[i:]
        roots.append(U.AlgebraicNumber(tuple(p), U.RealInterval.point(U.ZERO), multiplicity, exact=Fraction(0)))
    if U.degree(work) > 0:
        defining = tuple(U.primitive(work))
        k = U.cauchy_bound_log2(work)
        bound = U.Dyadic(1, k)
        level = [(-bound, bound)]
        nw = len(work) - 1
        while nw >= 0 and work[nw] == 0:
            nw -= 1
        pbits = _coeff_bits(work, nw)
        pmod = [c % _ZQ for c in work]
        while level:
            vs = variations_batch(work, level, pbits)
            nxt = []
            for (a, b), v in zip(level, vs):
                if v == 0:
                    continue
                if v == 1:
                    roots.append(U.AlgebraicNumber(defining, U.RealInterval(a, b), multiplicity))
                    continue
                for m in U._interior_points(a, b):
                    if _nonzero_at(work, pmod, m, U):
                        break
                else:  # pragma: no cover
                    raise ArithmeticError("no non-root subdivision point found")
                nxt.append((a, m))
                nxt.append((m, b))
            level = nxt
    roots.sort(key=lambda r: r.interval.midpoint().as_fraction())
    return U._make_disjoint(roots)

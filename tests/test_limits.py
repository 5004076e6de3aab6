"""Inputs beyond shared memory / the NTT primes: the drop-in accepts every size
the reference accepts (modpoly.py:156-189, upoly.py:338-346 have no limits).

  * zp_resultant_uni at degree 5,000 (operands in a global slice per pair),
  * zp_interpolate with 13,000 points (global slice per problem),
  * the modular gcd at degree 30,000 (global slice per pair),
  * the Descartes test at degree 4,096 (NTT length 2^14, twiddles from L2) and
    at degree >= 8,192 (direct correlations: 2n+1 exceeds the primes' 2^14
    roots of unity), the direct mode pinned against the oracle at small n.
Each is compared with the C oracle (oracle/ckoracle.c) or a size-independent
property."""

import os
import random
from dataclasses import dataclass

import pytest

pytestmark = pytest.mark.gpu


@dataclass(frozen=True)
class Dy:
    man: int
    exp: int


def _horner(c, x, p):
    acc = 0
    for v in reversed(c):
        acc = (acc * x + v) % p
    return acc


def test_uni_resultant_degree_5000(oracle_mod):
    from paper_1201_1548_b200.modpoly import zp_resultant_batch
    rng = random.Random(50)
    p = 2147483629
    cases = []
    for da, db in ((5000, 4999), (4500, 5200), (5000, 1)):
        a = [rng.randrange(p) for _ in range(da + 1)]
        b = [rng.randrange(p) for _ in range(db + 1)]
        a[-1] = a[-1] or 1
        b[-1] = b[-1] or 1
        cases.append((a, b, p))
    got = zp_resultant_batch(cases)
    assert got == [oracle_mod.zp_resultant(a, b, p) for a, b, p in cases]


def test_interpolate_13000_points(oracle_mod):
    from paper_1201_1548_b200.modpoly import zp_interpolate
    rng = random.Random(13)
    p = 1073692673
    n = 13000
    pts = rng.sample(range(1, p), n)
    vals = [rng.randrange(p) for _ in range(n)]
    got = zp_interpolate(pts, vals, p)
    c = list(got.coeffs)
    for i in rng.sample(range(n), 25):
        assert _horner(c, pts[i], p) == vals[i]
    small = zp_interpolate(pts[:600], vals[:600], p)
    assert list(small.coeffs) == oracle_mod.zp_interp(pts[:600], vals[:600], p)


def test_gcd_degree_30000(oracle_mod):
    from paper_1201_1548_b200.modpoly import zp_gcd_batch
    rng = random.Random(30)
    p = 1073643521
    d = [rng.randrange(p) for _ in range(201)]
    d[-1] = 1
    u = [rng.randrange(p) for _ in range(29801)]
    v = [rng.randrange(p) for _ in range(29501)]
    u[-1] = v[-1] = 1

    def mul(x, y):  # y short: one pass of x per coefficient of y
        out = [0] * (len(x) + len(y) - 1)
        for i, c in enumerate(y):
            if c:
                out[i:i + len(x)] = [(o + c * xv) % p for o, xv in zip(out[i:i + len(x)], x)]
        return out
    a = mul(u, d)
    b = mul(v, d)
    (g,) = zp_gcd_batch([(a, b, p)])
    assert g == oracle_mod.zp_gcd(a, b, p)
    assert len(g) - 1 >= 200


def test_descartes_direct_mode_matches_oracle():
    """The direct-correlation mode (forced at small n) against the oracle."""
    from oracle import oracle
    from paper_1201_1548_b200 import upoly
    rng = random.Random(8)
    os.environ["CKB_DESC_DIRECT"] = "1"
    try:
        for _ in range(12):
            deg = rng.randint(2, 120)
            p = [rng.randint(-2 ** 50, 2 ** 50) for _ in range(deg + 1)]
            p[-1] = p[-1] or 5
            a = Dy(rng.randint(-2 ** 30, 2 ** 30), rng.randint(-40, 2))
            b = Dy(a.man + rng.randint(1, 2 ** 30), a.exp)
            got = upoly.variations_batch(list(p), [(a, b)])[0]  # a fresh list: a fresh (direct) handle
            assert got == oracle.variations_on(p, a.man, a.exp, b.man, b.exp)
    finally:
        del os.environ["CKB_DESC_DIRECT"]


def test_descartes_degree_4096_vs_oracle():
    """2n+1 = 8193 -> NTT length 2^14: X, Y in shared memory, twiddles from L2."""
    from oracle import oracle
    from paper_1201_1548_b200 import upoly
    rng = random.Random(4096)
    p = [rng.choice([-1, 1]) * rng.randint(1, 9) for _ in range(4097)]
    a, b = Dy(0, 0), Dy(1, 0)  # (0, 1): small operands keep the oracle to seconds
    got = upoly.variations_batch(p, [(a, b)])[0]
    assert got == oracle.variations_on(p, a.man, a.exp, b.man, b.exp)


def test_isolate_degree_8192(curvekit_mod):
    """x^8193 - x: roots -1, 0, 1 (the Descartes tests at degree 8192 take the
    direct mode), each isolated in an interval that contains it."""
    from fractions import Fraction
    from paper_1201_1548_b200 import upoly
    p = [0, -1] + [0] * 8191 + [1]
    roots = upoly.descartes_isolate(p)
    assert len(roots) == 3
    for r, want in zip(roots, (-1, 0, 1)):
        iv = r.interval
        lo, hi = iv.lo.as_fraction(), iv.hi.as_fraction()
        assert lo <= Fraction(want) <= hi


def test_interpolate_consecutive_points_vs_oracle(oracle_mod):
    """Points x_0, x_0 + 1, ... take the forward-difference path of k_interp_points
    (the reference's t = 0, 1, 2, ... of modular_subres_profile)."""
    from paper_1201_1548_b200.modpoly import zp_interpolate_batch
    rng = random.Random(21)
    probs = []
    for n, x0, p in ((2, 0, 7), (3, 5, 101), (700, 0, 1073692673), (1301, 123456, 2147483629), (257, 1000, 1009)):
        probs.append((list(range(x0, x0 + n)), [rng.randrange(p) for _ in range(n)], p))
    got = zp_interpolate_batch(probs)
    for (pts, vals, p), c in zip(probs, got):
        assert c == oracle_mod.zp_interp(pts, vals, p)

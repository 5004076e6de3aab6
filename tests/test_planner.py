"""Host planner (CPU): bounds, point counts, prime choice, limb packing."""

import random

import numpy as np

import planner_ref
from conftest import ints_in, load_golden, terms_in
from paper_1201_1548_b200 import planner, workmodel
from paper_1201_1548_b200.bivpoly import BivPoly
from paper_1201_1548_b200.primes30 import NTT_LOG2, PRIMES30


def _cases(small):
    for case in small["random50"]:
        f, g = BivPoly(terms_in(case["f"])), BivPoly(terms_in(case["g"]))
        yield f, g, ints_in(case["res_y"])
        yield f.swap(), g.swap(), ints_in(case["res_x"])


def test_bounds_and_point_counts_are_valid(small):
    n = 0
    for f, g, res in _cases(small):
        fc, gc = f.coeffs_wrt_y(), g.coeffs_wrt_y()
        if len(fc) < 2 or len(gc) < 2:
            continue
        b = planner_ref.det_coeff_bound(fc, gc)
        assert b <= planner_ref.det_coeff_bound_ref(fc, gc)
        assert all(abs(c) <= b for c in res)
        N = planner.point_count(fc, gc, f.deg_x(), g.deg_x(), f.total_degree(), g.total_degree())
        assert len(res) <= N
        n += 1
    assert n > 50


def test_bezout_point_count_is_tight_for_dense_inputs():
    from paper_1201_1548_b200.synth import make_pair
    f, g = (BivPoly(t) for t in make_pair("cfg4", 0))
    fc, gc = f.coeffs_wrt_y(), g.coeffs_wrt_y()
    assert planner.point_count(fc, gc, f.deg_x(), g.deg_x(), 40, 40) == 40 * 40 + 1  # reference: 3201


def test_golden_big_results_within_bounds():
    from paper_1201_1548_b200.synth import make_pair
    for cfg, name in (("cfg2", "cfg2_seed0.json.gz"), ("cfg3", "cfg3_seed0.json.gz")):
        gold = load_golden(name)
        res = [int(c, 16) for c in gold["res"]]
        f, g = (BivPoly(t) for t in make_pair(cfg, 0))
        fc, gc = f.coeffs_wrt_y(), g.coeffs_wrt_y()
        b = planner_ref.det_coeff_bound(fc, gc)
        assert max(abs(c) for c in res) <= b
        plan = planner.plan_resultant(fc, gc, f.total_degree(), g.total_degree(), f.deg_x(), g.deg_x())
        mod = 1
        for p in plan.primes.tolist():
            mod *= p
        assert mod > 4 * b and plan.N >= len(res)
        assert (mod.bit_length() + 31) // 32 == plan.LW


def test_prime_table_properties():
    assert len(PRIMES30) > 3000
    seen = set()
    for p, g in PRIMES30[:400]:
        assert (1 << 29) < p < (1 << 30) and (p - 1) % (1 << NTT_LOG2) == 0
        assert pow(g, (p - 1) // 2, p) == p - 1  # a generator is a non-residue
        assert p not in seen
        seen.add(p)


def _factor_small(n):
    fs, d = set(), 2
    while d * d <= n:
        while n % d == 0:
            fs.add(d)
            n //= d
        d += 1 if d == 2 else 2
    if n > 1:
        fs.add(n)
    return fs


def test_prime_table_generators_are_primitive_roots():
    """The geometric point plan needs g of order exactly p - 1 (distinct points
    g^u for u < p - 1, and w = g^((p-1)/8) a primitive 8th root): g^((p-1)/q) != 1
    for every prime q | p - 1, over the whole table (p - 1 = 2^14 m, m < 2^16)."""
    from paper_1201_1548_b200.modpoly import _is_prime
    for p, g in PRIMES30:
        assert _is_prime(p)
        for q in _factor_small(p - 1):
            assert pow(g, (p - 1) // q, p) != 1, (p, g, q)


def test_product_prime_table_and_stream_match_reference(small):
    """The product's restated prime_table / prime_stream (modpoly.py:31-73)
    against the reference's recorded table and seeded streams."""
    from paper_1201_1548_b200 import modpoly
    pt = small["prime_table"]
    t = modpoly.prime_table()
    assert len(t) == pt["count"] and list(t[:8]) == pt["first"] and list(t[-8:]) == pt["last"]
    assert list(modpoly.prime_stream(0))[:8] == pt["stream0_8"]
    assert list(modpoly.prime_stream(7))[:8] == pt["stream7_8"]


def test_choose_primes_skips_vanishing_leading_coefficients():
    p0, p1 = PRIMES30[0][0], PRIMES30[1][0]
    primes, gens, mod = planner_ref.choose_primes(10 ** 30, [p0 * 7, p0], [1], 0)
    assert p0 not in primes and p1 == primes[0]
    assert mod > 4 * 10 ** 30


def test_pack_grid_roundtrip():
    rng = random.Random(4)
    for bits in (5, 40, 62, 63, 64, 200):
        fc = [[rng.randint(-2 ** bits, 2 ** bits) for _ in range(rng.randint(0, 6))] for _ in range(4)]
        gc = [[rng.randint(-2 ** bits, 2 ** bits) for _ in range(rng.randint(0, 6))] for _ in range(3)]
        fc = [[c for c in col] for col in fc]
        for col in fc + gc:
            while col and col[-1] == 0:
                col.pop()
        fc[-1] = fc[-1] or [1]
        gc[-1] = gc[-1] or [1]
        pk = planner.pack_grid(fc, gc)
        vals = planner.limbs_to_ints(pk.limbs, pk.C, pk.L)
        pos = 0
        for cs, dx in ((fc, pk.dfx), (gc, pk.dgx)):
            for col in cs:
                row = vals[pos:pos + dx + 1]
                assert row[:len(col)] == col and not any(row[len(col):])
                pos += dx + 1
        assert list(pk.degs) == [len(c) - 1 for c in fc] + [len(c) - 1 for c in gc]


def test_limb_roundtrip():
    rng = random.Random(5)
    vals = [rng.randint(-2 ** 500, 2 ** 500) for _ in range(100)] + [0, -1, 1, 2 ** 31, -2 ** 31]
    limbs, L = planner.ints_to_limbs(vals)
    assert planner.limbs_to_ints(limbs, len(vals), L) == vals
    assert limbs.dtype == np.uint32


def test_work_model():
    # m = n = 2: first remainder one step of nominal degree 2 (4 products),
    # then one fused remainder with divisor degree 1 (3 products)
    assert workmodel.elim_products(2, 2) == 4 + 3
    assert workmodel.elim_products(1, 1) == 2
    assert workmodel.elim_products(40, 40) == 80 + 3 * 780
    assert workmodel.elim_products(24, 23) == 2 * 24 + 2 * 23 + 3 * (22 * 23 // 2)
    assert workmodel.eval_products([0, 1, 2], [3, -1]) == 6
    d = 40
    degs = [d - j for j in range(d + 1)]
    assert workmodel.eval_products(degs, degs) == d * (d + 1)


def test_log2_bound_matches_exact_bound():
    import math
    rng = random.Random(3)
    for _ in range(300):
        m, n = rng.randint(1, 9), rng.randint(1, 9)
        fc = [[rng.randint(-2 ** rng.randint(1, 80), 2 ** 80) for _ in range(rng.randint(1, 5))] for _ in range(m + 1)]
        gc = [[rng.randint(-2 ** rng.randint(1, 80), 2 ** 80) for _ in range(rng.randint(1, 5))] for _ in range(n + 1)]
        fc[-1] = fc[-1] or [1]
        gc[-1] = gc[-1] or [1]
        exact = math.log2(planner_ref.det_coeff_bound(fc, gc))
        fast = planner.log2_coeff_bound(fc, gc)
        assert exact - 1e-6 <= fast <= exact + 1e-6
        primes, _ = planner.choose_primes_log2(fast, fc[-1], gc[-1])
        mod = 1
        for p in primes:
            mod *= p
        assert mod > 4 * planner_ref.det_coeff_bound(fc, gc)


def test_limbs_roundtrip_c_helper_and_python():
    """ints -> two's-complement limbs -> ints through the C helper (30-bit digit
    repacking) and the pure-Python fallback, 1 to 5,632 bits, signs and edges."""
    import random

    from paper_1201_1548_b200 import planner
    rng = random.Random(5)
    for bits in (1, 5, 29, 30, 31, 32, 33, 59, 60, 61, 63, 64, 65, 100, 3000, 5632):
        vals = [rng.randint(-(2 ** bits), 2 ** bits) for _ in range(200)]
        vals += [0, -1, 1, 2 ** bits - 1, -(2 ** bits), -(2 ** (bits - 1)), 2 ** (bits - 1)]
        L = (bits + 2 + 31) // 32 + 1
        limbs, _ = planner.ints_to_limbs(vals, L)
        assert planner.limbs_to_ints(limbs, len(vals), L) == vals, bits
        saved = planner._ckb_limbs
        planner._ckb_limbs = None
        try:
            assert planner.limbs_to_ints(limbs, len(vals), L) == vals, bits
        finally:
            planner._ckb_limbs = saved


def _pack_both(f, g, swap):
    F, G = (BivPoly(f), BivPoly(g)) if isinstance(f, dict) else (f, g)
    if swap:
        F, G = F.swap(), G.swap()
    fc, gc = F.coeffs_wrt_y(), G.coeffs_wrt_y()
    return planner.pack_terms(f, g, swap), planner.pack_grid(fc, gc), fc, gc, F, G


def test_pack_terms_matches_coeffs_path():
    """The one-pass C packer (host/ckb_limbs.c terms_grid) gives pack_grid's grid
    and plan_resultant's plan, for dicts and BivPoly objects, both variables."""
    if planner._ckb_limbs is None:
        import pytest
        pytest.skip("host helper not built")
    from paper_1201_1548_b200.synth import make_pair
    rng = random.Random(5)
    cases = [make_pair(c, 0) for c in ("cfg1", "cfg2", "cfg4")]
    # limb-boundary magnitudes (the digit repacking and the sign word): +-2^k, +-(2^k - 1), 2^k + 1
    edge = [s * (2 ** k + d) for k in (29, 30, 31, 32, 60, 62, 63, 64, 90, 96) for d in (-1, 0, 1) for s in (1, -1)]
    cases.append(({(i % 5, i // 5): c for i, c in enumerate(edge)}, {(0, 1): 1, (2, 0): -(2 ** 64)}))
    for _ in range(40):
        f, g = {}, {}
        for t in (f, g):
            dx, dy = rng.randint(0, 9), rng.randint(1, 9)
            bits = rng.choice([3, 31, 32, 63, 64, 65, 200])
            for i in range(dx + 1):
                for j in range(dy + 1):
                    if rng.random() < 0.6:
                        t[(i, j)] = rng.randint(-2 ** bits, 2 ** bits)  # zeros included
            t[(rng.randint(0, dx), dy)] = rng.choice([1, -1]) * rng.randint(1, 2 ** bits)
        cases.append((f, g))
    n = 0
    for f, g in cases:
        for swap in (False, True):
            for wrap in (False, True):
                a, b = (BivPoly(f), BivPoly(g)) if wrap else (f, g)
                pk, ref, fc, gc, F, G = _pack_both(a, b, swap)
                if ref.m == 0 or ref.n == 0:
                    continue
                assert pk is not None
                assert (pk.C, pk.L, pk.m, pk.n, pk.dfx, pk.dgx) == (ref.C, ref.L, ref.m, ref.n, ref.dfx, ref.dgx)
                assert np.array_equal(pk.limbs, ref.limbs) and np.array_equal(pk.degs, ref.degs)
                assert (pk.tdf, pk.tdg, pk.lcf, pk.lcg) == (F.total_degree(), G.total_degree(), fc[-1], gc[-1])
                p1 = planner.plan_packed(pk)
                p2 = planner.plan_resultant(fc, gc, F.total_degree(), G.total_degree(), ref.dfx, ref.dgx)
                assert np.array_equal(p1.primes, p2.primes) and (p1.N, p1.LW) == (p2.N, p2.LW)
                assert abs(planner.log2_bound_from_norms(pk.norms[:pk.m + 1], pk.norms[pk.m + 1:])
                           - planner.log2_coeff_bound(fc, gc)) < 1e-9
                n += 1
    assert n > 100


def test_pack_terms_declines_what_it_cannot_read():
    if planner._ckb_limbs is None:
        import pytest
        pytest.skip("host helper not built")
    one = {(0, 1): 1, (0, 0): 2}
    assert planner.pack_terms({(0, 1): 1.5}, one) is None           # non-int coefficient
    assert planner.pack_terms({(0, 1): True}, one) is None          # bool is not a plain int
    assert planner.pack_terms({(-1, 1): 3}, one) is None            # negative exponent
    assert planner.pack_terms({(0, 1): np.int64(3)}, one) is None   # numpy scalar
    assert planner.pack_terms({(0, 1): 10 ** 400}, one) is None     # 1-norm overflows a double
    assert planner.pack_terms({}, one) is None                      # zero polynomial
    assert planner.pack_terms([1, 2], one) is None


def test_host_mod_list_matches_python():
    """The host helper's residues (modular_subres_profile's single-prime
    reduction) equal Python's % for big, negative and edge-case integers."""
    import random as _r
    try:
        from paper_1201_1548_b200.ckb_limbs import mod_list
    except ImportError:
        import pytest
        pytest.skip("host helper not built")
    rng = _r.Random(3)
    xs = [rng.randint(-2 ** 6000, 2 ** 6000) for _ in range(300)] + [0, 1, -1, 2 ** 30, -(2 ** 30), 2 ** 64 - 1]
    for p in (2, 3, 7, 1073692673, 2147483647, 4294967291):
        assert mod_list(xs, p) == [x % p for x in xs]


def test_host_limbs_to_ints_round_trip():
    """The output conversion (digits written straight into the int objects):
    random big ints of both signs and the edge cases of the two's-complement
    sign handling (0, +-1, +-2^k, -2^k exactly, all-ones limbs)."""
    import random as _r
    from paper_1201_1548_b200.planner import ints_to_limbs, limbs_to_ints
    rng = _r.Random(9)
    vals = [rng.randint(-2 ** 5400, 2 ** 5400) for _ in range(200)]
    vals += [0, 1, -1, 2, -2, 2 ** 29, 2 ** 30, -(2 ** 30), 2 ** 31, -(2 ** 31), 2 ** 32 - 1, -(2 ** 32),
             2 ** 64, -(2 ** 64), (1 << 5000) - 1, -(1 << 5000), -(1 << 5000) + 1, 123456789]
    limbs, L = ints_to_limbs(vals)
    assert limbs_to_ints(limbs, len(vals), L) == vals
    limbs, L = ints_to_limbs(vals, L + 3)  # extra sign-extension limbs
    assert limbs_to_ints(limbs, len(vals), L) == vals


def test_host_limbs_to_ints_every_width():
    """The grouped digit extraction (four 30-bit digits per 15 bytes, a bounds-checked
    tail) at every limb count 1..40, values filling the whole width, both signs."""
    import random as _r
    from paper_1201_1548_b200 import planner
    rng = _r.Random(3)
    for L in range(1, 41):
        vals = [0, -1, 1, -(1 << (32 * L - 1)), (1 << (32 * L - 1)) - 1]
        for _ in range(40):
            b = rng.randint(1, 32 * L - 1)
            vals.append(rng.randint(-(1 << b) + 1, (1 << b) - 1))
            vals.append(-(1 << rng.randint(0, 32 * L - 1)))
        buf, _ = planner.ints_to_limbs(vals, L)
        assert planner.limbs_to_ints(buf, len(vals), L) == vals, L


def test_host_limbs_to_ints_split_path():
    """Results of >= 1 M limbs are filled by two threads (host/ckb_limbs.c): the same ints
    as the pure-Python conversion, with both signs and every limb width around the split."""
    import numpy as np
    from paper_1201_1548_b200 import planner
    rng = np.random.default_rng(7)
    N, LW = 8193, 140
    buf = rng.integers(0, 2 ** 32, size=N * LW, dtype=np.uint64).astype(np.uint32)
    buf[5 * LW:6 * LW] = 0                      # zero
    buf[7 * LW:8 * LW] = 0xFFFFFFFF             # -1
    got = planner.limbs_to_ints(buf, N, LW)
    saved = planner._ckb_limbs
    planner._ckb_limbs = None
    try:
        want = planner.limbs_to_ints(buf, N, LW)
    finally:
        planner._ckb_limbs = saved
    assert got == want

"""GPU parity: every entry point against the reference's golden vectors and the oracle.

Bit-exact for everything (integer arithmetic).  Full-size configurations are
checked against committed golden outputs of the unmodified reference (cfg2,
cfg3) and, at cfg4 size, through the specialisation property
res_y(f, g)(a) = res(f(a, y), g(a, y)) modulo independent primes.
"""

import ctypes
import hashlib
import random

import numpy as np
import pytest

from conftest import ints_in, load_golden, terms_in

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mp():
    from paper_1201_1548_b200 import modpoly
    return modpoly


# ---------------------------------------------------------------------------
# bivariate resultant (modpoly.py:348-394)
# ---------------------------------------------------------------------------

def test_known_answers(mp):
    # test_modpoly.py:29-38
    circle = {(2, 0): 1, (0, 2): 1, (0, 0): -1}
    assert mp.biv_resultant(circle, {(0, 1): 2}, "y") == [-4, 0, 4]
    assert mp.biv_resultant({(0, 2): 1, (3, 0): -1}, {(0, 1): 2}, "y") == [0, 0, 0, -4]
    assert mp.biv_resultant(circle, {(0, 1): 1, (1, 0): -1}, "y") == [-1, 0, 2]


def test_golden_resultant_cases(mp, small):
    for case in small["resultant_cases"]:
        got = mp.biv_resultant(terms_in(case["f"]), terms_in(case["g"]), case["var"])
        assert got == ints_in(case["res"]), case


def test_golden_random50_both_directions(mp, small):
    for case in small["random50"]:
        f, g = terms_in(case["f"]), terms_in(case["g"])
        assert mp.biv_resultant(f, g, "y") == ints_in(case["res_y"])
        assert mp.biv_resultant(f, g, "x") == ints_in(case["res_x"])


def test_errors(mp):
    with pytest.raises(ValueError):
        mp.biv_resultant({}, {(0, 1): 1})
    with pytest.raises(ValueError):
        mp.biv_resultant({(0, 1): 1}, {(0, 1): 1}, "z")


def test_random_vs_oracle(mp, oracle_mod):
    rng = random.Random(77)
    for _ in range(40):
        d1, d2 = rng.randint(1, 9), rng.randint(1, 9)
        bits = rng.choice([3, 20, 70, 140])
        f = {(i, j): rng.randint(-2 ** bits, 2 ** bits) for i in range(d1 + 1) for j in range(d1 + 1 - i)
             if rng.random() < 0.7}
        g = {(i, j): rng.randint(-2 ** bits, 2 ** bits) for i in range(d2 + 1) for j in range(d2 + 1 - i)
             if rng.random() < 0.7}
        f = {k: v for k, v in f.items() if v} or {(0, 1): 1}
        g = {k: v for k, v in g.items() if v} or {(1, 1): 1}
        for var in ("y", "x"):
            assert mp.biv_resultant(f, g, var) == oracle_mod.biv_resultant(f, g, var)


def test_wide_coefficients_and_thin_shapes_vs_oracle(mp, oracle_mod):
    """Coefficients of 600-3,000 bits (more than 16 limbs: the reduction's general limb
    loop, in K1 and in the point-scale role), pure-y polynomials (x-degree 0), y-degree 1
    on either side, and very unequal y-degrees, both variables."""
    rng = random.Random(91)
    cases = []
    for bits in (600, 1500, 3000):
        f = {(i, j): rng.randint(-2 ** bits, 2 ** bits) or 1 for i in range(4) for j in range(4 - i)}
        g = {(i, j): rng.randint(-2 ** bits, 2 ** bits) or 1 for i in range(3) for j in range(3 - i)}
        cases.append((f, g))
    cases.append(({(0, j): rng.randint(-99, 99) or 1 for j in range(7)}, {(2, 1): 5, (0, 0): -3}))   # x-degree 0
    cases.append(({(1, 1): 7, (3, 0): 2}, {(i, j): rng.randint(-9, 9) or 1 for i in range(5) for j in range(9)}))
    cases.append(({(i, 1): rng.randint(-2 ** 40, 2 ** 40) or 1 for i in range(12)},
                  {(0, 1): 1, (5, 0): -(2 ** 70)}))                                                  # m = n = 1
    cases.append(({(i, j): rng.randint(-2 ** 20, 2 ** 20) or 1 for i in range(3) for j in range(31)},
                  {(1, 2): 3, (0, 0): 1}))                                                          # 30 vs 2
    for f, g in cases:
        for var in ("y", "x"):
            assert mp.biv_resultant(f, g, var) == oracle_mod.biv_resultant(f, g, var), (len(f), len(g), var)


def test_cfg2_golden(mp):
    from paper_1201_1548_b200.synth import make_pair
    gold = load_golden("cfg2_seed0.json.gz")
    f, g = make_pair("cfg2", 0)
    got = mp.biv_resultant(f, g, "y")
    assert hashlib.sha256(repr(got).encode()).hexdigest()[:16] == gold["sha16_repr"]
    assert got == [int(c, 16) for c in gold["res"]]


def test_cfg3_golden(mp):
    from paper_1201_1548_b200.synth import make_pair
    gold = load_golden("cfg3_seed0.json.gz")
    f, g = make_pair("cfg3", 0)
    got = mp.biv_resultant(f, g, "y")
    assert hashlib.sha256(repr(got).encode()).hexdigest()[:16] == gold["sha16_repr"] == "2273dd0debe66770"
    assert got == [int(c, 16) for c in gold["res"]]
    # the reference's square-free structure: R is square-free, gcd(R, R') = 1
    assert mp.int_gcd_uni(got, [i * c for i, c in enumerate(got)][1:]) == ints_in(gold["gcd_r_dr"])


def _specialisation_check(mp, oracle_mod, f, g, res, rng, trials=6):
    fc, gc = oracle_mod.coeffs_wrt_y(f), oracle_mod.coeffs_wrt_y(g)
    for _ in range(trials):
        q = rng.choice(oracle_mod.prime_table()[100:400])
        a = rng.randrange(q)
        fu = [sum(c * pow(a, i, q) for i, c in enumerate(col)) % q for col in fc]
        gu = [sum(c * pow(a, i, q) for i, c in enumerate(col)) % q for col in gc]
        if fu[-1] == 0 or gu[-1] == 0:
            continue
        want = oracle_mod.zp_resultant(fu, gu, q)
        got = sum(c * pow(a, i, q) for i, c in enumerate(res)) % q
        assert got == want


def test_cfg4_specialisation(mp, oracle_mod):
    from paper_1201_1548_b200.synth import make_pair
    f, g = make_pair("cfg4", 0)
    res = mp.biv_resultant(f, g, "y")
    assert len(res) == 1601
    _specialisation_check(mp, oracle_mod, f, g, res, random.Random(4))


def test_cfg4_full_golden(mp):
    """Every coefficient of the headline configuration, bit for bit, against the
    pinned oracle's full cfg4 resultant (tests/golden/make_oracle_golden.py;
    the fixture itself is tied to the reference by test_oracle.py's
    test_cfg4_full_golden_matches_reference_prime)."""
    from paper_1201_1548_b200.synth import make_pair
    gold = load_golden("cfg4_full.json.gz")
    f, g = make_pair("cfg4", 0)
    got = mp.biv_resultant(f, g, "y")
    assert len(got) - 1 == gold["degree"] == 1600
    assert hashlib.sha256(repr(got).encode()).hexdigest() == gold["sha256_repr"]
    assert got == [int(c, 16) for c in gold["res"]]


def test_cfg5_specialisation(mp, oracle_mod):
    """cfg5 (d = 64, 256-bit): ~1,150 primes x 4,097 points, NTT length 2^14."""
    from paper_1201_1548_b200.synth import make_pair
    f, g = make_pair("cfg5", 0)
    res = mp.biv_resultant(f, g, "y")
    assert len(res) == 64 * 64 + 1
    _specialisation_check(mp, oracle_mod, f, g, res, random.Random(5), trials=4)


def test_cfg3_f_fy_and_x_direction_specialisation(mp, oracle_mod):
    from paper_1201_1548_b200.synth import make_pair
    f, g = make_pair("cfg3", 1)
    swap = lambda t: {(j, i): c for (i, j), c in t.items()}
    res = mp.biv_resultant(f, g, "x")
    _specialisation_check(mp, oracle_mod, swap(f), swap(g), res, random.Random(6), trials=4)


def test_cfg4_one_prime_of_the_reference_loop(mp, oracle_mod):
    """Residues of the GPU result mod the reference's first cfg4 prime equal
    the reference loop body's interpolated polynomial at that prime."""
    from paper_1201_1548_b200.synth import make_pair
    gold = load_golden("cfg4_prime0.json.gz")
    f, g = make_pair("cfg4", 0)
    res = mp.biv_resultant(f, g, "y")
    p = gold["p"]
    assert [c % p for c in res] == gold["poly"] + [0] * (len(res) - len(gold["poly"]))


# ---------------------------------------------------------------------------
# per-prime entry points
# ---------------------------------------------------------------------------

def test_zp_resultant_golden(mp, small):
    batch = [(c["f"], c["g"], c["p"]) for c in small["zp_resultant"]]
    assert mp.zp_resultant_batch(batch) == [c["res"] for c in small["zp_resultant"]]
    p = 7
    f = mp.ModPoly.make([-1, 0, 1], p)
    assert mp.zp_resultant_uni(f, mp.ModPoly.make([-2, 1], p)) == 3
    assert mp.zp_resultant_uni(f, mp.ModPoly.make([5], p)) == pow(5, 2, p)
    assert mp.zp_resultant_uni(f, f) == 0
    with pytest.raises(ValueError):
        mp.zp_resultant_uni(f, mp.ModPoly.make([1], 5))


def test_zp_resultant_random_degrees_vs_oracle(mp, oracle_mod):
    rng = random.Random(8)
    ps = [1073692673, 536952833, 2147483647, 2147483629, 101, 7]
    batch = []
    for _ in range(400):
        p = rng.choice(ps)
        la, lb = rng.randint(1, 65), rng.randint(1, 65)
        a = [rng.randrange(p) if rng.random() < 0.8 else 0 for _ in range(la)]
        b = [rng.randrange(p) if rng.random() < 0.8 else 0 for _ in range(lb)]
        batch.append((a, b, p))
    got = mp.zp_resultant_batch(batch)
    want = [oracle_mod.zp_resultant(a, b, p) for a, b, p in batch]
    assert got == want


def test_zp_interpolate_golden(mp, small):
    for c in small["zp_interpolate"]:
        assert list(mp.zp_interpolate(c["x"], c["v"], c["p"]).coeffs) == c["c"]
    with pytest.raises(ValueError):
        mp.zp_interpolate([1, 1], [0, 0], 5)


def test_crt_golden(mp, small):
    for c in small["crt"]:
        assert mp.crt_reconstruct(mp.ResidueSystem(tuple(c["primes"]), tuple(c["res"]))) == int(c["x"])


@pytest.mark.parametrize("K,extra", [(1, 0), (33, 1), (200, 0), (700, 130)])
def test_crt_lift_roundtrip_large(mp, K, extra):
    """Tensor-core CRT: K primes (chunks of 32, ring of 4 stages), several 128-row tiles."""
    from paper_1201_1548_b200.primes30 import PRIMES30
    rng = random.Random(12 + K)
    primes = [p for p, _ in PRIMES30[:K]]
    M = 1
    for p in primes:
        M *= p
    vals = [rng.randint(-(M // 2) + 1, M // 2) for _ in range(300 + extra)] + [0, 1, -1, M // 2, -(M // 2) + 1]
    # every magnitude: long runs of sign-extension limbs exercise the carry propagation across lanes and chunks
    vals += [s * rng.randint(1, 2 ** b) for b in range(0, M.bit_length() - 2, 23) for s in (-1, 1)]
    vals += [s * (2 ** b - 1) for b in range(1, M.bit_length() - 2, 61) for s in (-1, 1)]
    res = np.array([[v % p for v in vals] for p in primes], dtype=np.uint32)
    assert mp.crt_lift(res, primes) == vals


def test_int_gcd_golden(mp, small):
    for c in small["int_gcd"]:
        assert mp.int_gcd_uni(ints_in(c["f"]), ints_in(c["g"])) == ints_in(c["gcd"]), c


def test_zp_gcd_sylvester_golden(mp, small):
    cases = small["zp_gcd_sylvester"]
    for c in cases[:3]:
        got = mp.zp_gcd_sylvester(mp.ModPoly.make(c["f"], c["p"]), mp.ModPoly.make(c["g"], c["p"]))
        assert list(got.coeffs) == c["gcd"]
    got = mp.zp_gcd_batch([(c["f"], c["g"], c["p"]) for c in cases[3:]])
    for c, gm in zip(cases[3:], got):
        want = c["euclid"] or [1]
        assert (gm if len(gm) > 1 else [1]) == (want if len(want) > 1 else [1])
        assert list(mp.zp_gcd_sylvester(mp.ModPoly.make(c["f"], c["p"]),
                                        mp.ModPoly.make(c["g"], c["p"])).coeffs) == c["gcd"]


def test_reduce_matches_python_mod():
    from paper_1201_1548_b200 import _lib
    from paper_1201_1548_b200.planner import ints_to_limbs
    rng = random.Random(3)
    vals = [rng.randint(-2 ** 300, 2 ** 300) for _ in range(500)] + [0, -1, 2 ** 31, -(2 ** 64)]
    limbs, L = ints_to_limbs(vals)
    primes = np.array([1073692673, 2147483647, 7, 536952833], dtype=np.uint32)
    out = np.empty((4, len(vals)), dtype=np.uint32)
    lib = _lib.lib()
    _lib.check(lib.ckb_reduce(_lib.ptr(limbs), len(vals), L, _lib.ptr(primes), 4, _lib.ptr(out)), "reduce")
    for k, p in enumerate(primes.tolist()):
        assert out[k].tolist() == [v % p for v in vals]


def test_geometric_interpolation_roundtrip():
    """values at the planned points x_t = q^t interpolate back to the polynomial."""
    from paper_1201_1548_b200 import _lib
    from paper_1201_1548_b200.primes30 import PRIMES30
    rng = random.Random(5)
    lib = _lib.lib()
    for N in (1, 2, 3, 17, 300, 1601):
        K = 3
        primes = np.array([p for p, _ in PRIMES30[10:10 + K]], dtype=np.uint32)
        gens = np.array([g for _, g in PRIMES30[10:10 + K]], dtype=np.uint32)
        pts = np.empty((K, N), dtype=np.uint32)
        _lib.check(lib.ckb_interp_plan_points(_lib.ptr(primes), _lib.ptr(gens), K, N, _lib.ptr(pts)), "plan")
        polys = [[rng.randrange(int(p)) for _ in range(N)] for p in primes.tolist()]
        vals = np.empty((K, N), dtype=np.uint32)
        for k, p in enumerate(primes.tolist()):
            assert pts[k, 0] == 1 and len(set(pts[k].tolist())) == N
            for t in range(N):
                x = int(pts[k, t])
                acc = 0
                for c in reversed(polys[k]):
                    acc = (acc * x + c) % p
                vals[k, t] = acc
        out = np.empty((K, N), dtype=np.uint32)
        _lib.check(lib.ckb_interp_geometric(_lib.ptr(vals), _lib.ptr(primes), _lib.ptr(gens), K, N,
                                            _lib.ptr(out)), "interp")
        for k in range(K):
            assert out[k].tolist() == polys[k], N


# ---------------------------------------------------------------------------
# modular subresultant degree profiles (modpoly.py:428-474)
# ---------------------------------------------------------------------------

def test_subres_profile_golden(mp, small):
    # test_modpoly.py:218-261 cases plus random f, f_y pairs, reference outputs
    for c in small["subres_profile"]:
        pr = mp.modular_subres_profile(terms_in(c["f"]), terms_in(c["g"]), ints_in(c["rstar"]), c["p"])
        assert pr.prime == c["p"]
        assert list(pr.chain_degrees) == c["chain"], c
        assert list(pr.factor_degrees) == c["d"], c


def test_subres_profile_unlucky(mp):
    circle = {(2, 0): 1, (0, 2): 1, (0, 0): -1}
    # leading y-coefficient 3 vanishes mod 3 (modpoly.py:437-439)
    with pytest.raises(mp.UnluckyPrime):
        mp.modular_subres_profile({(0, 2): 3, (0, 0): -1, (1, 0): 1}, {(0, 1): 6}, [1, 1], 3)
    # rstar drops degree mod p (modpoly.py:462-463)
    with pytest.raises(mp.UnluckyPrime):
        mp.modular_subres_profile(circle, {(0, 1): 2}, [-1, 0, 7], 7)


def test_cfg3_subres_profile_golden(mp):
    """The reference's 82 s profile of cfg3 (R square-free: chain 552, 0, ...)."""
    from paper_1201_1548_b200.synth import make_pair
    gold = load_golden("cfg3_seed0.json.gz")
    f, g = make_pair("cfg3", 0)
    res = [int(c, 16) for c in gold["res"]]
    content = int(gold["sqf_content"])
    assert all(c % content == 0 for c in res)
    rstar = [c // content for c in res]
    pr = mp.modular_subres_profile(f, g, rstar, gold["profile"]["p"])
    assert list(pr.chain_degrees) == gold["profile"]["chain"]
    assert list(pr.factor_degrees) == gold["profile"]["d"]


def test_graph_replay_and_reallocation(mp):
    """Repeated calls replay a captured CUDA graph; a larger problem in between
    reallocates the work buffers (dropping the graph) and results stay exact."""
    from paper_1201_1548_b200.synth import make_pair
    f2, g2 = make_pair("cfg2", 0)
    want2 = mp.biv_resultant(f2, g2, "y")
    small = [({(2, 0): 1, (0, 2): 1, (0, 0): -1}, {(0, 1): 1, (1, 0): -1}, [-1, 0, 2])]
    for _ in range(4):
        assert mp.biv_resultant(f2, g2, "y") == want2
    f3, g3 = make_pair("cfg3", 0)
    want3 = mp.biv_resultant(f3, g3, "y")
    for _ in range(3):
        assert mp.biv_resultant(f3, g3, "y") == want3
        assert mp.biv_resultant(f2, g2, "y") == want2
        for f, g, r in small:
            assert mp.biv_resultant(f, g, "y") == r


def test_sparse_structured_vs_oracle(mp, oracle_mod):
    """Sparse inputs whose remainder sequences skip degrees at every point: all
    images take the general (warp, _zp_resultant restatement) kernel."""
    rng = random.Random(31)
    cases = [
        ({(0, 6): 1, (1, 3): 1, (2, 0): 1, (0, 0): 1}, {(0, 4): 1, (3, 1): 1, (0, 0): 2}),
        ({(0, 8): 3, (2, 4): -5, (4, 0): 7}, {(0, 6): 1, (1, 2): 2, (5, 0): -1}),
        ({(0, 5): 1, (3, 0): -1}, {(0, 3): 2, (1, 0): 1}),
        ({(0, 10): 1, (1, 5): 1, (0, 0): -1}, {(0, 10): 2, (3, 0): 1}),
    ]
    for _ in range(6):  # random sparse: few terms, large gaps
        f = {(rng.randint(0, 6), rng.randint(0, 9)): rng.randint(-2 ** 40, 2 ** 40) for _ in range(4)}
        g = {(rng.randint(0, 6), rng.randint(0, 9)): rng.randint(-2 ** 40, 2 ** 40) for _ in range(4)}
        f[(0, 9)] = 1
        g[(0, 7)] = -3
        cases.append(({k: v for k, v in f.items() if v}, {k: v for k, v in g.items() if v}))
    for f, g in cases:
        for var in ("y", "x"):
            assert mp.biv_resultant(f, g, var) == oracle_mod.biv_resultant(f, g, var), (f, g, var)


def test_degenerate_branches(mp):
    # m = 0 or n = 0 (modpoly.py:363-369) and a zero resultant (common factor)
    assert mp.biv_resultant({(2, 0): 3}, {(1, 0): 2}, "y") == [1]
    assert mp.biv_resultant({(2, 0): 3, (0, 0): 1}, {(0, 2): 1, (1, 0): 1}, "y") == [1, 0, 6, 0, 9]
    assert mp.biv_resultant({(0, 2): 1, (1, 0): 1}, {(1, 0): 2}, "y") == [0, 0, 4]
    common = {(0, 1): 1, (1, 0): -1}
    f = {(0, 2): 1, (1, 1): -1}            # y (y - x)
    g = {(0, 1): 1, (1, 0): -1}  # y - x
    assert mp.biv_resultant(f, g, "y") == []
    assert mp.biv_resultant(common, common, "x") == []


def test_high_y_degree_general_path(mp, oracle_mod):
    """y-degrees beyond the register kernel's buckets (> 64) run every image
    through the general warp kernel; large univariate resultants likewise."""
    rng = random.Random(41)
    f = {(0, 70): 1, (1, 35): rng.randint(-99, 99), (3, 0): rng.randint(1, 99), (0, 12): -5}
    g = {(0, 66): 3, (2, 1): rng.randint(-99, 99), (0, 0): 7}
    assert mp.biv_resultant(f, g, "y") == oracle_mod.biv_resultant(f, g, "y")
    # x-degree 80 as the resultant variable's partner: res_x swaps the roles
    h = {(80, 0): 1, (0, 2): 1, (7, 1): -2}
    k = {(75, 0): 2, (0, 1): 1, (1, 0): 1}
    assert mp.biv_resultant(h, k, "x") == oracle_mod.biv_resultant(h, k, "x")
    p = oracle_mod.prime_table()[0]
    a = [rng.randrange(p) for _ in range(150)]
    b = [rng.randrange(p) for _ in range(121)]
    a[-1] = a[-1] or 1
    b[-1] = b[-1] or 1
    assert mp.zp_resultant_uni(mp.ModPoly.make(a, p), mp.ModPoly.make(b, p)) == oracle_mod.zp_resultant(a, b, p)


def test_interpolate_large_batch(mp):
    """Newton interpolation with batched inverses: 5,000 points and a batch of
    mixed sizes, checked by evaluating the result back at the points."""
    from paper_1201_1548_b200.primes30 import PRIMES30
    rng = random.Random(8)
    probs = []
    for n, p in ((5000, PRIMES30[3][0]), (1, 1000003), (2, 7), (300, 2147483647), (1500, PRIMES30[9][0])):
        pts = rng.sample(range(p), n)
        vals = [rng.randrange(p) for _ in range(n)]
        probs.append((pts, vals, p))
    outs = mp.zp_interpolate_batch(probs)
    for (pts, vals, p), co in zip(probs, outs):
        assert len(co) <= len(pts)
        for x, v in zip(pts[:200], vals[:200]):
            acc = 0
            for c in reversed(co):
                acc = (acc * x + c) % p
            assert acc == v


def test_biv_resultant_batch_golden(mp, small):
    """several res problems per library call (own streams),
    identical to the reference's results; degenerate and mixed-size entries."""
    from paper_1201_1548_b200 import _lib
    probs, want = [], []
    for case in small["random50"][:24]:
        f, g = terms_in(case["f"]), terms_in(case["g"])
        probs += [(f, g, "y"), (f, g, "x")]
        want += [ints_in(case["res_y"]), ints_in(case["res_x"])]
    for case in small["resultant_cases"]:
        probs.append((terms_in(case["f"]), terms_in(case["g"]), case["var"]))
        want.append(ints_in(case["res"]))
    n0 = _lib.launch_count()
    for rep in range(2):  # second pass replays the per-slot graphs
        assert mp.biv_resultant_batch(probs) == want
    assert _lib.launch_count() > n0
    # a cfg2-size problem next to tiny ones in one call
    from paper_1201_1548_b200.synth import make_pair
    f2, g2 = make_pair("cfg2", 0)
    gold = load_golden("cfg2_seed0.json.gz")
    circle = {(2, 0): 1, (0, 2): 1, (0, 0): -1}
    got = mp.biv_resultant_batch([(circle, {(0, 1): 2}, "y"), (f2, g2, "y"), (circle, {(0, 1): 1, (1, 0): -1}, "y")])
    assert got[0] == [-4, 0, 4] and got[2] == [-1, 0, 2]
    assert got[1] == [int(c, 16) for c in gold["res"]]
    with pytest.raises(ValueError):
        mp.biv_resultant_batch([(circle, {}, "y")])


def test_int_gcd_uni_batch_golden(mp, small):
    cases = small["int_gcd"]
    got = mp.int_gcd_uni_batch([(ints_in(c["f"]), ints_in(c["g"])) for c in cases])
    assert got == [ints_in(c["gcd"]) for c in cases]


def test_point_scale_when_leading_coefficient_vanishes_at_roots_of_unity(mp, oracle_mod):
    """lc_y(f) = x^8 - 1 vanishes at the first coset {w^j} of every prime's planned
    points, so every prime must shift its point set (c != 1; the reference skips such
    points, modpoly.py:380-390).  Also with lc_y(g) = x^16 - 1 and a constant lc."""
    rng = random.Random(17)
    for lcf, lcg in (([-1] + [0] * 7 + [1], [3]), ([-1] + [0] * 7 + [1], [-1] + [0] * 15 + [1]),
                     ([5], [-1] + [0] * 15 + [1])):
        for my, ny in ((6, 5), (12, 12)):
            f = {(i, j): rng.randint(-999, 999) for j in range(my) for i in range(10)}
            g = {(i, j): rng.randint(-999, 999) for j in range(ny) for i in range(7)}
            f.update({(i, my): c for i, c in enumerate(lcf) if c})
            g.update({(i, ny): c for i, c in enumerate(lcg) if c})
            f = {k: v for k, v in f.items() if v}
            g = {k: v for k, v in g.items() if v}
            assert mp.biv_resultant(f, g, "y") == oracle_mod.biv_resultant(f, g, "y")


def test_c_abi_rejects_bad_arguments():
    """The C-ABI validates its inputs: bad sizes, handles and shapes return < 0
    with a message (no device work, no crash), and the library stays usable."""
    from paper_1201_1548_b200 import _lib
    lib = _lib.lib()
    z = np.zeros(16, dtype=np.uint32)
    d = np.zeros(16, dtype=np.int16)
    primes = np.array([1000000007], dtype=np.uint32)
    st = np.zeros(4, dtype=np.uint32)
    # C does not match (m+1)(dfx+1) + (n+1)(dgx+1)
    rc = lib.ckb_biv_resultant(_lib.ptr(z), 5, 1, _lib.ptr(d), 1, 1, 1, 1, _lib.ptr(primes), _lib.ptr(primes), 1, 4,
                               1, _lib.ptr(z), _lib.ptr(st), None)
    assert rc < 0 and b"C mismatch" in lib.ckb_last_error()
    # an even "prime"
    bad = np.array([1000000008], dtype=np.uint32)
    assert lib.ckb_reduce(_lib.ptr(z), 1, 1, _lib.ptr(bad), 1, _lib.ptr(z)) < 0
    # unknown Descartes handle, batch of zero intervals
    v = np.zeros(4, dtype=np.int32)
    lds = np.zeros(4, dtype=np.int32)
    assert lib.ckb_descartes_variations_batch(12345, _lib.ptr(z), 1, _lib.ptr(lds), 1, 1, 1, _lib.ptr(v)) < 0
    # bivariate gcd images need m >= n
    od = np.zeros(16, dtype=np.int32)
    assert lib.ckb_biv_gcd_images(_lib.ptr(z), 5, 1, _lib.ptr(d), 0, 1, 1, 1, 0, _lib.ptr(primes), 1, 2,
                                  _lib.ptr(z), 2, _lib.ptr(od)) < 0
    # batched resultants: 0 or more than 4 problems
    ptrs = (ctypes.c_void_p * 1)(None)
    ints = np.zeros(8, dtype=np.int32)
    assert lib.ckb_biv_resultant_batch(0, ptrs, _lib.ptr(ints), _lib.ptr(ints), ptrs, _lib.ptr(ints), _lib.ptr(ints),
                                       _lib.ptr(ints), _lib.ptr(ints), ptrs, ptrs, _lib.ptr(ints), _lib.ptr(ints),
                                       _lib.ptr(ints), ptrs, _lib.ptr(st)) < 0
    # still usable afterwards
    from paper_1201_1548_b200 import modpoly
    assert modpoly.biv_resultant({(2, 0): 1, (0, 2): 1, (0, 0): -1}, {(0, 1): 2}) == [-4, 0, 4]


def test_structured_even_y_inputs(mp, oracle_mod):
    """f = F(x, y^2), g = G(x, y^2): every image's remainder sequence drops the
    degree by two (non-generic), so the images take the general path; small sizes
    against the oracle, the 'sparse' bench configuration (d = 40) by specialisation."""
    from paper_1201_1548_b200.synth import make_pair, random_even_terms
    rng = random.Random(12)
    for d, bits in ((6, 10), (10, 40), (14, 64)):
        f, g = random_even_terms(rng, d, bits), random_even_terms(rng, d, bits)
        for var in ("y", "x"):
            assert mp.biv_resultant(f, g, var) == oracle_mod.biv_resultant(f, g, var)
    f, g = make_pair("sparse", 0)
    res = mp.biv_resultant(f, g, "y")
    _specialisation_check(mp, oracle_mod, f, g, res, random.Random(40), trials=4)


def test_cfg5_full_golden(mp):
    """cfg5 (d = 64, 256-bit, ~1,100 primes): the whole resultant against the pinned
    oracle's (tests/golden/make_oracle_golden.py, 30 min on 8 threads): sha256 of
    repr(R), degree, bit length, and R modulo three 61-bit primes."""
    from paper_1201_1548_b200.synth import make_pair
    gold = load_golden("cfg5_full.json.gz")
    f, g = make_pair("cfg5", 0)
    got = mp.biv_resultant(f, g, "y")
    assert len(got) - 1 == gold["degree"] == 4096
    assert max(abs(c).bit_length() for c in got) == gold["max_bits"]
    for q, want in gold["mod_fingerprint"].items():
        assert [c % int(q) for c in got] == want
    assert hashlib.sha256(repr(got).encode()).hexdigest() == gold["sha256_repr"]

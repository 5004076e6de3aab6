"""Generate golden fixtures by running the UNMODIFIED reference (curvekit).

Runs only in the build container, where the reference is importable from
/root/reference/pkg/src (read-only).  The fixtures it writes are committed so
that the GPU box, where /root/reference does not exist, can check parity.

    python tests/golden/make_golden.py small      # seconds
    python tests/golden/make_golden.py cfg1       # ~10 s (Bisolve end to end)
    python tests/golden/make_golden.py cfg2       # ~3 min
    python tests/golden/make_golden.py cfg3       # ~12 min (+ Yun, gcd, profile)
    python tests/golden/make_golden.py cfg4prime  # ~1 min (one prime of cfg4)
    python tests/golden/make_golden.py descartes  # Descartes tests of real-root isolation

Every fixture records which reference function produced it (file:line).
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import random
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.path[:0] = [REF_SRC, REF_TESTS, REPO]

from curvekit import upoly  # noqa: E402
from curvekit import modpoly as M  # noqa: E402
from curvekit.bivpoly import BivPoly  # noqa: E402

from paper_1201_1548_b200.synth import make_pair  # noqa: E402


def terms_out(t):
    if isinstance(t, BivPoly):
        t = t.terms
    return [[i, j, str(c)] for (i, j), c in sorted(t.items())]


def ints_out(xs):
    return [str(int(x)) for x in xs]


def sha16(obj) -> str:
    return hashlib.sha256(repr(obj).encode()).hexdigest()[:16]


def dump(name, obj, gz=False):
    path = os.path.join(HERE, name + (".json.gz" if gz else ".json"))
    data = json.dumps(obj, separators=(",", ":")).encode()
    if gz:
        with gzip.open(path, "wb", compresslevel=9) as fh:
            fh.write(data)
    else:
        with open(path, "wb") as fh:
            fh.write(data)
    print("wrote", path, len(data), "bytes")


def _random_total_degree(rng, dmax, bits):
    # pkg/tests/test_modpoly.py:51-62
    d = rng.randint(1, dmax)
    terms = {}
    for i in range(d + 1):
        for j in range(d + 1 - i):
            if rng.random() < 0.6:
                c = rng.randint(-(2**bits), 2**bits)
                if c:
                    terms[(i, j)] = c
    if not terms:
        terms[(0, 1)] = 1
    return BivPoly(terms)


def gen_small():
    from oracles import int_det, resultant_oracle_y  # pkg/tests/oracles.py
    out = {"source": "curvekit (pkg/src/curvekit/modpoly.py, upoly.py) run unmodified"}

    circle = BivPoly({(2, 0): 1, (0, 2): 1, (0, 0): -1})
    line = BivPoly({(0, 1): 1, (1, 0): -1})
    fy = BivPoly({(0, 1): 2})
    cusp = BivPoly({(0, 2): 1, (3, 0): -1})
    res_cases = []
    # known answers, test_modpoly.py:29-38
    for f, g, var in [(circle, fy, "y"), (cusp, fy, "y"), (circle, line, "y"),
                      (circle, line, "x"), (circle, fy, "x"), (cusp, cusp.diff("y"), "y"),
                      (cusp, cusp.diff("x"), "x")]:
        res_cases.append({"f": terms_out(f), "g": terms_out(g), "var": var,
                          "res": ints_out(M.biv_resultant(f, g, var))})
    # degenerate branches modpoly.py:363-369
    for f, g in [(BivPoly({(2, 0): 3, (0, 0): 1}), BivPoly({(1, 0): 2, (0, 0): -1})),
                 (BivPoly({(2, 0): 3, (0, 0): 1}), circle),
                 (circle, BivPoly({(1, 0): 5, (0, 0): 7}))]:
        res_cases.append({"f": terms_out(f), "g": terms_out(g), "var": "y",
                          "res": ints_out(M.biv_resultant(f, g, "y"))})
    # common factor -> [] (test_bisolve.py:48-53)
    f, g = circle * line, circle * fy
    res_cases.append({"f": terms_out(f), "g": terms_out(g), "var": "y",
                      "res": ints_out(M.biv_resultant(f, g, "y"))})
    # sparse structured inputs that break pivot-free elimination at every point
    for f, g in [(BivPoly({(0, 4): 1, (1, 0): 1}), BivPoly({(0, 2): 1, (0, 0): 1})),
                 (BivPoly({(0, 5): 1, (2, 1): -3, (0, 0): 1}), BivPoly({(0, 3): 1, (1, 0): 1})),
                 (BivPoly({(0, 3): 2, (1, 1): 1}), BivPoly({(1, 2): 1, (0, 0): -1})),
                 (BivPoly({(1, 2): 1, (0, 0): 1}), BivPoly({(2, 1): 1, (1, 0): -1}))]:
        for var in ("y", "x"):
            res_cases.append({"f": terms_out(f), "g": terms_out(g), "var": var,
                              "res": ints_out(M.biv_resultant(f, g, var))})
    out["resultant_cases"] = res_cases

    # 50 random pairs vs the Bareiss oracle, test_modpoly.py:41-48
    rng = random.Random(11)
    rand = []
    for _ in range(50):
        f = _random_total_degree(rng, 5, 10)
        g = _random_total_degree(rng, 5, 10)
        if f.deg_y() < 0 or g.deg_y() < 0:
            continue
        r = M.biv_resultant(f, g, "y")
        assert r == resultant_oracle_y(f, g)
        rx = M.biv_resultant(f, g, "x")
        rand.append({"f": terms_out(f), "g": terms_out(g), "res_y": ints_out(r),
                     "res_x": ints_out(rx)})
    out["random50"] = rand

    # zp_resultant_uni examples + 40 random vs int_det, test_modpoly.py:114-141
    p = M.prime_table()[0]
    zr = []
    rng = random.Random(5)
    for _ in range(40):
        fa = [rng.randint(-9, 9) for _ in range(rng.randint(2, 6))]
        gb = [rng.randint(-9, 9) for _ in range(rng.randint(2, 6))]
        fa[-1] = fa[-1] or 1
        gb[-1] = gb[-1] or 1
        m, n = len(fa) - 1, len(gb) - 1
        size = m + n
        rows = []
        for i in range(n):
            rows.append([0] * i + list(reversed(fa)) + [0] * (size - m - 1 - i))
        for i in range(m):
            rows.append([0] * i + list(reversed(gb)) + [0] * (size - n - 1 - i))
        want = int_det(rows) % p
        got = M.zp_resultant_uni(M.ModPoly.make(fa, p), M.ModPoly.make(gb, p))
        assert got == want
        zr.append({"p": p, "f": fa, "g": gb, "res": got})
    # random residue pairs of mixed degree (exercise degree drops)
    rng = random.Random(55)
    for _ in range(200):
        p = rng.choice(M.prime_table()[:16] + (7, 13, 101))
        fa = [rng.randrange(p) if rng.random() < 0.7 else 0 for _ in range(rng.randint(1, 12))]
        gb = [rng.randrange(p) if rng.random() < 0.7 else 0 for _ in range(rng.randint(1, 12))]
        fa[-1] = fa[-1] or 1
        gb[-1] = gb[-1] or 1
        zr.append({"p": p, "f": fa, "g": gb,
                   "res": M.zp_resultant_uni(M.ModPoly.make(fa, p), M.ModPoly.make(gb, p))})
    out["zp_resultant"] = zr

    # interpolation, test_modpoly.py:144-149 + random
    zi = [{"p": 5, "x": [0, 1], "v": [1, 2], "c": [1, 1]},
          {"p": 7, "x": [3], "v": [4], "c": [4]},
          {"p": 7, "x": [0, 1, 2], "v": [0, 1, 4], "c": [0, 0, 1]}]
    rng = random.Random(66)
    for _ in range(30):
        p = rng.choice(M.prime_table()[:8])
        n = rng.randint(1, 60)
        xs = rng.sample(range(0, 400), n)
        vs = [rng.randrange(p) for _ in range(n)]
        zi.append({"p": p, "x": xs, "v": vs,
                   "c": list(M.zp_interpolate(xs, vs, p).coeffs)})
    out["zp_interpolate"] = zi

    # CRT, test_modpoly.py:152-168
    crt = [{"primes": [5, 7], "res": [2, 3], "x": "17"},
           {"primes": [101], "res": [100], "x": "-1"},
           {"primes": [5, 7, 11], "res": [0, 0, 0], "x": "0"}]
    rng = random.Random(2)
    primes = M.prime_table()[:6]
    Mod = 1
    for q in primes:
        Mod *= q
    for _ in range(50):
        v = rng.randint(-(Mod // 2) + 1, Mod // 2)
        rs = M.ResidueSystem(tuple(primes), tuple(v % q for q in primes))
        assert M.crt_reconstruct(rs) == v
        crt.append({"primes": list(primes), "res": [v % q for q in primes], "x": str(v)})
    out["crt"] = crt

    # int_gcd_uni examples + planted factors, test_modpoly.py:171-186
    gcds = [{"f": ["-1", "0", "1"], "g": ["1", "-2", "1"],
             "gcd": ints_out(M.int_gcd_uni([-1, 0, 1], [1, -2, 1]))},
            {"f": ["2", "4"], "g": [], "gcd": ints_out(M.int_gcd_uni([2, 4], []))},
            {"f": ["0", "1"], "g": ["-1", "1"], "gcd": ints_out(M.int_gcd_uni([0, 1], [-1, 1]))}]
    rng = random.Random(9)
    for _ in range(40):
        common = [rng.randint(-5, 5) for _ in range(rng.randint(1, 3))] + [rng.randint(1, 5)]
        f = upoly.mul(common, [rng.randint(-9, 9) for _ in range(2)] + [rng.randint(1, 9)])
        g = upoly.mul(common, [rng.randint(-9, 9) for _ in range(3)] + [rng.randint(1, 9)])
        gcds.append({"f": ints_out(f), "g": ints_out(g), "gcd": ints_out(M.int_gcd_uni(f, g))})
    # larger planted factors with big coefficients
    rng = random.Random(99)
    for _ in range(20):
        common = [rng.randint(-2**40, 2**40) for _ in range(rng.randint(1, 12))] + [rng.randint(1, 2**40)]
        f = upoly.mul(common, [rng.randint(-2**30, 2**30) for _ in range(rng.randint(1, 20))] + [1])
        g = upoly.mul(common, [rng.randint(-2**30, 2**30) for _ in range(rng.randint(1, 20))] + [3])
        gcds.append({"f": ints_out(f), "g": ints_out(g), "gcd": ints_out(M.int_gcd_uni(f, g))})
    out["int_gcd"] = gcds

    # zp_gcd_sylvester, test_modpoly.py:189-215
    syl = []
    for p, fa, gb in [(5, [-1, 0, 1], [-1, 1]), (5, [0, 1], [-1, 1]),
                      (7, upoly.mul([-1, 1], [-1, 1]), upoly.mul([-1, 1], [-2, 1]))]:
        syl.append({"p": p, "f": [c % p for c in fa], "g": [c % p for c in gb],
                    "gcd": list(M.zp_gcd_sylvester(M.ModPoly.make(fa, p), M.ModPoly.make(gb, p)).coeffs)})
    rng = random.Random(13)
    p = M.prime_table()[1]
    for _ in range(500):
        fa = [rng.randrange(p) for _ in range(rng.randint(2, 7))]
        gb = [rng.randrange(p) for _ in range(rng.randint(2, 7))]
        fa[-1] = fa[-1] or 1
        gb[-1] = gb[-1] or 1
        syl.append({"p": p, "f": fa, "g": gb, "euclid": M._zp_gcd(fa, gb, p),
                    "gcd": list(M.zp_gcd_sylvester(M.ModPoly.make(fa, p), M.ModPoly.make(gb, p)).coeffs)})
    out["zp_gcd_sylvester"] = syl

    # subresultant profiles, test_modpoly.py:218-261
    prof = []
    p0 = M.prime_table()[0]
    for f, g, rstar in [(circle, fy, [-1, 0, 1]), (cusp, cusp.diff("y"), [0, 1])]:
        pr = M.modular_subres_profile(f, g, rstar, p0)
        prof.append({"f": terms_out(f), "g": terms_out(g), "rstar": ints_out(rstar), "p": p0,
                     "chain": list(pr.chain_degrees), "d": list(pr.factor_degrees)})
    rng = random.Random(21)
    p2 = M.prime_table()[2]
    for _ in range(10):
        terms = {(0, rng.randint(2, 4)): 1}
        for i in range(1, 4):
            for j in range(0, max(terms)[1]):
                if rng.random() < 0.5:
                    terms[(i, j)] = rng.randint(-4, 4)
        f = BivPoly({k: v for k, v in terms.items() if v})
        fyy = f.diff("y")
        if fyy.is_zero():
            continue
        r = M.biv_resultant(f, fyy, "y")
        if not r or upoly.degree(r) == 0:
            continue
        dec = upoly.squarefree_decompose(r)
        rstar = [1]
        for fac, _ in dec.factors:
            rstar = upoly.mul(rstar, list(fac))
        pr = M.modular_subres_profile(f, fyy, rstar, p2)
        prof.append({"f": terms_out(f), "g": terms_out(fyy), "rstar": ints_out(rstar), "p": p2,
                     "res": ints_out(r), "chain": list(pr.chain_degrees), "d": list(pr.factor_degrees)})
    out["subres_profile"] = prof

    # square-free decomposition, test_upoly.py:16-44
    sqf = []
    cases = [[2, -3, 0, 1], [-2, 0, 1], [0, 0, 4]]
    rng = random.Random(7)
    for _ in range(60):
        q = [rng.choice([-1, 1]) * rng.randint(1, 4)]
        for _ in range(rng.randint(1, 3)):
            factor = [rng.randint(-5, 5) for _ in range(rng.randint(1, 3))] + [rng.randint(1, 4)]
            q = upoly.mul(q, upoly.pow_(factor, rng.randint(1, 3)))
        cases.append(q)
    for q in cases:
        dec = upoly.squarefree_decompose(q)
        sqf.append({"p": ints_out(q), "content": str(dec.content),
                    "factors": [[ints_out(fac), mult] for fac, mult in dec.factors]})
    out["squarefree"] = sqf

    # prime table, modpoly.py:57-73
    t = M.prime_table()
    out["prime_table"] = {"count": len(t), "first": list(t[:8]), "last": list(t[-8:]),
                          "sha16": sha16(t),
                          "stream0_first": [next(iter(M.prime_stream(0)))],
                          "stream0_8": list(M.prime_stream(0))[:8],
                          "stream7_8": list(M.prime_stream(7))[:8]}
    dump("small", out)


def gen_cfg1():
    """Bisolve end to end on cfg1 (d=6, 10-bit), combinatorial filter only."""
    from curvekit import bisolve
    from curvekit.bisolve import solve
    out = {"source": "curvekit.bisolve.solve(f, g, filters={'combinatorial'}) "
                     "(pkg/src/curvekit/bisolve.py:541-556) run unmodified",
           "systems": []}
    for seed in range(5):
        ft, gt = make_pair("cfg1", seed)
        f, g = BivPoly(ft), BivPoly(gt)
        t0 = time.time()
        ry = M.biv_resultant(f, g, "y")
        rx = M.biv_resultant(f, g, "x")
        t_res = time.time() - t0
        t0 = time.time()
        sols = solve(f, g, filters=frozenset({"combinatorial"}), seed=0)
        t_solve = time.time() - t0
        boxes = []
        for s in sols:
            xi, yi = s.x.interval, s.y.interval
            boxes.append([[str(xi.lo.man), xi.lo.exp], [str(xi.hi.man), xi.hi.exp],
                          [str(yi.lo.man), yi.lo.exp], [str(yi.hi.man), yi.hi.exp]])
        dec = upoly.squarefree_decompose(ry)
        out["systems"].append({"seed": seed, "f": terms_out(ft), "g": terms_out(gt),
                               "res_y": ints_out(ry), "res_x": ints_out(rx),
                               "sqf_y": [[ints_out(fac), mult] for fac, mult in dec.factors],
                               "lead_gcd": ints_out(M.int_gcd_uni(f.lead_coeff_y(), g.lead_coeff_y())),
                               "boxes": boxes, "t_res_s": t_res, "t_solve_s": t_solve})
        print("cfg1 seed", seed, "res %.2fs solve %.2fs" % (t_res, t_solve), len(boxes), "boxes")
    # known-x suite (test_bisolve.py:142-195) under the combinatorial filter
    sys.path.insert(0, REF_TESTS)
    import test_bisolve as TB
    rng = random.Random(1234)
    kx = []
    for _ in range(30):
        f, g, q, comp = TB._known_x_system(rng)
        sols = solve(f, g, filters=frozenset({"combinatorial"}))
        boxes = []
        for s in sols:
            xi, yi = s.x.interval, s.y.interval
            boxes.append([[str(xi.lo.man), xi.lo.exp], [str(xi.hi.man), xi.hi.exp],
                          [str(yi.lo.man), yi.lo.exp], [str(yi.hi.man), yi.hi.exp]])
        kx.append({"f": terms_out(f), "g": terms_out(g), "boxes": boxes})
    out["known_x"] = kx
    _ = bisolve
    dump("cfg1_bisolve", out)


def gen_big(config):
    ft, gt = make_pair(config, 0)
    f, g = BivPoly(ft), BivPoly(gt)
    t0 = time.time()
    r = M.biv_resultant(f, g, "y")
    dt = time.time() - t0
    obj = {"source": "curvekit.modpoly.biv_resultant (pkg/src/curvekit/modpoly.py:348-394) "
                     "run unmodified", "config": config, "seed": 0, "seconds": dt,
           "f": terms_out(ft), "g": terms_out(gt),
           "res": [format(c, "x") for c in r], "sha16_repr": sha16(r),
           "deg": len(r) - 1, "max_bits": max(abs(c).bit_length() for c in r)}
    print(config, "res in %.1fs" % dt, "sha16", obj["sha16_repr"])
    if config == "cfg3":
        t0 = time.time()
        dec = upoly.squarefree_decompose(r)
        if len(dec.factors) == 1 and list(dec.factors[0][0]) == upoly.primitive(r):
            obj["sqf"] = [["primitive(res)", dec.factors[0][1]]]  # keep the fixture small
        else:
            obj["sqf"] = [[[format(c, "x") for c in fac], mult] for fac, mult in dec.factors]
        obj["sqf_content"] = str(dec.content)
        obj["t_sqf_s"] = time.time() - t0
        t0 = time.time()
        gg = M.int_gcd_uni(r, upoly.derivative(r))
        obj["gcd_r_dr"] = ints_out(gg)
        obj["t_gcd_s"] = time.time() - t0
        rstar = [1]
        for fac, _ in dec.factors:
            rstar = upoly.mul(rstar, list(fac))
        p = M.prime_table()[0]
        t0 = time.time()
        pr = M.modular_subres_profile(f, g, rstar, p)
        obj["profile"] = {"p": p, "chain": list(pr.chain_degrees), "d": list(pr.factor_degrees)}
        obj["t_profile_s"] = time.time() - t0
    dump(config + "_seed0", obj, gz=True)


def gen_cfg4prime():
    """One prime of the reference loop body (modpoly.py:376-391) at cfg4."""
    ft, gt = make_pair("cfg4", 0)
    f, g = BivPoly(ft), BivPoly(gt)
    fc, gc = f.coeffs_wrt_y(), g.coeffs_wrt_y()
    m, n = len(fc) - 1, len(gc) - 1
    deg_bound = f.deg_x() * n + g.deg_x() * m
    p = next(iter(M.prime_stream(0)))
    t0 = time.time()
    fpc = [[c % p for c in cf] for cf in fc]
    gpc = [[c % p for c in cg] for cg in gc]
    points, values = [], []
    t = 0
    while len(points) < deg_bound + 1:
        if M._zp_eval(fpc[-1], t, p) and M._zp_eval(gpc[-1], t, p):
            fu = M._zp_trim([M._zp_eval(cf, t, p) for cf in fpc])
            gu = M._zp_trim([M._zp_eval(cg, t, p) for cg in gpc])
            points.append(t)
            values.append(M._zp_resultant(fu, gu, p))
        t += 1
    t_img = time.time() - t0
    # interpolating all 3201 points is 43 s in the reference; the result has
    # degree <= 1600 so the first 1601 points already determine it
    t0 = time.time()
    poly = M._zp_interp(points[:1601], values[:1601], p)
    t_int = time.time() - t0
    obj = {"source": "curvekit.modpoly loop body modpoly.py:376-391 (one prime, cfg4 seed 0)",
           "p": p, "values": values, "poly": poly, "t_images_s": t_img, "t_interp1601_s": t_int}
    print("cfg4 prime", p, "images %.1fs interp %.1fs deg %d" % (t_img, t_int, len(poly) - 1))
    dump("cfg4_prime0", obj, gz=True)


def gen_descartes():
    """The Descartes test of real-root isolation, upoly._variations_on (upoly.py:338-346):
    every (polynomial, interval) a reference isolation visits, recorded with its count,
    plus the reference's isolating intervals (descartes_isolate, upoly.py:358-408)."""
    from curvekit.dyadic import Dyadic
    rng = random.Random(61)
    polys = []
    # resultants of small curves (what Bisolve isolates) and random square-free polynomials
    for seed in range(3):
        f, g = make_pair("cfg1", seed)
        r = M.biv_resultant(BivPoly(f), BivPoly(g), "y")
        polys.append(("cfg1_seed%d_res_y" % seed, upoly.primitive(r)))
    for deg in (5, 17, 40, 90):
        for k in range(2):
            p = [rng.randint(-2 ** 40, 2 ** 40) for _ in range(deg + 1)]
            p[-1] = p[-1] or 1
            polys.append(("random_deg%d_%d" % (deg, k), p))
    f, g = make_pair("cfg2", 0)
    polys.append(("cfg2_res_y", upoly.primitive(M.biv_resultant(BivPoly(f), BivPoly(g), "y"))))
    cases, isol = [], []
    orig = upoly._variations_on
    for name, p in polys:
        if upoly.degree(M.int_gcd_uni(p, upoly.derivative(p))) > 0:
            continue
        seen = []

        def rec(q, a, b, _seen=seen):
            v = orig(q, a, b)
            _seen.append((a.man, a.exp, b.man, b.exp, v))
            return v
        upoly._variations_on = rec
        t0 = time.time()
        try:
            roots = upoly.descartes_isolate(p)
        finally:
            upoly._variations_on = orig
        dt = time.time() - t0
        isol.append({"name": name, "p": ints_out(p), "seconds": dt, "tests": len(seen),
                     "roots": [[str(r.interval.lo.man), r.interval.lo.exp, str(r.interval.hi.man), r.interval.hi.exp]
                               for r in roots]})
        step = max(1, len(seen) // 40)
        for (am, ae, bm, be, v) in seen[::step]:
            cases.append({"name": name, "am": str(am), "ae": ae, "bm": str(bm), "be": be, "v": v})
        print(name, "deg", upoly.degree(p), "tests", len(seen), "roots", len(roots), "%.1f s" % dt)
    for _ in range(60):  # arbitrary intervals, including ones that need many primes
        deg = rng.randint(1, 60)
        p = [rng.randint(-2 ** 30, 2 ** 30) for _ in range(deg + 1)]
        p[-1] = p[-1] or 1
        ae, be = rng.randint(-30, 3), rng.randint(-30, 3)
        am, bm = rng.randint(-2 ** 20, 2 ** 20), rng.randint(-2 ** 20, 2 ** 20)
        a, b = Dyadic(am, ae), Dyadic(bm, be)
        if b <= a:
            a, b = b, a
        cases.append({"name": "arbitrary", "p": ints_out(p), "am": str(a.man), "ae": a.exp, "bm": str(b.man),
                      "be": b.exp, "v": orig(p, a, b)})
    dump("descartes", {"source": "upoly._variations_on (upoly.py:338-346), descartes_isolate (:358-408)",
                       "polys": {name: ints_out(p) for name, p in polys}, "cases": cases, "isolations": isol},
         gz=True)


def gen_descartes_cfg3():
    """Isolating intervals of cfg3's resultant R (square-free; upoly.descartes_isolate, upoly.py:358-408)."""
    import math
    gold = json.load(gzip.open(os.path.join(HERE, "cfg3_seed0.json.gz"), "rt"))
    r = [int(c, 16) for c in gold["res"]]
    c = 0
    for v in r:
        c = math.gcd(c, v)
    p = [v // c for v in r]
    t0 = time.time()
    roots = upoly.descartes_isolate(p)
    dt = time.time() - t0
    print("cfg3 isolation", len(roots), "roots, %.1f s" % dt)
    dump("descartes_cfg3", {"source": "upoly.descartes_isolate (upoly.py:358-408) on primitive(res_y) of cfg3 seed 0",
                            "seconds": dt, "degree": len(p) - 1,
                            "roots": [[str(x.interval.lo.man), x.interval.lo.exp, str(x.interval.hi.man),
                                       x.interval.hi.exp] for x in roots]})


def gen_gcdbiv():
    """gcd_biv / is_squarefree_biv / square_part (bivpoly.py:266-320) on known
    answers (test_modpoly.py:264-269), planted common factors, singular curves."""
    from curvekit.bivpoly import gcd_biv, is_squarefree_biv, square_part

    def rnd(rng, d, bits, dens=1.0):
        t = {}
        for i in range(d + 1):
            for j in range(d + 1 - i):
                if rng.random() < dens:
                    c = rng.randint(-(2**bits), 2**bits)
                    if c:
                        t[(i, j)] = c
        return BivPoly(t or {(0, 1): 1})

    circle = BivPoly({(2, 0): 1, (0, 2): 1, (0, 0): -1})
    line = BivPoly({(0, 1): 1, (1, 0): -1})
    cases = [(circle * line, circle * BivPoly({(0, 1): 1})), (circle, line), (circle, BivPoly()),
             (BivPoly(), BivPoly({(0, 1): -3, (1, 0): 6})), (BivPoly({(2, 0): 4, (0, 0): -4}), BivPoly({(1, 0): 6, (0, 0): 6})),
             (BivPoly({(2, 0): 4, (0, 0): -4}), circle * BivPoly({(1, 0): 2, (0, 0): 2})),
             (circle * BivPoly({(0, 1): 2, (1, 0): 1}), line * BivPoly({(0, 1): 2, (1, 0): 1})),
             (circle.scale(6) * BivPoly({(1, 0): 1, (0, 0): 1}), circle.scale(-4) * BivPoly({(2, 0): 1, (0, 0): -1}))]
    rng = random.Random(31)
    for d, dh, bits in [(3, 1, 6), (4, 2, 8), (5, 2, 10), (6, 3, 10), (8, 4, 16), (10, 5, 16), (12, 6, 32),
                        (14, 3, 40), (16, 8, 24)]:
        for _ in range(3):
            h = rnd(rng, dh, bits)
            cases.append((rnd(rng, d - dh, bits) * h, rnd(rng, d - dh, bits, 0.7) * h))
    for d, bits in [(4, 8), (8, 16)]:  # coprime
        cases.append((rnd(rng, d, bits), rnd(rng, d, bits)))
    gcds = []
    for f, g in cases:
        t0 = time.time()
        r = gcd_biv(f, g)
        gcds.append({"f": terms_out(f), "g": terms_out(g), "gcd": terms_out(r), "seconds": time.time() - t0})
    sq = []
    for d, bits, sing in [(6, 10, False), (10, 16, False), (16, 32, False), (4, 8, True), (6, 10, True),
                          (8, 12, True)]:
        if sing:  # f1^2 f2: a repeated factor
            f1 = rnd(rng, d // 2, bits)
            f = f1 * f1 * rnd(rng, d // 2, bits)
        else:
            f = rnd(rng, d, bits)
        t0 = time.time()
        isq = is_squarefree_biv(f)
        t1 = time.time()
        spart = square_part(f)
        sq.append({"f": terms_out(f), "squarefree": isq, "square_part": terms_out(spart),
                   "seconds_squarefree": t1 - t0, "seconds_square_part": time.time() - t1})
        print("sqfree", d, bits, sing, isq, "%.2f s" % (t1 - t0))
    dump("gcd_biv", {"source": "curvekit.bivpoly.gcd_biv / is_squarefree_biv / square_part (bivpoly.py:266-320)",
                     "gcd": gcds, "squarefree": sq})


if __name__ == "__main__":
    which = sys.argv[1:] or ["small"]
    for w in which:
        if w == "small":
            gen_small()
        elif w == "cfg1":
            gen_cfg1()
        elif w in ("cfg2", "cfg3"):
            gen_big(w)
        elif w == "cfg4prime":
            gen_cfg4prime()
        elif w == "descartes":
            gen_descartes()
        elif w == "gcdbiv":
            gen_gcdbiv()
        elif w == "descartes_cfg3":
            gen_descartes_cfg3()
        else:
            raise SystemExit("unknown fixture " + w)

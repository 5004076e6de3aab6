"""GPU parity of the modular bivariate gcd.

paper_1201_1548_b200.bivpoly.gcd_biv / is_squarefree_biv / square_part replace
curvekit.bivpoly's primitive-PRS versions (pkg/src/curvekit/bivpoly.py:266-320).
Every expected value below was produced by the unmodified reference
(tests/golden/make_golden.py gcdbiv -> tests/golden/gcd_biv.json): known answers
of test_modpoly.py:264-269, planted common factors up to total degree 16 with
40-bit coefficients, coprime pairs, zero inputs, integer and x-contents, and
square-free / singular curves (f1^2 f2).  Results must be identical terms.
"""

import os
import sys
import time

import pytest

from conftest import REPO, load_golden, terms_in

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def golden():
    return load_golden("gcd_biv.json")


def test_gcd_biv_matches_reference(golden):
    from paper_1201_1548_b200 import _lib
    from paper_1201_1548_b200.bivpoly import BivPoly, gcd_biv
    n0 = _lib.launch_count()
    for case in golden["gcd"]:
        f, g = BivPoly(terms_in(case["f"])), BivPoly(terms_in(case["g"]))
        got = gcd_biv(f, g)
        assert isinstance(got, BivPoly)
        assert got.terms == terms_in(case["gcd"]), (case["f"], case["g"])
    assert _lib.launch_count() > n0


def test_gcd_biv_symmetric_and_dict_input(golden):
    from paper_1201_1548_b200.bivpoly import gcd_biv
    for case in golden["gcd"][:12]:
        got = gcd_biv(terms_in(case["g"]), terms_in(case["f"]))
        assert got.terms == terms_in(case["gcd"])


def test_squarefree_and_square_part(golden):
    from paper_1201_1548_b200.bivpoly import BivPoly, is_squarefree_biv, square_part
    for case in golden["squarefree"]:
        f = BivPoly(terms_in(case["f"]))
        t0 = time.perf_counter()
        assert is_squarefree_biv(f) == case["squarefree"]
        dt = time.perf_counter() - t0
        assert square_part(f).terms == terms_in(case["square_part"])
        print(f"is_squarefree_biv deg {f.total_degree()}: {dt:.3f} s (reference {case['seconds_squarefree']:.2f} s)")


def test_installed_into_reference(golden, ref_bivpoly):
    BP = ref_bivpoly

    import paper_1201_1548_b200 as pkg
    from paper_1201_1548_b200 import bivpoly as ours
    saved = pkg.install()
    try:
        assert BP.gcd_biv is ours.gcd_biv
        for case in golden["squarefree"]:
            f = BP.BivPoly(terms_in(case["f"]))
            assert BP.is_squarefree_biv(f) == case["squarefree"]
            sp = BP.square_part(f)
            assert isinstance(sp, BP.BivPoly) and sp.terms == terms_in(case["square_part"])
    finally:
        pkg.uninstall(saved)
    assert BP.gcd_biv is not ours.gcd_biv


def test_squarefree_cfg3_curve():
    """GeoTop's square-freeness check of cfg3's f (degree 24, 64-bit): the
    reference's PRS does not finish in hours; the result must be True for a
    random dense curve, and f * f_1 (a planted square) must be detected."""
    from paper_1201_1548_b200.bivpoly import BivPoly, gcd_biv, is_squarefree_biv
    from paper_1201_1548_b200.synth import make_pair
    f, _ = make_pair("cfg3", 0)
    F = BivPoly(f)
    t0 = time.perf_counter()
    assert is_squarefree_biv(F)
    print(f"is_squarefree_biv cfg3 f: {time.perf_counter() - t0:.3f} s")
    h = BivPoly({(1, 1): 3, (2, 0): -5, (0, 1): 7, (0, 0): 1})
    prod = {}
    for (i, j), a in F.terms.items():
        for (k, l), b in h.terms.items():
            prod[(i + k, j + l)] = prod.get((i + k, j + l), 0) + a * b
    G = BivPoly(prod)
    t0 = time.perf_counter()
    got = gcd_biv(G, BivPoly({(k, l): 2 * b for (k, l), b in h.terms.items()}))
    print(f"gcd_biv(cfg3 f * h, 2h): {time.perf_counter() - t0:.3f} s")
    # the primitive gcd is h up to sign; the largest monomial x^2 has coefficient -5 -> -h
    assert got.terms == {k: -a for k, a in h.terms.items()}

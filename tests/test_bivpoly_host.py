"""Host-side parts of the modular bivariate gcd (CPU, no GPU): the restated
contents, exact divisions and sign convention of curvekit.bivpoly
(pkg/src/curvekit/bivpoly.py:183-240, :298-304) against the reference itself on
the gcd fixture's polynomials (tests/golden/gcd_biv.json)."""

import os
import sys

import pytest

from conftest import REPO, load_golden, terms_in


def _cols(terms):
    from paper_1201_1548_b200.bivpoly import BivPoly
    return BivPoly(terms).coeffs_wrt_y()


def test_content_and_primitive_part_match_reference(ref_bivpoly):
    from oracle import oracle
    from paper_1201_1548_b200.bivpoly import content_y, div_uni_x
    gold = load_golden("gcd_biv.json")
    import curvekit.modpoly as RM
    for case in gold["gcd"]:
        for key in ("f", "g"):
            t = terms_in(case[key])
            if not t:
                continue
            want = ref_bivpoly.BivPoly(t).content_y(gcd_fn=RM.int_gcd_uni)
            got = content_y(_cols(t), gcd_fn=oracle.int_gcd_uni)
            assert got == want
            assert div_uni_x(_cols(t), got) == ref_bivpoly.BivPoly(t).div_uni_x(want).coeffs_wrt_y()


def test_exact_division_matches_reference(ref_bivpoly):
    from paper_1201_1548_b200.bivpoly import divexact_cols
    gold = load_golden("gcd_biv.json")
    for case in gold["gcd"]:
        f, d = terms_in(case["f"]), terms_in(case["gcd"])
        if not f or not d:
            continue
        q = divexact_cols(_cols(f), _cols(d))
        want = ref_bivpoly.divexact_biv(ref_bivpoly.BivPoly(f), ref_bivpoly.BivPoly(d))
        assert q is not None and q == want.coeffs_wrt_y()
        # a non-divisor: f / (d + 1) is inexact unless d is a unit
        if len(d) > 1:
            d1 = dict(d)
            d1[(0, 0)] = d1.get((0, 0), 0) + 1
            try:
                ref_bivpoly.divexact_biv(ref_bivpoly.BivPoly(f), ref_bivpoly.BivPoly(d1))
                inexact = False
            except ArithmeticError:
                inexact = True
            assert (divexact_cols(_cols(f), _cols(d1)) is None) == inexact


def test_sign_normalisation_matches_reference(ref_bivpoly):
    from paper_1201_1548_b200.bivpoly import _normalize_sign
    for t in ({(2, 0): -5, (1, 1): 3}, {(0, 3): 7, (3, 0): -1}, {(0, 0): -2}, {}):
        want = ref_bivpoly._normalize_sign(ref_bivpoly.BivPoly(t)).terms
        assert _normalize_sign(dict(t)) == want

"""End-to-end parity through the reference's own consumer.

The unmodified reference package (installed offline into baseline/_ref, see
DESIGN.md) runs Bisolve (pkg/src/curvekit/bisolve.py:541-556) with its
resultants, gcds and square-free decompositions served by the B200 engine
(paper_1201_1548_b200.install(), rebinding modpoly.py's names and the names
bisolve.py:26 bound at import).  The isolating boxes must equal the ones the
reference produced on its own (tests/golden/cfg1_bisolve.json).
"""

import os
import sys

import pytest

from conftest import REPO, load_golden, terms_in


def test_install_rebinds_and_restores(curvekit_mod):
    import curvekit.bisolve as B
    import curvekit.modpoly as M

    import paper_1201_1548_b200 as pkg
    from paper_1201_1548_b200 import modpoly as ours
    orig = (M.biv_resultant, M.int_gcd_uni, B.biv_resultant, B.int_gcd_uni)
    saved = pkg.install()
    try:
        assert M.biv_resultant is ours.biv_resultant and B.biv_resultant is ours.biv_resultant
        assert M.int_gcd_uni is ours.int_gcd_uni and B.int_gcd_uni is ours.int_gcd_uni
        assert M.zp_gcd_sylvester is ours.zp_gcd_sylvester
        import curvekit.upoly as U
        from paper_1201_1548_b200 import upoly as our_upoly
        assert U._variations_on is our_upoly.variations_on
    finally:
        pkg.uninstall(saved)
    assert (M.biv_resultant, M.int_gcd_uni, B.biv_resultant, B.int_gcd_uni) == orig


def _boxes(sols):
    out = []
    for s in sols:
        xi, yi = s.x.interval, s.y.interval
        out.append([[str(xi.lo.man), xi.lo.exp], [str(xi.hi.man), xi.hi.exp],
                    [str(yi.lo.man), yi.lo.exp], [str(yi.hi.man), yi.hi.exp]])
    return out


@pytest.mark.gpu
def test_bisolve_cfg1_boxes_match_reference(curvekit_mod):
    from curvekit.bisolve import solve
    from curvekit.bivpoly import BivPoly

    import paper_1201_1548_b200 as pkg
    gold = load_golden("cfg1_bisolve.json")
    saved = pkg.install()
    try:
        for sysd in gold["systems"]:
            f, g = BivPoly(terms_in(sysd["f"])), BivPoly(terms_in(sysd["g"]))
            sols = solve(f, g, filters=frozenset({"combinatorial"}), seed=0)
            assert _boxes(sols) == sysd["boxes"], sysd["seed"]
    finally:
        pkg.uninstall(saved)


@pytest.mark.gpu
def test_bisolve_known_x_suite_matches_reference(curvekit_mod):
    # test_bisolve.py:142-195's 30 systems under the combinatorial filter
    from curvekit.bisolve import solve
    from curvekit.bivpoly import BivPoly

    import paper_1201_1548_b200 as pkg
    gold = load_golden("cfg1_bisolve.json")
    saved = pkg.install()
    try:
        for case in gold["known_x"]:
            f, g = BivPoly(terms_in(case["f"])), BivPoly(terms_in(case["g"]))
            sols = solve(f, g, filters=frozenset({"combinatorial"}))
            assert _boxes(sols) == case["boxes"]
    finally:
        pkg.uninstall(saved)


@pytest.mark.gpu
def test_reference_squarefree_uses_gpu_gcd(curvekit_mod):
    from curvekit import upoly

    import paper_1201_1548_b200 as pkg
    from paper_1201_1548_b200 import _lib
    small = load_golden("small.json")
    saved = pkg.install()
    try:
        n0 = _lib.launch_count()
        for c in small["squarefree"]:
            dec = upoly.squarefree_decompose([int(v) for v in c["p"]])
            assert str(dec.content) == c["content"]
            assert [[list(map(str, f)), m] for f, m in dec.factors] == c["factors"]
        assert _lib.launch_count() > n0, "the reference's Yun must reach the GPU gcd"
    finally:
        pkg.uninstall(saved)


def _ps_key(ps):
    dec = None if ps.decomposition is None else (str(ps.decomposition.content),
                                                  [[list(map(str, f)), m] for f, m in ps.decomposition.factors])
    roots = [(str(r.interval.lo.man), r.interval.lo.exp, str(r.interval.hi.man), r.interval.hi.exp)
             for r in ps.roots]
    return ps.axis, [str(c) for c in ps.resultant], dec, roots, [str(c) for c in ps.lead_gcd]


@pytest.mark.gpu
def test_batched_biproject_matches_reference(curvekit_mod):
    """paper_1201_1548_b200.bisolve.biproject (both resultants in
    one batched GPU call, both lead gcds in one gcd batch) returns the projection
    sets of the reference's biproject (bisolve.py:103-114)."""
    import curvekit.bisolve as B
    from curvekit.bivpoly import BivPoly

    import paper_1201_1548_b200 as pkg
    from paper_1201_1548_b200 import bisolve as ours
    gold = load_golden("cfg1_bisolve.json")
    systems = [(BivPoly(terms_in(s["f"])), BivPoly(terms_in(s["g"]))) for s in gold["systems"][:3]]
    want = [tuple(_ps_key(ps) for ps in B.biproject(f, g)) for f, g in systems]  # the unmodified reference
    saved = pkg.install()
    try:
        assert B.biproject is ours.biproject
        got = [tuple(_ps_key(ps) for ps in B.biproject(f, g)) for f, g in systems]
    finally:
        pkg.uninstall(saved)
    assert got == want
    # a common factor: both resultants vanish -> CommonFactorError carrying gcd_biv
    circle = BivPoly({(2, 0): 1, (0, 2): 1, (0, 0): -1})
    line = BivPoly({(0, 1): 1, (1, 0): -1})
    saved = pkg.install()
    try:
        with pytest.raises(B.CommonFactorError) as ei:
            B.biproject(circle * line, circle * BivPoly({(0, 1): 1}))
    finally:
        pkg.uninstall(saved)
    assert ei.value.factor == circle


def test_install_twice_then_uninstall_restores_reference(curvekit_mod):
    import curvekit.bisolve as B
    import curvekit.modpoly as M
    import curvekit.upoly as U

    import paper_1201_1548_b200 as pkg
    orig = (M.biv_resultant, U.descartes_isolate, B.biproject)
    first = pkg.install()
    second = pkg.install()  # already installed: must still return the reference's functions
    assert second == first
    pkg.uninstall(second)
    assert (M.biv_resultant, U.descartes_isolate, B.biproject) == orig

"""Batched projection step of Bisolve.

Drop-in for ``curvekit.bisolve.biproject`` (pkg/src/curvekit/bisolve.py:103-114):
the reference computes res_y and res_x one after the other (:107-108) and the
gcd of the leading coefficients once per axis (:118).  Here both resultants go
to the GPU in ONE library call (``modpoly.biv_resultant_batch``: each pipeline on
its own stream, their kernels overlapping) and both leading-coefficient gcds in
one modular gcd batch; the square-free decomposition and real-root isolation of
each resultant are the reference's own functions (served by the GPU gcd and
Descartes test once ``install()`` has rebound them).  Same return value, same
errors (``ValueError`` on a zero input, ``CommonFactorError(gcd_biv(f, g))`` when
a resultant vanishes).
"""

from __future__ import annotations

from .bivpoly import as_biv
from .modpoly import biv_resultant_batch, int_gcd_uni_batch


def biproject(f, g, seed: int = 0) -> tuple:
    """Project the solutions onto both axes; errors out on common factors."""
    import importlib
    ref = importlib.import_module("curvekit.bisolve")
    upoly = importlib.import_module("curvekit.upoly")
    if f.is_zero() or g.is_zero():
        raise ValueError("zero input polynomial")
    r_y, r_x = biv_resultant_batch([(f, g, "y"), (f, g, "x")], seed)
    if not r_y or not r_x:
        raise ref.CommonFactorError(ref.gcd_biv(f, g))
    F, G = as_biv(f), as_biv(g)
    lcs = [(F.lead_coeff_y(), G.lead_coeff_y()), (F.swap().lead_coeff_y(), G.swap().lead_coeff_y())]
    want = [i for i, (a, b) in enumerate(lcs) if a or b]
    gcds = int_gcd_uni_batch([lcs[i] for i in want])
    lead = [[], []]
    for i, gv in zip(want, gcds):
        lead[i] = gv

    def projection_set(axis, resultant, lead_gcd):
        # bisolve.py:117-124 with the lead gcd precomputed
        if upoly.degree(resultant) < 1:
            return ref.ProjectionSet(axis, resultant, None, [], lead_gcd)
        dec = upoly.squarefree_decompose(resultant)
        roots = upoly.isolate_decomposition(dec)
        return ref.ProjectionSet(axis, resultant, dec, roots, lead_gcd)

    return projection_set("x", r_y, lead[0]), projection_set("y", r_x, lead[1])

"""B200-native multi-modular resultant / gcd engine (drop-in for curvekit.modpoly).

Reference: arXiv 1201.1548 artifact ``curvekit`` (pure Python); hot path
pkg/src/curvekit/modpoly.py.  See DESIGN.md.
"""

__version__ = "0.1.0"


def install():
    """Rebind the reference's hot-path names to the B200 implementations.

    Rebinds ``curvekit.modpoly.{biv_resultant, int_gcd_uni, zp_resultant_uni,
    zp_interpolate, zp_gcd_sylvester, crt_reconstruct, modular_subres_profile}``
    and the names
    ``curvekit.bisolve`` bound at import (bisolve.py:26).  ``upoly`` and
    ``bivpoly`` import ``int_gcd_uni`` lazily (upoly.py:258,372,538,569;
    bivpoly.py:186,268), so they pick up the GPU gcd through the first rebinding.
    Also rebinds ``curvekit.upoly._variations_on`` (the Descartes test of
    descartes_isolate, upoly.py:338-346) to the GPU version, and
    ``curvekit.upoly.descartes_isolate`` (upoly.py:358-408) to a breadth-first
    version that tests a whole subdivision level per GPU call.
    Rebinds ``curvekit.bivpoly.gcd_biv`` (bivpoly.py:266-295; ``is_squarefree_biv`` and
    ``square_part`` look it up at call time) and the name ``curvekit.bisolve``
    bound at import (bisolve.py:21) to the modular GPU gcd.
    Rebinds ``curvekit.bisolve.biproject`` to the batched projection
    (paper_1201_1548_b200.bisolve: res_y and res_x in one GPU call).
    Returns the previous bindings (pass them to ``uninstall``).
    """
    import importlib

    from . import modpoly as ours
    ref = importlib.import_module("curvekit.modpoly")
    saved = {}
    for name in ("biv_resultant", "int_gcd_uni", "zp_resultant_uni", "zp_interpolate",
                 "zp_gcd_sylvester", "crt_reconstruct", "modular_subres_profile"):
        saved[("curvekit.modpoly", name)] = getattr(ref, name)
        setattr(ref, name, getattr(ours, name))
    # the Descartes test of real-root isolation (upoly.py:338-346), looked up
    # by descartes_isolate at call time
    up = importlib.import_module("curvekit.upoly")
    from . import upoly as our_upoly
    saved[("curvekit.upoly", "_variations_on")] = getattr(up, "_variations_on")
    setattr(up, "_variations_on", our_upoly.variations_on)
    # breadth-first isolation: one batched GPU call per subdivision level
    # (upoly.py:358-408; isolate_decomposition :411-421 and :573 look it up at call time)
    saved[("curvekit.upoly", "descartes_isolate")] = getattr(up, "descartes_isolate")
    setattr(up, "descartes_isolate", our_upoly.descartes_isolate)
    bp = importlib.import_module("curvekit.bivpoly")
    from . import bivpoly as our_bivpoly
    saved[("curvekit.bivpoly", "gcd_biv")] = getattr(bp, "gcd_biv")
    setattr(bp, "gcd_biv", our_bivpoly.gcd_biv)
    try:
        bis = importlib.import_module("curvekit.bisolve")
    except ImportError:  # bisolve needs mpmath
        bis = None
    if bis is not None:
        for name in ("biv_resultant", "int_gcd_uni"):
            saved[("curvekit.bisolve", name)] = getattr(bis, name)
            setattr(bis, name, getattr(ours, name))
        saved[("curvekit.bisolve", "gcd_biv")] = getattr(bis, "gcd_biv")
        setattr(bis, "gcd_biv", our_bivpoly.gcd_biv)
        # both resultants of the projection in one batched GPU call (bisolve.py:103-114,
        # looked up by Bisolve.__init__ at bisolve.py:412)
        from . import bisolve as our_bisolve
        saved[("curvekit.bisolve", "biproject")] = getattr(bis, "biproject")
        setattr(bis, "biproject", our_bisolve.biproject)
    return saved


def uninstall(saved):
    import importlib
    for (mod, name), fn in saved.items():
        setattr(importlib.import_module(mod), name, fn)

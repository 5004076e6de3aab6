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
    saved = {}
    for mod, name, repl in _bindings():
        try:
            m = importlib.import_module(mod)
        except ImportError:  # curvekit.bisolve needs mpmath
            continue
        cur = getattr(m, name)
        # installing twice must still hand back the reference's own function
        orig = _ORIGINALS.get((mod, name), cur) if cur is repl else cur
        _ORIGINALS.setdefault((mod, name), orig)
        saved[(mod, name)] = orig
        setattr(m, name, repl)
    return saved


_ORIGINALS = {}


def _bindings():
    """(module, name, replacement) for every rebinding install() makes."""
    import importlib
    from . import bisolve as our_bisolve
    from . import bivpoly as our_bivpoly
    from . import modpoly as ours
    from . import upoly as our_upoly
    out = [("curvekit.modpoly", name, getattr(ours, name))
           for name in ("biv_resultant", "int_gcd_uni", "zp_resultant_uni", "zp_interpolate",
                        "zp_gcd_sylvester", "crt_reconstruct", "modular_subres_profile")]
    # the Descartes test (upoly.py:338-346) and the breadth-first isolation
    # (upoly.py:358-408; isolate_decomposition :411-421 and :573 look it up at call time)
    out += [("curvekit.upoly", "_variations_on", our_upoly.variations_on),
            ("curvekit.upoly", "descartes_isolate", our_upoly.descartes_isolate),
            ("curvekit.bivpoly", "gcd_biv", our_bivpoly.gcd_biv)]
    # names bisolve.py binds at import (:21, :26), and the projection (:103-114,
    # looked up by _Solver.__init__ at :412)
    out += [("curvekit.bisolve", "biv_resultant", ours.biv_resultant),
            ("curvekit.bisolve", "int_gcd_uni", ours.int_gcd_uni),
            ("curvekit.bisolve", "gcd_biv", our_bivpoly.gcd_biv),
            ("curvekit.bisolve", "biproject", our_bisolve.biproject)]
    # the other direction: while installed, the engine raises and returns the
    # reference's own exception and value types (UnluckyPrime, modpoly.py:23-24;
    # ModPoly :80-93; ResidueSystem :258-261; ModularSubresultantProfile :421-425),
    # so callers' `except UnluckyPrime` / isinstance / == checks behave as before
    try:
        ref = importlib.import_module("curvekit.modpoly")
    except ImportError:
        return out
    out += [("paper_1201_1548_b200.modpoly", name, getattr(ref, name))
            for name in ("UnluckyPrime", "ModPoly", "ResidueSystem", "ModularSubresultantProfile")]
    return out


def uninstall(saved):
    import importlib
    for (mod, name), fn in saved.items():
        setattr(importlib.import_module(mod), name, fn)

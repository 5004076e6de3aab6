"""cfg3 of BASELINE.json end to end — GeoTop's symbolic steps on f (degree 24,
64-bit) through the reference's OWN functions with install() (every modular step
on the GPU), each output checked against the unmodified reference's recorded
result (tests/golden/cfg3_seed0.json.gz, descartes_cfg3.json) and timed beside
the reference's recorded time.

    res_y(f, f_y)                       modpoly.biv_resultant      (reference 635 s)
    square-free decomposition of R      upoly.squarefree_decompose (0.14 s)
    gcd(R, R')                          modpoly.int_gcd_uni        (0.11 s)
    subresultant degree profile         modpoly.modular_subres_profile (82.6 s)
    real-root isolation of R*           upoly.isolate_decomposition (168.8 s)
    square-freeness of the curve        bivpoly.is_squarefree_biv  (PRS; not finished in hours)
"""
import json
import math
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "baseline", "_ref"))
sys.path.insert(0, os.path.join(REPO, "tests"))
import curvekit.bivpoly as BP  # noqa: E402
import curvekit.modpoly as M  # noqa: E402
import curvekit.upoly as U  # noqa: E402
from conftest import load_golden  # noqa: E402

import paper_1201_1548_b200 as pkg  # noqa: E402
from paper_1201_1548_b200.synth import make_pair  # noqa: E402

gold = load_golden("cfg3_seed0.json.gz")
iso_gold = load_golden("descartes_cfg3.json")
f, fy = make_pair("cfg3", 0)
F, FY = BP.BivPoly(f), BP.BivPoly(fy)
saved = pkg.install()
rows = []
try:
    M.biv_resultant(BP.BivPoly({(1, 1): 1}), BP.BivPoly({(0, 1): 1, (1, 0): 1}), "y")  # context up front

    def step(name, ref_s, fn):
        t0 = time.perf_counter()
        out = fn()
        dt = time.perf_counter() - t0
        rows.append({"step": name, "seconds": dt, "reference_seconds": ref_s})
        return out

    R = step("res_y(f, f_y)", gold["seconds"], lambda: M.biv_resultant(F, FY, "y"))
    assert R == [int(c, 16) for c in gold["res"]]
    dec = step("squarefree_decompose(R)", gold["t_sqf_s"], lambda: U.squarefree_decompose(R))
    assert str(dec.content) == gold["sqf_content"] and len(dec.factors) == 1
    g = step("int_gcd_uni(R, R')", gold["t_gcd_s"], lambda: M.int_gcd_uni(R, U.derivative(R)))
    assert g == [int(c) for c in gold["gcd_r_dr"]]
    content = int(gold["sqf_content"])
    rstar = [c // content for c in R]
    pr = step("modular_subres_profile", gold["t_profile_s"],
              lambda: M.modular_subres_profile(F, FY, rstar, gold["profile"]["p"]))
    assert list(pr.chain_degrees) == gold["profile"]["chain"] and list(pr.factor_degrees) == gold["profile"]["d"]
    roots = step("isolate_decomposition(R)", iso_gold["seconds"], lambda: U.isolate_decomposition(dec))
    assert [[str(x.interval.lo.man), x.interval.lo.exp, str(x.interval.hi.man), x.interval.hi.exp]
            for x in roots] == iso_gold["roots"]
    sq = step("is_squarefree_biv(f)", None, lambda: BP.is_squarefree_biv(F))
    assert sq is True
finally:
    pkg.uninstall(saved)
tot = sum(r["seconds"] for r in rows)
ref = sum(r["reference_seconds"] for r in rows if r["reference_seconds"] is not None)
for r in rows:
    rs = r["reference_seconds"]
    print(f"{r['step']:28s} {r['seconds'] * 1e3:9.1f} ms   reference {'%.2f s' % rs if rs is not None else 'n/a'}")
print(f"total {tot:.3f} s vs reference {ref:.1f} s (+ is_squarefree_biv, which the reference's PRS does not finish)")
print(json.dumps({"cfg3_geotop": rows}))

"""Time the reference's descartes_isolate with the GPU Descartes test (cfg2, cfg4 resultants)."""
import math
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "baseline", "_ref"))
import curvekit.upoly as U  # noqa: E402

import paper_1201_1548_b200 as pkg  # noqa: E402
from paper_1201_1548_b200 import modpoly as mp  # noqa: E402
from paper_1201_1548_b200 import upoly as ours  # noqa: E402
from paper_1201_1548_b200.synth import make_pair  # noqa: E402

if os.environ.get("NO_GC"):
    import gc
    gc.disable()
saved = pkg.install()
calls = {"n": 0}
orig = ours.variations_on


def counted(p, a, b):
    calls["n"] += 1
    return orig(p, a, b)


U._variations_on = counted
for cfg in sys.argv[1:] or ["cfg2", "cfg4"]:
    f, g = make_pair(cfg, 0)
    r = mp.biv_resultant(f, g, "y")
    c = 0
    for v in r:
        c = math.gcd(c, v)
    p = [v // c for v in r]
    for rep in ("cold", "warm", "warm", "warm", "warm"):
        calls["n"] = 0
        t0 = time.time()
        roots = U.descartes_isolate(p)
        dt = time.time() - t0
        print(f"{cfg} ({rep}): degree {len(p) - 1}, {len(roots)} real roots, {calls['n']} single Descartes tests, "
              f"{dt:.3f} s")
pkg.uninstall(saved)

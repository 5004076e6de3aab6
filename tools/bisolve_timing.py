"""Bisolve end to end (the reference's solve) with and without install(), cfg1-style systems."""
import os
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "baseline", "_ref"))
from curvekit.bisolve import solve  # noqa: E402
from curvekit.bivpoly import BivPoly  # noqa: E402

import paper_1201_1548_b200 as pkg  # noqa: E402
from paper_1201_1548_b200 import modpoly  # noqa: E402
from paper_1201_1548_b200.synth import make_pair  # noqa: E402

modpoly.biv_resultant({(1, 1): 1}, {(0, 1): 1, (1, 0): 1}, "y")  # CUDA context up front
for d in (6, 8, 10):
    rows = []
    for mode in ("reference", "installed"):
        saved = pkg.install() if mode == "installed" else None
        try:
            t_tot, nsol = 0.0, 0
            for seed in range(3):
                if d == 6:
                    f, g = make_pair("cfg1", seed)
                else:
                    import random
                    rng = random.Random(seed)
                    f = {(i, j): rng.choice([-1, 1]) * rng.randint(1, 2 ** 10 - 1)
                         for i in range(d + 1) for j in range(d + 1 - i)}
                    g = {(i, j): rng.choice([-1, 1]) * rng.randint(1, 2 ** 10 - 1)
                         for i in range(d + 1) for j in range(d + 1 - i)}
                t0 = time.time()
                sols = solve(BivPoly(f), BivPoly(g), filters=frozenset({"combinatorial"}), seed=0)
                t_tot += time.time() - t0
                nsol += len(sols)
            rows.append((mode, t_tot, nsol))
        finally:
            if saved:
                pkg.uninstall(saved)
    print(f"degree {d}: " + "; ".join(f"{m} {t:.2f} s ({n} solutions)" for m, t, n in rows))

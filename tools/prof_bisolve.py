import cProfile
import os
import pstats
import random
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "baseline", "_ref"))
from curvekit.bisolve import solve  # noqa: E402
from curvekit.bivpoly import BivPoly  # noqa: E402

import paper_1201_1548_b200 as pkg  # noqa: E402
from paper_1201_1548_b200 import modpoly  # noqa: E402

modpoly.biv_resultant({(1, 1): 1}, {(0, 1): 1, (1, 0): 1}, "y")
pkg.install()
d = 10
rng = random.Random(0)
f = {(i, j): rng.choice([-1, 1]) * rng.randint(1, 2 ** 10 - 1) for i in range(d + 1) for j in range(d + 1 - i)}
g = {(i, j): rng.choice([-1, 1]) * rng.randint(1, 2 ** 10 - 1) for i in range(d + 1) for j in range(d + 1 - i)}
cProfile.run("solve(BivPoly(f), BivPoly(g), filters=frozenset({'combinatorial'}), seed=0)", "/tmp/b.prof")
pstats.Stats("/tmp/b.prof").sort_stats("cumtime").print_stats(25)

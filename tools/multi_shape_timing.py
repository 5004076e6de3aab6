"""A Bisolve-style stream of res_y calls over many distinct shapes (degrees 4-18,
random dense 16-bit pairs): each shape has its own primes/N plan and CRT tables.
Pass 1 pays the cold builds; pass 2 shows whether the caches keep them (the round-1
caches held 4 plans / 8 CRT tables: pass 2 was cold again beyond 4 shapes)."""
import os
import random
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1201_1548_b200 import modpoly as mp  # noqa: E402


def pair(d, seed, bits=16):
    rng = random.Random(seed)
    mk = lambda: {(i, j): rng.choice([-1, 1]) * rng.randint(1, 2 ** bits - 1)  # noqa: E731
                  for i in range(d + 1) for j in range(d + 1 - i)}
    return mk(), mk()


shapes = [pair(d, d) for d in range(4, 19)]
mp.biv_resultant(*pair(3, 0))  # library init
for p in (1, 2, 3):
    ts = []
    for f, g in shapes:
        t = time.perf_counter()
        mp.biv_resultant(f, g, "y")
        ts.append(time.perf_counter() - t)
    print(f"pass {p}: {len(shapes)} shapes, mean {statistics.mean(ts) * 1e3:.3f} ms, max {max(ts) * 1e3:.3f} ms",
          flush=True)

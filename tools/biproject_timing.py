"""biproject (bisolve.py:103-114): the reference, the reference with the GPU
engine installed but the projection unbatched (res_y, res_x, lead gcds one call
each), and the batched drop-in (paper_1201_1548_b200.bisolve.biproject)."""
import os
import random
import statistics
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "baseline", "_ref"))
import curvekit.bisolve as B  # noqa: E402
from curvekit.bivpoly import BivPoly  # noqa: E402

import paper_1201_1548_b200 as pkg  # noqa: E402
from paper_1201_1548_b200 import modpoly  # noqa: E402

REF_BIPROJECT = B.biproject


def system(d, seed, bits=10):
    rng = random.Random(seed)
    mk = lambda: BivPoly({(i, j): rng.choice([-1, 1]) * rng.randint(1, 2 ** bits - 1)  # noqa: E731
                          for i in range(d + 1) for j in range(d + 1 - i)})
    return mk(), mk()


def resultants_only(fn, f, g, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn(f, g)
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts)


modpoly.biv_resultant({(1, 1): 1}, {(0, 1): 1, (1, 0): 1}, "y")  # CUDA context up front
for d in (6, 10, 16, 24):
    f, g = system(d, 0)
    seq = lambda f, g: (modpoly.biv_resultant(f, g, "y"), modpoly.biv_resultant(f, g, "x"))  # noqa: E731
    bat = lambda f, g: modpoly.biv_resultant_batch([(f, g, "y"), (f, g, "x")])  # noqa: E731
    seq(f, g), bat(f, g)
    t_seq, t_bat = resultants_only(seq, f, g, 20), resultants_only(bat, f, g, 20)
    line = f"degree {d}: res_y+res_x sequential {1e3 * t_seq:.2f} ms, batched {1e3 * t_bat:.2f} ms"
    if d <= 10:
        t0 = time.perf_counter()
        want = REF_BIPROJECT(f, g)
        t_ref = time.perf_counter() - t0
        saved = pkg.install()
        try:
            B.biproject = REF_BIPROJECT  # GPU engine, unbatched projection
            REF_BIPROJECT(f, g)
            t0 = time.perf_counter()
            REF_BIPROJECT(f, g)
            t_unb = time.perf_counter() - t0
            from paper_1201_1548_b200 import bisolve as ours
            ours.biproject(f, g)
            t0 = time.perf_counter()
            got = ours.biproject(f, g)
            t_b = time.perf_counter() - t0
        finally:
            pkg.uninstall(saved)
        assert [p.resultant for p in got] == [p.resultant for p in want]
        line += f"; biproject reference {t_ref:.3f} s, GPU unbatched {t_unb:.3f} s, GPU batched {t_b:.3f} s"
    print(line, flush=True)

"""Quick device timing of one res_y per config (development aid)."""
import sys
import time

sys.path.insert(0, ".")
from paper_1201_1548_b200 import modpoly  # noqa: E402
from paper_1201_1548_b200.bivpoly import BivPoly  # noqa: E402
from paper_1201_1548_b200.synth import make_pair  # noqa: E402

for cfg in sys.argv[1:] or ["cfg2", "cfg4"]:
    f, g = make_pair(cfg, 0)
    F, G = BivPoly(f), BivPoly(g)
    fc, gc = F.coeffs_wrt_y(), G.coeffs_wrt_y()
    for it in range(4):
        t0 = time.perf_counter()
        res, info = modpoly._biv_resultant_gpu(fc, gc, F.total_degree(), G.total_degree())
        t1 = time.perf_counter()
        print(cfg, it, "wall %.2f ms" % ((t1 - t0) * 1e3), info)

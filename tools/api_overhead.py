"""Where a Python-API res_y call spends its time (cfg1, cfg2, cfg4).

Two host paths: term dicts straight into the limb grid (planner.pack_terms,
one C pass) and the coeffs_wrt_y + pack_grid + plan_resultant path taken for
inputs the C packer declines."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1201_1548_b200 import modpoly as mp  # noqa: E402
from paper_1201_1548_b200.bivpoly import as_biv  # noqa: E402
from paper_1201_1548_b200.planner import pack_grid, pack_terms, plan_packed, plan_resultant  # noqa: E402
from paper_1201_1548_b200.synth import make_pair  # noqa: E402


def timed(fn, reps=20):
    fn()
    t = time.perf_counter()
    for _ in range(reps):
        r = fn()
    return (time.perf_counter() - t) / reps * 1e3, r


for cfg in ("cfg1", "cfg2", "cfg4"):
    f, g = make_pair(cfg, 0)
    t_api, _ = timed(lambda: mp.biv_resultant(f, g, "y"))
    t_pt, pk = timed(lambda: pack_terms(f, g))
    t_pp, _ = timed(lambda: plan_packed(pk))
    t_gpu, (_, info) = timed(lambda: mp._biv_resultant_gpu(None, None, pk.tdf, pk.tdg, pk))
    F, G = as_biv(f), as_biv(g)
    t_c, (fc, gc) = timed(lambda: (F.coeffs_wrt_y(), G.coeffs_wrt_y()))
    t_p, pg = timed(lambda: pack_grid(fc, gc))
    t_pl, _ = timed(lambda: plan_resultant(fc, gc, F.total_degree(), G.total_degree(), pg.dfx, pg.dgx))
    print(f"{cfg}: api {t_api:.3f} ms | pack_terms {t_pt:.3f} plan_packed {t_pp:.3f} "
          f"plan+gpu-call+conversion {t_gpu:.3f} (device {info['device_ms']:.3f}) | "
          f"old path: coeffs_wrt_y {t_c:.3f} pack_grid {t_p:.3f} plan_resultant {t_pl:.3f}")

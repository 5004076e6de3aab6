"""Where a Python-API res_y call spends its time (cfg1 and cfg4)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1201_1548_b200 import modpoly as mp  # noqa: E402
from paper_1201_1548_b200.bivpoly import as_biv  # noqa: E402
from paper_1201_1548_b200.planner import limbs_to_ints, pack_grid, plan_resultant  # noqa: E402
from paper_1201_1548_b200.synth import make_pair  # noqa: E402

for cfg in ("cfg1", "cfg2", "cfg4"):
    f, g = make_pair(cfg, 0)
    for _ in range(3):
        mp.biv_resultant(f, g, "y")
    reps = 20
    t = time.perf_counter()
    for _ in range(reps):
        mp.biv_resultant(f, g, "y")
    tot = (time.perf_counter() - t) / reps
    F, G = as_biv(f), as_biv(g)
    t = time.perf_counter()
    for _ in range(reps):
        fc, gc = F.coeffs_wrt_y(), G.coeffs_wrt_y()
    t_c = (time.perf_counter() - t) / reps
    t = time.perf_counter()
    for _ in range(reps):
        pk = pack_grid(fc, gc)
    t_p = (time.perf_counter() - t) / reps
    t = time.perf_counter()
    for _ in range(reps):
        pl = plan_resultant(fc, gc, F.total_degree(), G.total_degree(), pk.dfx, pk.dgx)
    t_pl = (time.perf_counter() - t) / reps
    t = time.perf_counter()
    for _ in range(reps):
        _, info = mp._biv_resultant_gpu(fc, gc, F.total_degree(), G.total_degree())
    t_gpu = (time.perf_counter() - t) / reps
    print(f"{cfg}: api {tot*1e3:.3f} ms | coeffs_wrt_y {t_c*1e3:.3f} pack {t_p*1e3:.3f} plan {t_pl*1e3:.3f} "
          f"gpu-call incl. conversion {t_gpu*1e3:.3f} (device {info['device_ms']:.3f})")

"""Wall-time breakdown of one Python-API res_y at cfg4 (modpoly.biv_resultant):
packing, planning, the C-ABI call (device work + copies), the int conversion."""
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1201_1548_b200 import _lib, modpoly as mp  # noqa: E402
from paper_1201_1548_b200.planner import limbs_to_ints, pack_terms, plan_packed  # noqa: E402
from paper_1201_1548_b200.synth import make_pair  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
f, g = make_pair(cfg, 0)
lib = _lib.lib()
for _ in range(5):
    mp.biv_resultant(f, g, "y")
acc = {k: [] for k in ("api", "pack", "plan", "call", "device", "convert")}
for _ in range(30):
    t0 = time.perf_counter()
    mp.biv_resultant(f, g, "y")
    acc["api"].append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    pk = pack_terms(f, g, False)
    t1 = time.perf_counter()
    plan = plan_packed(pk, 0)
    t2 = time.perf_counter()
    K, N, LW = len(plan.primes), plan.N, plan.LW
    out = _lib.pinned.get("biv_out", N * LW)
    status = np.zeros(1, dtype=np.uint32)
    ms = np.zeros(1, dtype=np.float32)
    lib.ckb_biv_resultant(_lib.ptr(pk.limbs), pk.C, pk.L, _lib.ptr(pk.degs), pk.m, pk.n, pk.dfx, pk.dgx,
                          _lib.ptr(plan.primes), _lib.ptr(plan.gens), K, N, LW, _lib.ptr(out), _lib.ptr(status),
                          _lib.ptr(ms))
    t3 = time.perf_counter()
    limbs_to_ints(out, N, LW)
    t4 = time.perf_counter()
    for k, v in zip(("pack", "plan", "call", "convert"), (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
        acc[k].append(v)
    acc["device"].append(float(ms[0]) * 1e-3)
print(cfg, " ".join(f"{k} {statistics.median(v) * 1e3:.3f}" for k, v in acc.items()), "(ms, medians)")

"""Host-side cost of one C-ABI res_y call (cfg4, page-locked buffers, graph replay):
ckb_host_times = [entry -> work enqueued, enqueued -> finished] in microseconds,
beside the call's wall time and the device time of the same pipeline."""
import os
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1201_1548_b200 import _lib  # noqa: E402
from paper_1201_1548_b200.planner import pack_terms, plan_packed  # noqa: E402
from paper_1201_1548_b200.synth import make_pair  # noqa: E402

f, g = make_pair(sys.argv[1] if len(sys.argv) > 1 else "cfg4", 0)
lib = _lib.lib()
pk = pack_terms(f, g, False)
plan = plan_packed(pk, 0)
K, N, LW = len(plan.primes), plan.N, plan.LW
hl = _lib.pinned.get("in", pk.limbs.size)
hl[:] = pk.limbs.reshape(-1)
ho = _lib.pinned.get("out", N * LW)
st = np.zeros(1, dtype=np.uint32)
ms = np.zeros(1, dtype=np.float32)
args = (_lib.ptr(hl), pk.C, pk.L, _lib.ptr(pk.degs), pk.m, pk.n, pk.dfx, pk.dgx, _lib.ptr(plan.primes),
        _lib.ptr(plan.gens), K, N, LW, _lib.ptr(ho), _lib.ptr(st), _lib.ptr(ms))
ht = np.zeros(2, dtype=np.float32)
rows = []
for i in range(40):
    t = time.perf_counter()
    lib.ckb_biv_resultant(*args)
    w = (time.perf_counter() - t) * 1e6
    lib.ckb_host_times(_lib.ptr(ht), 2)
    if i >= 5:
        rows.append((w, float(ht[0]), float(ht[1]), float(ms[0]) * 1e3))
med = [statistics.median(r[k] for r in rows) for k in range(4)]
print("wall %.1f us | host until enqueued %.1f us | wait %.1f us | events ev0->ev1 %.1f us" % tuple(med))

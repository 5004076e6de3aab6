"""Host-buffer C-ABI call (bench.py's e2e path) vs the device time it reports."""
import os
import statistics
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import numpy as np  # noqa: E402

from paper_1201_1548_b200 import _lib  # noqa: E402
from paper_1201_1548_b200.bivpoly import BivPoly  # noqa: E402
from paper_1201_1548_b200.planner import pack_grid, plan_resultant  # noqa: E402
from paper_1201_1548_b200.synth import make_pair  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
lib = _lib.lib()
f, g = make_pair(cfg, 0)
F, G = BivPoly(f), BivPoly(g)
fc, gc = F.coeffs_wrt_y(), G.coeffs_wrt_y()
pk = pack_grid(fc, gc)
p1 = plan_resultant(fc, gc, F.total_degree(), G.total_degree(), pk.dfx, pk.dgx)
hin = _lib.pinned.get("gap_in", pk.limbs.size)
hin[:] = pk.limbs.reshape(-1)
hout = _lib.pinned.get("gap_out", p1.N * p1.LW)
status = np.zeros(1, dtype=np.uint32)
ms = np.zeros(1, dtype=np.float32)
args = (_lib.ptr(hin), pk.C, pk.L, _lib.ptr(pk.degs), pk.m, pk.n, pk.dfx, pk.dgx, _lib.ptr(p1.primes),
        _lib.ptr(p1.gens), len(p1.primes), p1.N, p1.LW, _lib.ptr(hout), _lib.ptr(status), _lib.ptr(ms))
for _ in range(5):
    lib.ckb_biv_resultant(*args)
wall, dev = [], []
for _ in range(50):
    t0 = time.perf_counter()
    lib.ckb_biv_resultant(*args)
    wall.append(time.perf_counter() - t0)
    dev.append(float(ms[0]))
args_nodev = args[:-1] + (None,)
wall2 = []
for _ in range(50):
    t0 = time.perf_counter()
    lib.ckb_biv_resultant(*args_nodev)
    wall2.append(time.perf_counter() - t0)
print(f"{cfg}: wall {1e3 * statistics.median(wall):.4f} ms, device incl. copies {statistics.median(dev):.4f} ms, "
      f"wall without device_ms {1e3 * statistics.median(wall2):.4f} ms, out {hout.nbytes} B")

"""Per-rank device work of the sharded res_y at 1/2/4/8 GPUs, measured on ONE GPU.

A rank of an N-GPU run does: modular images for its K/N primes (reduce,
choose_c, images, interpolation) and, with the coefficient-sharded CRT
(SURVEY §8e option B), the CRT of all K primes for N_pts/N coefficients; with
option A rank 0 runs the CRT of all coefficients.  Each part is timed here
alone (CUDA events, L2 flushed), the collective in between is not (one GPU).
"""
import argparse
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1201_1548_b200 import _lib  # noqa: E402
from paper_1201_1548_b200.bivpoly import BivPoly  # noqa: E402
from paper_1201_1548_b200.distributed import CudaBackend, plan_sharded  # noqa: E402
from paper_1201_1548_b200.synth import make_pair  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg4")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--worlds", default="1,2,4,8")
args = ap.parse_args()

dev = torch.device("cuda", 0)
lib = _lib.lib()
f, g = make_pair(args.config, 0)
F, G = BivPoly(f), BivPoly(g)
fc, gc = F.coeffs_wrt_y(), G.coeffs_wrt_y()
st = torch.cuda.Stream(dev)
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)


def timed(fn):
    ts = []
    for i in range(args.reps + 3):
        with torch.cuda.stream(st):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
        e1.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


for world in [int(w) for w in args.worlds.split(",")]:
    plan = plan_sharded(fc, gc, F.total_degree(), G.total_degree(), world)
    be = CudaBackend(fc, gc, dev)
    primes, gens = plan.shard(0)
    t_img = timed(lambda: be.modular_images(primes, gens, plan.N, st.cuda_stream))
    lib.ckb_set_timing(1)
    acc = np.zeros(4)
    for _ in range(args.reps):
        with torch.cuda.stream(st):
            flush.zero_()
        be.modular_images(primes, gens, plan.N, st.cuda_stream)
        sm = np.zeros(8, dtype=np.float32)
        n = lib.ckb_stage_times(_lib.ptr(sm), 8)
        acc += sm[:4] if n >= 4 else 0
    lib.ckb_set_timing(0)
    stages = " ".join(f"{k} {v * 1e3 / args.reps:.1f}" for k, v in zip(("reduce", "choose", "images", "interp"), acc))
    Nc = -(-plan.N // world)
    coeffs = torch.randint(0, 1 << 29, (len(plan.primes), Nc), dtype=torch.int32, device=dev)
    out = torch.empty((Nc, plan.LW), dtype=torch.int32, device=dev)
    hp = np.array(plan.primes, dtype=np.uint32)

    def crt():
        _lib.check(lib.ckb_dev_crt(coeffs.data_ptr(), len(plan.primes), Nc, _lib.ptr(hp), plan.LW, out.data_ptr(),
                                   st.cuda_stream), "ckb_dev_crt")
    t_crt = timed(crt)
    coeffs_all = torch.randint(0, 1 << 29, (len(plan.primes), plan.N), dtype=torch.int32, device=dev)
    out_all = torch.empty((plan.N, plan.LW), dtype=torch.int32, device=dev)

    def crt_all():
        _lib.check(lib.ckb_dev_crt(coeffs_all.data_ptr(), len(plan.primes), plan.N, _lib.ptr(hp), plan.LW,
                                   out_all.data_ptr(), st.cuda_stream), "ckb_dev_crt")
    t_crt_all = timed(crt_all)
    print(f"{args.config} world {world}: K {len(plan.primes)} ({plan.per_rank}/rank), images+interp {t_img * 1e3:.1f} us, "
          f"CRT of N/{world} coefficients {t_crt * 1e3:.1f} us (option B), CRT of all {t_crt_all * 1e3:.1f} us "
          f"(option A, rank 0); stages (us): {stages}", flush=True)

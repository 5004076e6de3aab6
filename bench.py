#!/usr/bin/env python
"""Benchmark of the B200 multi-modular resultant (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg4] [--impl ours|reference]

Workload: cfg4 of BASELINE.json -- res_y(f, g) for random dense degree-40
bivariates with 64-bit coefficients (synthetic, seed 0; SURVEY.md §8(d)
generator).  A step is one complete res_y (reduce -> plan -> fused
evaluation + resultant per (prime, point) -> interpolation -> CRT to limbs).
  value  res_y per second with inputs resident in HBM (device time, CUDA
         events on the launching stream, L2 flushed between steps, max over
         ranks); at N > 1 the primes are sharded, one NCCL all-to-all gives
         every rank all residues of its block of N/W coefficients and each rank
         lifts its block by CRT (strong scaling; SURVEY §8e option B).
  e2e    the same metric through the C-ABI call with HOST buffers
         (ckb_biv_resultant: H2D of the limbs, D2H of the result limbs; at
         N > 1 per rank: H2D of the limbs, D2H of its coefficient block), plus
         the Python-level time of modpoly.biv_resultant (packing, planning and
         int conversion) reported beside it.
  --impl reference: the CPU reference path -- the C port of the reference's
         res_y (oracle/, all host threads) computing the complete workload per
         step (the steps that fit a ~150 s budget are run and reported), with
         the unmodified Python reference (baseline/_ref) timed beside it on a
         bounded sample and extrapolated (cpu_baseline.python).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

from paper_1201_1548_b200.bivpoly import BivPoly  # noqa: E402
from paper_1201_1548_b200.synth import CONFIGS, make_pair  # noqa: E402

METRIC = "res_y(f,g) wall time & modular images/sec at 1/2/4/8 B200 vs CPU ref"
UNIT = "res_y/s"


def workload(config):
    d, bits, kind = CONFIGS[config]
    f, g = make_pair(config, 0)
    F, G = BivPoly(f), BivPoly(g)
    return F, G, {"workload": f"{config}: res_y(f,{'f_y' if kind == 'fy' else 'g'}) dense total degree {d}, "
                              f"{bits}-bit coefficients, seed 0", "degree": d, "coeff_bits": bits}


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------

_NVML_POLL = r"""
import sys, time
import pynvml
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
bits = [pynvml.nvmlClocksThrottleReasonHwSlowdown, pynvml.nvmlClocksThrottleReasonHwThermalSlowdown,
        pynvml.nvmlClocksThrottleReasonSwThermalSlowdown, pynvml.nvmlClocksThrottleReasonSwPowerCap]
mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
out = sys.stdout
while True:
    sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
    rs = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
    out.write("%d %d %d %s\n" % (time.monotonic_ns(), sm, mx, "".join("1" if rs & b else "0" for b in bits)))
    out.flush()
    time.sleep(0.002)
"""


class Clocks:
    """SM clock and throttle reasons sampled DURING the timed region.

    A separate process polls NVML (nvidia-ml-py) every ~2 ms with monotonic
    timestamps (no contention with this process's GIL); the samples inside the
    timed window are kept (faster polling measurably perturbs a 0.06 ms step:
    cfg2 +6% at 0.5 ms).  Without NVML: `nvidia-smi -lms 100`."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []      # nvidia-smi rows, or NVML lines "t sm max bits"
        self.proc = None
        self.nvml = False
        self.t0 = self.t1 = None

    def _start(self, cmd, nvml):
        self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        self.nvml = nvml
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def __enter__(self):
        started = False
        if not os.environ.get("CKB_BENCH_NO_NVML"):
            try:
                import pynvml  # noqa: F401
                self._start([sys.executable, "-c", _NVML_POLL, str(self.index)], True)
                deadline = time.time() + 20
                while not self.rows and self.proc.poll() is None and time.time() < deadline:
                    time.sleep(0.01)
                started = bool(self.rows)
                if not started:
                    self._stop()
            except (ImportError, OSError):
                started = False
        if not started:
            try:
                self.rows = []
                self._start(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                             "--format=csv,noheader,nounits", "-lms", "100"], False)
            except OSError:
                self.proc = None
        self.t0 = time.monotonic_ns()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append(line.strip())

    def _stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def __exit__(self, *a):
        self.t1 = time.monotonic_ns()
        if self.proc and not self.nvml:
            time.sleep(0.25)
        elif self.proc:
            time.sleep(0.002)  # let the poller report past the end of the window
        self._stop()

    def summary(self):
        if self.nvml:
            pts = []
            for r in self.rows:
                f = r.split()
                if len(f) == 4 and f[0].isdigit():
                    pts.append((int(f[0]), int(f[1]), int(f[2]), f[3]))
            inside = [x for x in pts if self.t0 <= x[0] <= self.t1]
            # a window shorter than the poll period still gets its nearest samples
            use = inside or sorted(pts, key=lambda x: abs(x[0] - (self.t0 + self.t1) // 2))[:2]
            if use:
                sm = [x[1] for x in use]
                reasons = sorted({n for x in use for n, bit in zip(self.NAMES, x[3]) if bit == "1"})
                return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(x[2] for x in use), "sm_min_mhz": min(sm),
                        "reasons": reasons, "samples": len(use), "samples_in_window": len(inside),
                        "window_ms": (self.t1 - self.t0) / 1e6, "source": "nvml (separate process)"}
        rows = [[x.strip() for x in r.split(",")] for r in self.rows if "," in r]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[k] for r in rows for k in range(4) if len(r) > 5 + k and r[5 + k] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "source": "nvidia-smi"}


# ---------------------------------------------------------------------------
# CPU reference (oracle port of modpoly.py's loop) on a bounded sample
# ---------------------------------------------------------------------------

def cpu_reference(F, G, target_s: float = 12.0, threads=None):
    """Time the reference's per-prime loop body (modpoly.py:376-391, ported to C,
    all host threads) on a sample of its own primes; extrapolate to one res_y."""
    from oracle import oracle
    threads = threads or os.cpu_count() or 1
    fc, gc = F.coeffs_wrt_y(), G.coeffs_wrt_y()
    m, n = len(fc) - 1, len(gc) - 1
    npts = F.deg_x() * n + G.deg_x() * m + 1          # the reference's point count (:371)
    bound = oracle.det_coeff_bound(fc, gc)
    stream = oracle._stream(0)
    k_ref, mod = 0, 1
    while mod <= 2 * bound:
        mod *= stream[k_ref]
        k_ref += 1
    # calibrate: one prime on one thread
    t0 = time.perf_counter()
    oracle.prime_images(fc, gc, [stream[0]], npts, threads=1)
    t1 = time.perf_counter() - t0
    per_round = t1  # one prime per thread per round
    rounds = max(1, min(8, int(target_s / max(per_round, 1e-3))))
    sample = min(k_ref, threads * rounds)
    t0 = time.perf_counter()
    oracle.prime_images(fc, gc, list(stream[:sample]), npts, threads=threads)
    ts = time.perf_counter() - t0
    t_res = ts * k_ref / sample
    return {"value": 1.0 / t_res, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"{sample} of {k_ref} primes of the reference loop body (modpoly.py:376-391, "
                      f"{npts} points/prime, C port, {threads} threads) in {ts:.2f} s; res_y time "
                      f"extrapolated x{k_ref}/{sample} = {t_res:.1f} s",
            "seconds_per_res_y": t_res, "images_per_s": sample * npts / ts,
            "one_prime_one_thread_s": t1}


def python_reference(config, target_s: float = 10.0):
    """The UNMODIFIED Python reference (baseline/_ref, curvekit.modpoly) on one
    core: its own loop body (modpoly.py:376-391: _zp_eval of every y-coefficient,
    _zp_resultant, then _zp_interp) on the first prime of its stream, timed on a
    sample of points, with _zp_interp timed at a reduced point count and scaled
    by its exact O(n^2) operation count; per-prime time x the reference's prime
    count = one res_y.  Returns None when baseline/_ref is absent."""
    import importlib
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "curvekit")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    RM = importlib.import_module("curvekit.modpoly")
    RB = importlib.import_module("curvekit.bivpoly")
    f, g = make_pair(config, 0)
    F, G = RB.BivPoly(f), RB.BivPoly(g)
    fc, gc = F.coeffs_wrt_y(), G.coeffs_wrt_y()
    m, n = len(fc) - 1, len(gc) - 1
    bound = RM._det_coeff_bound(fc, gc)
    npts = F.deg_x() * n + G.deg_x() * m + 1
    k_ref, mod, first = 0, 1, None
    for p in RM.prime_stream(0):
        if mod > 2 * bound:
            break
        if not RM._zp_trim([c % p for c in fc[-1]]) or not RM._zp_trim([c % p for c in gc[-1]]):
            continue
        first = first or p
        mod *= p
        k_ref += 1
    p = first
    t0 = time.perf_counter()
    fpc = [[c % p for c in cf] for cf in fc]
    gpc = [[c % p for c in cg] for cg in gc]
    t_red = time.perf_counter() - t0
    pts, vals, t = [], [], 0
    t0 = time.perf_counter()
    while len(pts) < npts and time.perf_counter() - t0 < 0.45 * target_s:
        if RM._zp_eval(fpc[-1], t, p) and RM._zp_eval(gpc[-1], t, p):
            fu = RM._zp_trim([RM._zp_eval(cf, t, p) for cf in fpc])
            gu = RM._zp_trim([RM._zp_eval(cg, t, p) for cg in gpc])
            pts.append(t)
            vals.append(RM._zp_resultant(fu, gu, p))
        t += 1
    t_pt = (time.perf_counter() - t0) / len(pts)
    ns = min(npts, 200)
    while True:  # interpolation sample sized to ~45% of the budget
        xs = list(range(ns))
        vs = [(7 * i + 3) % p for i in range(ns)]
        t0 = time.perf_counter()
        RM._zp_interp(xs, vs, p)
        t_int = time.perf_counter() - t0
        if ns >= npts or t_int > 0.12 * target_s:
            break
        ns = min(npts, int(ns * 1.6) + 1)
    t_interp = t_int * (npts * (npts - 1)) / (ns * (ns - 1))
    per_prime = t_red + t_pt * npts + t_interp
    t_res = per_prime * k_ref
    return {"value": 1.0 / t_res, "unit": UNIT, "cores": 1, "kind": "python",
            "sample": f"unmodified reference (baseline/_ref curvekit.modpoly, pure Python, 1 core): loop body "
                      f"modpoly.py:376-391 on prime {p}: {len(pts)} of {npts} points (eval + _zp_resultant, "
                      f"{t_pt * 1e3:.2f} ms/point), _zp_interp at {ns} points ({t_int:.2f} s) scaled by "
                      f"n(n-1) to {npts} ({t_interp:.1f} s); per prime {per_prime:.1f} s x {k_ref} primes",
            "seconds_per_res_y": t_res}


def run_reference(args):
    """The reference arm: the C port of the reference's res_y (oracle/ckoracle.c:
    modpoly.py:348-394 with its per-prime loop body in C on every host thread,
    Garner CRT in Python ints) computing the COMPLETE workload per step -- no
    extrapolation; the steps actually run are capped by a time budget so the run
    ends within a few minutes and reported as such.  The unmodified Python
    reference is timed beside it on a bounded sample (cpu_baseline.python)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle
    threads = os.cpu_count() or 1
    F, G, cfg = workload(args.config)
    f, g = make_pair(args.config, 0)
    budget = float(os.environ.get("CKB_REF_BUDGET_S", "150"))
    times, first = [], None
    t_start = time.perf_counter()
    for _ in range(args.steps):
        t0 = time.perf_counter()
        res = oracle.biv_resultant(f, g, "y", threads=threads)
        times.append(time.perf_counter() - t0)
        first = first or res
        assert res == first
        if time.perf_counter() - t_start + times[-1] > budget:
            break
    wall = time.perf_counter() - t_start
    s_step = statistics.median(times)
    v = 1.0 / s_step
    py = python_reference(args.config, target_s=min(args.ref_seconds, 12.0))
    cb = {"value": v, "unit": UNIT, "cores": threads, "kind": "port",
          "sample": f"{len(times)} complete res_y of the workload by the C port of the reference "
                    f"(oracle.biv_resultant: modpoly.py:348-394, {threads} threads), {wall:.1f} s wall",
          "python": py}
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus, "steps": len(times),
            "steps_requested": args.steps, "warmup": 0, "ms_per_step": 1e3 * s_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32 (mod p < 2^31), exact integers",
            "data": "synthetic", "config": cfg, "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def run_devices(args, devices):
    """--gpus N outside torchrun: ONE process drives N devices through the C-ABI
    (ckb_init_devices + ckb_biv_resultant_multi: primes sharded over the
    device contexts, NCCL residue exchange over NVLink, coefficient-sharded
    CRT), i.e. the drop-in modpoly.biv_resultant with CKB_GPUS=N.  A step is one
    complete call with host buffers (page-locked), so value and e2e coincide
    here: value is the device time (CUDA events per context, max over
    contexts, copies included), e2e the wall time of the call."""
    import ctypes
    from paper_1201_1548_b200 import _lib, modpoly
    from paper_1201_1548_b200.planner import limbs_to_ints, plan_resultant

    lib = _lib.load()
    arr = (ctypes.c_int * len(devices))(*devices)
    _lib.check(lib.ckb_init_devices(len(devices), ctypes.cast(arr, ctypes.c_void_p)), "ckb_init_devices")
    _lib._ready = True
    G = len(devices)
    F, G_, cfg = workload(args.config)
    fc, gc = F.coeffs_wrt_y(), G_.coeffs_wrt_y()
    from paper_1201_1548_b200.planner import pack_grid
    pk = pack_grid(fc, gc)
    p1 = plan_resultant(fc, gc, F.total_degree(), G_.total_degree(), pk.dfx, pk.dgx)
    K, N, LW = len(p1.primes), p1.N, p1.LW
    hlimbs = _lib.pinned.get("bench_in", pk.limbs.size)
    hlimbs[:] = pk.limbs.reshape(-1)
    hout = _lib.pinned.get("bench_out", N * LW)
    status = np.zeros(1, dtype=np.uint32)
    ms = np.zeros(1, dtype=np.float32)
    args_c = (_lib.ptr(hlimbs), pk.C, pk.L, _lib.ptr(pk.degs), pk.m, pk.n, pk.dfx, pk.dgx, _lib.ptr(p1.primes),
              _lib.ptr(p1.gens), K, N, LW, G, _lib.ptr(hout), _lib.ptr(status), _lib.ptr(ms))
    t_cold = time.perf_counter()
    _lib.check(lib.ckb_biv_resultant_multi(*args_c), "ckb_biv_resultant_multi")
    t_cold = time.perf_counter() - t_cold
    got = modpoly._trim(limbs_to_ints(hout, N, LW))
    for _ in range(args.warmup):
        _lib.check(lib.ckb_biv_resultant_multi(*args_c), "ckb_biv_resultant_multi")
    n0 = lib.ckb_launch_count()
    dev_ms, wall = [], []
    with Clocks(devices[0]) as clk:
        for _ in range(args.steps):
            t0 = time.perf_counter()
            _lib.check(lib.ckb_biv_resultant_multi(*args_c), "ckb_biv_resultant_multi")
            wall.append(time.perf_counter() - t0)
            dev_ms.append(float(ms[0]))
    launches = int(lib.ckb_launch_count() - n0)
    again = modpoly._trim(limbs_to_ints(hout, N, LW))
    assert again == got, "replayed multi-device call differs from its first result"
    # the one-context result of the same library (bit-exact equality across device counts)
    one = np.zeros(N * LW, dtype=np.uint32)
    _lib.check(lib.ckb_biv_resultant(*args_c[:13], _lib.ptr(one), _lib.ptr(status), None), "ckb_biv_resultant")
    assert modpoly._trim(limbs_to_ints(one, N, LW)) == got, "multi-device result differs from one device"
    ms_step = sum(dev_ms) / len(dev_ms)
    e_ms = 1e3 * statistics.median(wall)
    line = {"metric": METRIC, "value": 1e3 / ms_step, "unit": UNIT, "n_gpus": G, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32 (mod p < 2^30), exact integers", "data": "synthetic",
            "config": dict(cfg, primes=K, points_per_prime=N, out_words=LW, devices=list(devices),
                           parallelism=f"one process, {G} device contexts: primes/{G}, "
                                       f"{_lib.last_exchange()} exchange, CRT coefficients/{G}",
                           l2="inputs from page-locked host memory every step (H2D + D2H inside the timed call)"),
            "value_note": "device time per call incl. its H2D/D2H (CUDA events per context, max over contexts)",
            "cold_first_call_ms": t_cold * 1e3, "clocks": clk.summary(), "gpu_launches": launches,
            "e2e": {"value": 1e3 / e_ms, "unit": UNIT, "ms_per_step": e_ms,
                    "h2d_bytes_per_step": int(pk.limbs.nbytes + pk.degs.nbytes) * G,
                    "d2h_bytes_per_step": int(N * LW * 4 + 4 * G),
                    "path": "ckb_biv_resultant_multi (C-ABI, one process, page-locked host buffers)"},
            "cpu_baseline": None}
    emit(line)
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1201_1548_b200 import _lib, modpoly, workmodel
    from paper_1201_1548_b200.distributed import (CudaBackend, gather_limbs, plan_sharded,
                                                  sharded_resultant_step_a2a)
    from paper_1201_1548_b200.planner import limbs_to_ints, pack_grid, plan_resultant

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ["CKB_DEVICE"] = str(local)
    sharded = world > 1 or args.sharded  # --sharded: the N > 1 code path on one rank (tests it)
    if sharded and "RANK" not in os.environ:  # --sharded without torchrun: a one-rank group
        os.environ.update({"RANK": "0", "WORLD_SIZE": "1", "LOCAL_RANK": "0", "MASTER_ADDR": "127.0.0.1",
                           "MASTER_PORT": os.environ.get("MASTER_PORT", "29533")})
    if sharded:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    lib = _lib.lib()
    F, G, cfg = workload(args.config)
    fc, gc = F.coeffs_wrt_y(), G.coeffs_wrt_y()
    tdf, tdg = F.total_degree(), G.total_degree()
    plan = plan_sharded(fc, gc, tdf, tdg, world)
    K, N, LW = len(plan.primes), plan.N, plan.LW
    backend = CudaBackend(fc, gc, dev)
    pk = backend.packed
    stream = torch.cuda.Stream(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device=dev)  # > 126 MB L2

    def barrier():
        if sharded:
            dist.barrier(device_ids=[local])

    hp_all = np.array(plan.primes, dtype=np.uint32)
    hg_all = np.array(plan.gens, dtype=np.uint32)
    d_out1 = torch.empty((N, LW), dtype=torch.int32, device=dev) if not sharded else None

    def step():
        if not sharded:  # the whole pipeline in one C-ABI call (replayed as a CUDA graph)
            _lib.check(lib.ckb_dev_biv_resultant(
                backend.d_limbs.data_ptr(), pk.C, pk.L, backend.d_degs.data_ptr(), _lib.ptr(backend.h_degs),
                pk.m, pk.n, pk.dfx, pk.dgx, _lib.ptr(hp_all), _lib.ptr(hg_all), K, N, LW, d_out1.data_ptr(),
                backend.d_status.data_ptr(), stream.cuda_stream), "ckb_dev_biv_resultant")
            return d_out1
        # primes sharded, residues exchanged by one all-to-all, every rank lifts
        # its coefficient block by CRT (SURVEY §8e option B); the step ends with
        # each rank's [N/W][LW] limbs in its HBM
        with torch.cuda.stream(stream):
            return sharded_resultant_step_a2a(backend, plan, rank, world, None, stream.cuda_stream)

    def assemble(blk):  # outside the timed region: all limb blocks on rank 0
        if not sharded:
            return blk
        with torch.cuda.stream(stream):
            full = gather_limbs(blk, plan, rank, world)
        torch.cuda.synchronize()
        return full

    # correctness of the timed path against the single-call API (rank 0)
    t_cold = time.perf_counter()
    out = step()
    torch.cuda.synchronize()
    t_cold = time.perf_counter() - t_cold
    out = assemble(out)
    if rank == 0:
        got = modpoly._trim(limbs_to_ints(out.cpu().numpy().view(np.uint32).reshape(-1), N, LW))
        ref, _ = modpoly._biv_resultant_gpu(fc, gc, tdf, tdg)
        assert got == ref, "sharded result differs from the single-GPU result"
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    graph, graph_launches = None, 0
    if sharded and not args.no_step_graph:
        # the whole sharded step (library kernels, the strided copy and the NCCL
        # all-to-all) as ONE CUDA graph: at 8 ranks a step is ~0.1 ms of device
        # work, comparable to enqueueing its parts from Python
        lib.ckb_set_graphs(0)
        try:
            graph = torch.cuda.CUDAGraph()
            c0 = lib.ckb_launch_count()
            with torch.cuda.graph(graph, stream=stream):
                graph_out = step()
            graph_launches = int(lib.ckb_launch_count() - c0)  # library kernels per replay
        except Exception as exc:  # noqa: BLE001 - fall back to enqueueing the parts (same on every rank)
            print(f"step graph capture failed, enqueueing the step's parts: {exc}", file=sys.stderr)
            graph, graph_launches = None, 0
        lib.ckb_set_graphs(1)
        torch.cuda.synchronize()
        barrier()
        if graph is not None:
            def step():  # noqa: F811 - replay the captured step
                graph.replay()
                return graph_out
    n0 = lib.ckb_launch_count()
    times = []
    with Clocks(local) as clk:
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                step()
                e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    launches = int(lib.ckb_launch_count() - n0) + (graph_launches * args.steps if graph is not None else 0)
    # the timed (graph-replayed) path still gives the reference's result; every
    # rank takes part in the step (it contains the collective), rank 0 checks
    last = assemble(step())
    torch.cuda.synchronize()
    if rank == 0 and last is not None:
        got2 = modpoly._trim(limbs_to_ints(last.cpu().numpy().view(np.uint32).reshape(-1), N, LW))
        assert got2 == ref, "replayed pipeline differs from the single-call API"
    barrier()
    torch.cuda.synchronize()
    tot = torch.tensor([sum(times)], dtype=torch.float64, device=dev)
    if sharded:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms_per_step = float(tot.item()) / args.steps
    clocks = clk.summary()

    # stage breakdown of the single-GPU pipeline (CUDA events between launches)
    stages = None
    peak = np.zeros(5, dtype=np.float32)
    if rank == 0:
        _lib.check(lib.ckb_measure_peak(_lib.ptr(peak), 5), "ckb_measure_peak")
        lib.ckb_set_timing(1)
        acc = np.zeros(5)
        reps = max(3, args.steps)
        d_out = torch.empty((N, LW), dtype=torch.int32, device=dev)
        hp = np.array(plan.primes, dtype=np.uint32)
        hg = np.array(plan.gens, dtype=np.uint32)
        for _ in range(reps):
            with torch.cuda.stream(stream):
                flush.zero_()
            _lib.check(lib.ckb_dev_biv_resultant(
                backend.d_limbs.data_ptr(), pk.C, pk.L, backend.d_degs.data_ptr(), _lib.ptr(backend.h_degs),
                pk.m, pk.n, pk.dfx, pk.dgx, _lib.ptr(hp), _lib.ptr(hg), K, N, LW, d_out.data_ptr(),
                backend.d_status.data_ptr(), stream.cuda_stream), "ckb_dev_biv_resultant")
            st = np.zeros(8, dtype=np.float32)
            cnt = lib.ckb_stage_times(_lib.ptr(st), 8)
            acc += st[:5] if cnt >= 5 else 0
        lib.ckb_set_timing(0)
        stages = dict(zip(["reduce", "choose_c", "images", "interp", "crt"], (acc / reps).tolist()))

    # e2e: through the C-ABI with host buffers (rank 0, single GPU), and the Python API;
    # at N > 1 every rank copies the input limbs from pinned memory, runs the sharded
    # step and reads its coefficient block back into pinned memory (max over ranks)
    e2e = None
    if sharded:
        h_in = torch.from_numpy(pk.limbs.view(np.int32).copy()).pin_memory()
        h_out = torch.empty((-(-N // world), LW), dtype=torch.int32).pin_memory()
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        barrier()
        et = 0.0
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            stream.synchronize()
            barrier()
            t0 = time.perf_counter()
            with torch.cuda.stream(stream):
                backend.d_limbs.copy_(h_in, non_blocking=True)
                blk = step()
                h_out.copy_(blk, non_blocking=True)
            stream.synchronize()
            et += time.perf_counter() - t0
        tt = torch.tensor([et], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e_ms = 1e3 * float(tt.item()) / args.steps
        e2e = {"value": 1e3 / e_ms, "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(pk.limbs.nbytes), "d2h_bytes_per_step": int(h_out.numel() * 4),
               "path": "SPMD over NCCL: per rank H2D of the input limbs (pinned), sharded step, D2H of the "
                       "rank's coefficient block (pinned); max over ranks, wall clock per step"}
    if rank == 0 and not sharded:
        p1 = plan_resultant(fc, gc, tdf, tdg, pk.dfx, pk.dgx)
        # page-locked host buffers, as the e2e contract states (inputs copied from pinned memory)
        hlimbs = _lib.pinned.get("bench_in", pk.limbs.size)
        hlimbs[:] = pk.limbs.reshape(-1)
        hout = _lib.pinned.get("bench_out", p1.N * p1.LW)
        status = np.zeros(1, dtype=np.uint32)
        args_c = (_lib.ptr(hlimbs), pk.C, pk.L, _lib.ptr(pk.degs), pk.m, pk.n, pk.dfx, pk.dgx,
                  _lib.ptr(p1.primes), _lib.ptr(p1.gens), len(p1.primes), p1.N, p1.LW, _lib.ptr(hout),
                  _lib.ptr(status), None)
        for _ in range(args.warmup):
            lib.ckb_biv_resultant(*args_c)
        et = []
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.zero_()
            stream.synchronize()
            t0 = time.perf_counter()
            _lib.check(lib.ckb_biv_resultant(*args_c), "ckb_biv_resultant")
            et.append(time.perf_counter() - t0)
        pt = []
        for _ in range(max(3, args.steps // 2)):
            t0 = time.perf_counter()
            modpoly.biv_resultant(F, G, "y")
            pt.append(time.perf_counter() - t0)
        e_ms = 1e3 * statistics.median(et)
        # share of the images the register kernel handed to the fallback (last C-ABI call)
        fb, nimg = _lib.last_fallback()
        e2e = {"value": 1e3 / e_ms, "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(pk.limbs.nbytes + pk.degs.nbytes + 4 * len(p1.gens)),
               "d2h_bytes_per_step": int(hout.nbytes + 4),
               "path": "ckb_biv_resultant (C-ABI, page-locked host buffers: H2D of the input and the result written into host memory by the CRT carry kernel (zero copy), both inside the timed region)",
               "python_api_ms": 1e3 * statistics.median(pt),
               "python_api_note": "modpoly.biv_resultant incl. packing, planning, int conversion"}

    if sharded:
        fb, nimg = 0, 0  # (the sharded step's kernels run through ckb_dev_modular_images)
    if rank == 0:
        dfs = [len(c) - 1 for c in fc]
        dgs = [len(c) - 1 for c in gc]
        img_prod = workmodel.images_products(pk.m, pk.n, dfs, dgs, K, N)
        p_shoup, p_mont = workmodel.images_products_split(pk.m, pk.n, dfs, dgs, K, N)
        t_img = stages["images"] * 1e-3
        achieved = img_prod / t_img / 1e12
        # ideal time of this product mix at the measured peaks of its two forms
        t_ideal = p_shoup / (float(peak[3]) * 1e12) + p_mont / (float(peak[4]) * 1e12)
        mix_peak = img_prod / t_ideal / 1e12
        traffic = None
        try:
            with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")) as fh:
                if args.config == "cfg4":
                    traffic = json.load(fh)["dram_bytes_per_launch"]["k_images"]
        except (OSError, KeyError, ValueError):
            traffic = None
        contract = workmodel.contract_imad(pk.m, pk.n, dfs, dgs, K, N, pk.C, pk.L)
        images = K * N
        cpu = cpu_reference(F, G, target_s=args.ref_seconds) if (world == 1 and not args.no_cpu) else None
        if cpu is not None:  # the unmodified Python reference beside the C port
            cpu["python"] = python_reference(args.config, target_s=min(args.ref_seconds, 12.0))
        line = {
            "metric": METRIC, "value": 1e3 / ms_per_step, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32 (mod p < 2^30), exact integers", "data": "synthetic",
            "config": dict(cfg, primes=K, points_per_prime=N, images_per_res_y=images, out_words=LW,
                           l2="flushed (256 MB write) before every timed step",
                           step_graph=bool(graph is not None), parallelism=(f"primes/{world}" if not sharded else
                                        f"primes/{world}, all-to-all, CRT coefficients/{world}")),
            "images_per_s": images * 1e3 / ms_per_step,
            "fallback": {"images": fb, "of": nimg, "share": fb / max(1, nimg),
                         "note": "images whose remainder sequence is not generic, recomputed one thread per "
                                 "image by the any-degree elimination (k_images_fallback_reg); structured inputs "
                                 "(an interior y-coefficient identically zero) run it in the register kernel itself"},
            "stages_ms": stages,
            "stages_note": ("CUDA events between the stages of one single-GPU pipeline call (timing mode: no graph)"
                            + ("" if world == 1 else "; measured on rank 0's GPU alone")),
            "cold_first_call_ms": t_cold * 1e3,
            "cold_note": "first res_y of the process: builds the cached interpolation plan and CRT tables "
                         "(input-independent, keyed by primes and N, like an FFT plan); value is warm",
            "roofline": {"bound": "imad", "kernel": "k_images (fused eval + elimination)",
                         "achieved": achieved, "peak": mix_peak, "unit": "T modular products/s",
                         "frac": achieved / mix_peak,
                         "peak_source": "measured live (csrc/ckb_peak.cu), mix-weighted: "
                                        f"{p_shoup:.3e} Shoup-form products at the Shoup-pair rate "
                                        f"{float(peak[3]):.2f} T/s + {p_mont:.3e} fused-remainder products at the "
                                        f"three-product Montgomery rate {float(peak[4]):.2f} T/s",
                         "algorithmic_products_per_launch": img_prod, "traffic": traffic,
                         "traffic_source": "ncu dram__bytes_read+write of k_images (profiles/ncu_traffic.json)",
                         "imad_peaks_tops": {"imad": float(peak[0]), "imad_hi": float(peak[1]),
                                             "imad_wide": float(peak[2])},
                         "contract": {"survey_W_imad_per_res_y": contract,
                                      "achieved_tops": contract / (ms_per_step * 1e-3) / 1e12,
                                      "frac_of_measured_imad": contract / (ms_per_step * 1e-3) / 1e12 / float(peak[0])}},
            "clocks": clocks, "gpu_launches": launches, "e2e": e2e,
            "cpu_baseline": cpu,
        }
        emit(line)
    if sharded:
        dist.barrier(device_ids=[local])
        dist.destroy_process_group()
    return 0


_JSON_OUT = None


def emit(line: dict):
    """The ONE JSON line, on the real stdout (library chatter was sent to stderr)."""
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    # NCCL / CUDA libraries may print to fd 1 (e.g. "NCCL version ..."): route fd 1
    # to stderr and keep a private handle on the real stdout for the JSON line
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="run the multi-GPU (all-to-all) step even at N=1")
    ap.add_argument("--no-step-graph", action="store_true", help="N > 1: enqueue the step's parts from Python")
    ap.add_argument("--devices", default="", help="one process over these device ids (may repeat: contexts "
                    "sharing a GPU, a correctness configuration); default with --gpus N outside torchrun: 0..N-1")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    if args.devices or (args.gpus > 1 and "WORLD_SIZE" not in os.environ):
        # one process driving several devices (the drop-in's multi-GPU mode)
        devices = [int(x) for x in args.devices.split(",")] if args.devices else list(range(args.gpus))
        import torch
        have = torch.cuda.device_count()
        if max(devices) >= have:
            print(f"bench.py: --gpus {args.gpus} needs devices {devices} but only {have} CUDA device(s) "
                  "are visible", file=sys.stderr)
            return 2
        return run_devices(args, devices)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

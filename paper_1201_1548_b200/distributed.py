"""Primes sharded over GPUs, one process per GPU (torch.distributed over NCCL).

The path partitions naturally: every
prime's images and interpolation are independent; the only exchange is the
residue gather before the CRT (option A).  Rank r takes a
contiguous block of K/W primes (K rounded up to a multiple of W -- extra
primes only enlarge the CRT modulus, which leaves the symmetric lift
unchanged), runs reduce -> plan -> images -> interpolation on its GPU, the
[K/W][N] coefficient residues are all-gathered over NCCL into prime order,
and rank 0 runs the mixed-radix CRT and returns the integers.

The device stages are behind a small backend object so the sharding,
padding, collective and assembly logic is testable on CPU with gloo
(tests/test_distributed.py) while the GPU backend is the C-ABI library.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .planner import (choose_primes_log2, limbs_to_ints, log2_coeff_bound, pack_grid, point_count)
from .primes30 import PRIMES30


@dataclass
class ShardPlan:
    primes: list        # all K primes (K % world == 0), CRT order
    gens: list
    N: int
    LW: int
    per_rank: int

    def shard(self, rank: int):
        a = rank * self.per_rank
        return self.primes[a:a + self.per_rank], self.gens[a:a + self.per_rank]


def plan_sharded(fc, gc, tdf: int, tdg: int, world: int, table=PRIMES30, start: int = 0) -> ShardPlan:
    m, n = len(fc) - 1, len(gc) - 1
    dfx = max(0, max(len(c) - 1 for c in fc))
    dgx = max(0, max(len(c) - 1 for c in gc))
    N = point_count(fc, gc, dfx, dgx, tdf, tdg)
    primes, gens = choose_primes_log2(log2_coeff_bound(fc, gc), fc[-1], gc[-1], start, table)
    mod = 1
    for p in primes:
        mod *= p
    start = table.index((primes[-1], gens[-1])) + 1
    while len(primes) % world:  # pad with the next admissible primes
        if start >= len(table):
            raise ArithmeticError("prime table exhausted in resultant computation")
        p, g = table[start]
        start += 1
        if all(c % p == 0 for c in fc[-1]) or all(c % p == 0 for c in gc[-1]):
            continue
        primes.append(p)
        gens.append(g)
        mod *= p
    LW = (mod.bit_length() + 31) // 32
    return ShardPlan(primes, gens, N, LW, len(primes) // world)


class CudaBackend:
    """Device stages through the C-ABI (device pointers from torch tensors)."""

    def __init__(self, fc, gc, device):
        import torch
        from . import _lib
        self.torch = torch
        self._lib = _lib
        self.lib = _lib.lib()
        self.packed = pack_grid(fc, gc)
        pk = self.packed
        self.d_limbs = torch.from_numpy(pk.limbs.view(np.int32).copy()).to(device)
        self.d_degs = torch.from_numpy(pk.degs.copy()).to(device)
        self.h_degs = np.ascontiguousarray(pk.degs)
        self.device = device
        self.d_status = torch.zeros(1, dtype=torch.int32, device=device)

    def buffer(self, name, shape):
        """Device buffer reused across calls (stable addresses let the library
        replay its captured CUDA graph); valid until the next call asks for it."""
        cache = self.__dict__.setdefault("_bufs", {})
        buf = cache.get(name)
        if buf is None or tuple(buf.shape) != tuple(shape):
            buf = self.torch.empty(shape, dtype=self.torch.int32, device=self.device)
            cache[name] = buf
        return buf

    def modular_images(self, primes, gens, N, stream):
        pk = self.packed
        K = len(primes)
        hp = np.array(primes, dtype=np.uint32)
        hg = np.array(gens, dtype=np.uint32)
        out = self.buffer("images_out", (K, N))
        # the status word accumulates (atomicOr) over the launch: clear it per step
        self.d_status.zero_()
        self._lib.check(self.lib.ckb_dev_modular_images(
            self.d_limbs.data_ptr(), pk.C, pk.L, self.d_degs.data_ptr(), self._lib.ptr(self.h_degs), pk.m, pk.n,
            pk.dfx, pk.dgx, self._lib.ptr(hp), self._lib.ptr(hg), K, N, out.data_ptr(), self.d_status.data_ptr(),
            stream), "ckb_dev_modular_images")
        return out

    def crt(self, coeffs, primes, N, LW, stream):
        hp = np.array(primes, dtype=np.uint32)
        out = self.buffer("crt_out", (N, LW))
        self._lib.check(self.lib.ckb_dev_crt(coeffs.data_ptr(), len(primes), N, self._lib.ptr(hp), LW,
                                             out.data_ptr(), stream), "ckb_dev_crt")
        return out


def coeff_slice(plan: ShardPlan, rank: int, world: int) -> tuple:
    """Coefficients [a, b) whose CRT rank `rank` runs in the coefficient-sharded
    exchange (contiguous blocks of ceil(N / world); the last may be short)."""
    nc = -(-plan.N // world)
    a = min(plan.N, rank * nc)
    return a, min(plan.N, a + nc)


def sharded_resultant_step_a2a(backend, plan: ShardPlan, rank: int, world: int, group=None, stream=None):
    """One res_y with the coefficient-sharded CRT (SURVEY.md §8(e) option B).

    Rank r computes the [K/W][N] residues of its primes, one all-to-all
    transposes them so that rank r holds ALL K residues of its coefficient block
    coeff_slice(r) (the block sent to rank s is the column block s of the local
    residues, received in prime order because ranks own contiguous prime
    blocks), and every rank lifts its block by CRT.  Returns this rank's
    [nc][LW] limbs (rows past N, on the last rank, are zero coefficients).
    """
    import torch
    import torch.distributed as dist
    primes, gens = plan.shard(rank)
    local = backend.modular_images(primes, gens, plan.N, stream)
    nc = -(-plan.N // world)
    if world == 1 and not dist.is_initialized():
        recv = local
    else:
        reuse = getattr(backend, "buffer", None)
        kr = plan.per_rank
        shape = (world, kr, nc)
        send = reuse("a2a_send", shape) if reuse else torch.empty(shape, dtype=local.dtype, device=local.device)
        recv = reuse("a2a_recv", shape) if reuse else torch.empty(shape, dtype=local.dtype, device=local.device)
        src = local
        if world * nc != plan.N:  # zero coefficients pad the last block
            src = torch.nn.functional.pad(local, (0, world * nc - plan.N))
        # send[s] = column block s of the local residues (one strided copy)
        send.copy_(src.view(kr, world, nc).permute(1, 0, 2))
        dist.all_to_all_single(recv, send, group=group)
        recv = recv.reshape(world * kr, nc)  # rows: rank-major prime blocks = plan.primes order
    return backend.crt(recv, plan.primes, nc, plan.LW, stream)


def sharded_resultant_step(backend, plan: ShardPlan, rank: int, world: int, group=None, stream=None):
    """One res_y: local primes -> all_gather -> CRT on rank 0 (returns limbs tensor or None)."""
    import torch.distributed as dist
    primes, gens = plan.shard(rank)
    local = backend.modular_images(primes, gens, plan.N, stream)
    if world > 1:
        import torch
        shape = (world * plan.per_rank, plan.N)
        reuse = getattr(backend, "buffer", None)
        gathered = reuse("gathered", shape) if reuse else torch.empty(shape, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(gathered, local.contiguous(), group=group)
    else:
        gathered = local
    if rank != 0:
        return None
    return backend.crt(gathered, plan.primes, plan.N, plan.LW, stream)


def biv_resultant_distributed(f, g, var: str = "y", group=None, exchange: str = "a2a") -> list | None:
    """res_var(f, g) over all ranks of the default process group (SPMD call).

    Every rank passes the same f, g; rank 0 returns the coefficient list,
    the others return None.  exchange="a2a" (default): coefficient-sharded CRT
    after an all-to-all, the limb blocks gathered to rank 0; "gather": residues
    all-gathered, CRT on rank 0 (SURVEY.md §8(e) options B and A).
    """
    import torch
    import torch.distributed as dist
    from .bivpoly import as_biv
    from .modpoly import _pow, _trim
    f, g = as_biv(f), as_biv(g)
    if f.is_zero() or g.is_zero():
        raise ValueError("resultant of zero polynomial")
    if var == "x":
        f, g = f.swap(), g.swap()
    elif var != "y":
        raise ValueError("var must be 'x' or 'y'")
    fc, gc = f.coeffs_wrt_y(), g.coeffs_wrt_y()
    m, n = len(fc) - 1, len(gc) - 1
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if m == 0 and n == 0:
        return [1] if rank == 0 else None
    if m == 0 or n == 0:
        return (_pow(fc[0], n) if m == 0 else _pow(gc[0], m)) if rank == 0 else None
    device = torch.device("cuda", torch.cuda.current_device())
    backend = CudaBackend(fc, gc, device)
    s = torch.cuda.current_stream(device)
    start = 0
    for _attempt in range(4):
        plan = plan_sharded(fc, gc, f.total_degree(), g.total_degree(), world, start=start)
        with torch.cuda.stream(s):
            if exchange == "a2a":
                blk = sharded_resultant_step_a2a(backend, plan, rank, world, group, s.cuda_stream)
                out = gather_limbs(blk, plan, rank, world, group)
            else:
                out = sharded_resultant_step(backend, plan, rank, world, group, s.cuda_stream)
        # a prime without an admissible point scale (bit 1) or a vanishing leading
        # coefficient at a point (bit 2) on ANY rank invalidates the CRT: agree on
        # the worst status and re-plan with the next primes, as the single-GPU path does
        if status_any(backend.d_status, group):
            start += len(plan.primes)
            continue
        if rank != 0:
            return None
        host = out.cpu().numpy().view(np.uint32).reshape(-1)
        return _trim(limbs_to_ints(host, plan.N, plan.LW))
    raise ArithmeticError("no admissible evaluation points after re-planning")


def status_any(d_status, group=None) -> bool:
    """Max of every rank's status word (one all-reduce; a local read at world 1)."""
    import torch.distributed as dist
    st = d_status.clone()
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(st, op=dist.ReduceOp.MAX, group=group)
    return bool(int(st.item()))


def gather_limbs(blk, plan: ShardPlan, rank: int, world: int, group=None):
    """The [nc][LW] limb blocks of all ranks -> [N][LW] on rank 0 (None elsewhere)."""
    import torch
    import torch.distributed as dist
    if world == 1 and not dist.is_initialized():
        return blk[:plan.N]
    full = torch.empty((world * blk.shape[0], blk.shape[1]), dtype=blk.dtype, device=blk.device)
    dist.all_gather_into_tensor(full, blk.contiguous(), group=group)
    return full[:plan.N] if rank == 0 else None

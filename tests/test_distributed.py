"""The multi-GPU path's host logic on CPU: 2 ranks over gloo.

paper_1201_1548_b200.distributed shards the primes (padded to a multiple of
the world size), all-gathers the [K/W][N] coefficient residues in prime order
and lets rank 0 run the CRT.  Here the device stages are replaced by a CPU
backend built on the oracle (test infrastructure), so the sharding, padding,
collective and assembly logic is exercised exactly as on the GPUs.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import REPO, ints_in, load_golden, terms_in


class OracleBackend:
    """CPU stand-in for distributed.CudaBackend (oracle = checker only)."""

    def __init__(self, fc, gc):
        self.fc, self.gc = fc, gc

    def modular_images(self, primes, gens, N, stream):
        from oracle import oracle
        m, n = len(self.fc) - 1, len(self.gc) - 1
        dfx = max(len(c) - 1 for c in self.fc)
        dgx = max(len(c) - 1 for c in self.gc)
        npts = dfx * n + dgx * m + 1  # the reference's own point count (modpoly.py:371)
        out = torch.zeros((len(primes), N), dtype=torch.int64)
        for k, (rc, poly) in enumerate(oracle.prime_images(self.fc, self.gc, list(primes), npts, threads=1)):
            assert rc >= 0
            assert len(poly) <= N
            out[k, :len(poly)] = torch.tensor(poly, dtype=torch.int64)
        return out

    def crt(self, coeffs, primes, N, LW, stream):
        from oracle import oracle
        res = coeffs.tolist()
        return [oracle.crt_reconstruct(list(primes), [res[i][k] for i in range(len(primes))]) for k in range(N)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, cases, q, mode):
    import sys
    sys.path.insert(0, REPO)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle
    from paper_1201_1548_b200.distributed import (coeff_slice, plan_sharded, sharded_resultant_step,
                                                  sharded_resultant_step_a2a)
    try:
        for f, g, want in cases:
            fc, gc = oracle.coeffs_wrt_y(f), oracle.coeffs_wrt_y(g)
            tdf = max(i + j for i, j in f)
            tdg = max(i + j for i, j in g)
            plan = plan_sharded(fc, gc, tdf, tdg, world)
            assert len(plan.primes) % world == 0 and plan.per_rank * world == len(plan.primes)
            if mode == "gather":
                got = sharded_resultant_step(OracleBackend(fc, gc), plan, rank, world)
                if rank == 0:
                    while got and got[-1] == 0:
                        got.pop()
                    q.put(got == want)
                else:
                    assert got is None
            else:  # coefficient-sharded CRT after the all-to-all (option B)
                blk = sharded_resultant_step_a2a(OracleBackend(fc, gc), plan, rank, world)
                a, b = coeff_slice(plan, rank, world)
                assert len(blk) == -(-plan.N // world) and not any(blk[b - a:])
                blocks = [None] * world
                dist.all_gather_object(blocks, blk[:b - a])
                if rank == 0:
                    got = [v for bl in blocks for v in bl]
                    assert len(got) == plan.N
                    while got and got[-1] == 0:
                        got.pop()
                    q.put(got == want)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["gather", "a2a"])
@pytest.mark.parametrize("world", [2, 3])
def test_sharded_resultant_gloo(world, mode, small):
    cases = []
    for case in small["random50"][:6]:
        f, g = terms_in(case["f"]), terms_in(case["g"])
        if max(j for _, j in f) < 1 or max(j for _, j in g) < 1:
            continue
        cases.append((f, g, ints_in(case["res_y"])))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, cases, q, mode), nprocs=world, join=True, start_method="spawn")
    results = [q.get(timeout=5) for _ in cases]
    assert results and all(results)


def test_plan_sharded_pads_with_admissible_primes():
    from paper_1201_1548_b200.distributed import plan_sharded
    from paper_1201_1548_b200.primes30 import PRIMES30
    fc = [[5, 1], [0, 3], [7]]
    gc = [[1, 2, 3], [PRIMES30[0][0] * 3]]  # lc(g) vanishes mod the first table prime
    plan = plan_sharded(fc, gc, 2, 3, 4)
    assert len(plan.primes) % 4 == 0
    assert PRIMES30[0][0] not in plan.primes
    assert len(set(plan.primes)) == len(plan.primes)

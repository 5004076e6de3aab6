"""Randomised parity sweep (GPU vs the CPU oracle): biv_resultant over many
shapes (m != n, skewed x-degrees, sparse and dense, 4..200-bit coefficients, both
directions), the batched entry, and gcd_biv on planted factors.  Prints a summary;
exits non-zero on the first mismatch.  A one-off validation tool beside tests/."""
import os
import random
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from oracle import oracle  # noqa: E402  (the checker)

from paper_1201_1548_b200 import modpoly as mp  # noqa: E402
from paper_1201_1548_b200.bivpoly import BivPoly, divexact_cols, gcd_biv  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 1
count = int(sys.argv[2]) if len(sys.argv) > 2 else 200
rng = random.Random(seed)


def rnd_poly(dy, dx, bits, dens, ystep=1):
    t = {}
    for j in range(0, dy + 1, ystep):  # ystep > 1: F(x, y^ystep), structured (non-generic) sequences
        for i in range(dx + 1):
            if rng.random() < dens:
                c = rng.randint(-(2 ** bits), 2 ** bits)
                if c:
                    t[(i, j)] = c
    t[(rng.randint(0, dx), dy - dy % ystep)] = rng.choice([-1, 1]) * rng.randint(1, 2 ** bits)  # keep deg_y
    return t


t0 = time.time()
n_res = 0
batch = []
for it in range(count):
    m, n = rng.randint(1, 30), rng.randint(1, 30)
    dfx, dgx = rng.randint(0, 25), rng.randint(0, 25)
    bits = rng.choice([4, 10, 32, 64, 100, 200])
    dens = rng.choice([0.2, 0.5, 1.0])
    ystep = rng.choice([1, 1, 1, 2, 3])
    f, g = rnd_poly(m, dfx, bits, dens, ystep), rnd_poly(n, dgx, bits, dens, ystep)
    var = rng.choice("xy")
    got = mp.biv_resultant(f, g, var)
    want = oracle.biv_resultant(f, g, var)
    if got != want:
        print("MISMATCH", it, m, n, dfx, dgx, bits, dens, var)
        sys.exit(1)
    n_res += 1
    batch.append((f, g, var, want))
# the batched entry on the same problems, 4 per call
for i in range(0, len(batch), 4):
    chunk = batch[i:i + 4]
    got = mp.biv_resultant_batch([(f, g, v) for f, g, v, _ in chunk])
    if got != [w for *_, w in chunk]:
        print("BATCH MISMATCH", i)
        sys.exit(1)
n_gcd = 0
for it in range(count // 4):
    h = rnd_poly(rng.randint(1, 6), rng.randint(0, 6), rng.choice([4, 20, 40]), 0.7)
    a = rnd_poly(rng.randint(0, 6), rng.randint(0, 6), 16, 0.7)
    b = rnd_poly(rng.randint(0, 6), rng.randint(0, 6), 16, 0.7)
    H, A, Bq = BivPoly(h), BivPoly(a), BivPoly(b)

    def mul(x, y):
        out = {}
        for (i, j), c in x.items():
            for (k, l), d in y.items():
                out[(i + k, j + l)] = out.get((i + k, j + l), 0) + c * d
        return {k: v for k, v in out.items() if v}
    F, G = BivPoly(mul(h, a)), BivPoly(mul(h, b))
    gg = gcd_biv(F, G)
    # gcd divides both and the cofactors are coprime (gcd 1 up to content)
    fc, gc, dc = F.coeffs_wrt_y(), G.coeffs_wrt_y(), gg.coeffs_wrt_y()
    qa, qb = divexact_cols(fc, dc), divexact_cols(gc, dc)
    if qa is None or qb is None:
        print("GCD DOES NOT DIVIDE", it)
        sys.exit(1)
    co = gcd_biv(BivPoly({(i, j): c for j, col in enumerate(qa) for i, c in enumerate(col) if c}),
                 BivPoly({(i, j): c for j, col in enumerate(qb) for i, c in enumerate(col) if c}))
    if co.total_degree() != 0:
        print("COFACTORS NOT COPRIME", it)
        sys.exit(1)
    hd = gcd_biv(gg, H)  # h divides the gcd: gcd(gcd, h) == h up to sign and content
    if hd.total_degree() != H.total_degree():
        print("PLANTED FACTOR LOST", it)
        sys.exit(1)
    n_gcd += 1
print(f"seed {seed}: {n_res} resultants (+ batched), {n_gcd} planted gcds: all match ({time.time() - t0:.1f} s)")

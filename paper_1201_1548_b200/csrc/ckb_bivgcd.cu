// Images of a dense modular bivariate gcd: one warp per
// (prime, point) image.
//
// The reference computes gcd_biv (pkg/src/curvekit/bivpoly.py:266-295) with a
// primitive PRS over Z[x][y]; its cost grows with the coefficient swell of
// the PRS (32 s for is_squarefree_biv of one dense degree-16 curve with
// 32-bit coefficients).  The B200 path is Brown's dense modular algorithm:
// for primitive A, B (in y) and Gamma = gcd(lc_y A, lc_y B) in Z[x], the
// polynomial H = (Gamma / lc_y G) G with G = gcd(A, B) has the image
//     H(x_t, y) mod p = Gamma(x_t) * monic gcd(A(x_t, y), B(x_t, y)) mod p
// at every (p, x_t) where neither leading coefficient vanishes and the image
// degree is minimal.  This kernel produces those images: evaluate every
// y-coefficient at x_t (Horner, lanes across the coefficients), run the
// division-free Euclid of _zp_gcd (modpoly.py:115-122; every remainder a
// nonzero multiple of the reference's) on the two univariate images in shared
// memory, make the gcd monic with one inverse and scale it by Gamma(x_t).
// The host (bivpoly.gcd_biv) keeps the images of minimal degree, interpolates
// them in x (k_interp_points), lifts them by CRT (tensor-core CRT) and
// verifies by exact trial division like the reference's int_gcd_uni.
#include "ckb_kernels.cuh"

namespace ckb {

constexpr int BG_WARPS = 4;

// res: [K][C] residues (A's grid (m+1)(dax+1), B's (n+1)(dbx+1), Gamma's dgam+1);
// degs: [m+n+2] x-degrees of the y-coefficients (-1 = zero)
__global__ void __launch_bounds__(32 * BG_WARPS) k_biv_gcd_images(const uint32_t* __restrict__ res, int C,
                                                                  const int16_t* __restrict__ degs, int m, int n,
                                                                  int dax, int dbx, int dgam,
                                                                  const Prime* __restrict__ primes, int K, int NP,
                                                                  uint32_t* __restrict__ out, int Wo,
                                                                  int32_t* __restrict__ odeg) {
  extern __shared__ uint32_t sm[];
  CKB_SMEM_POISON(sm);
  const int W = (m > n ? m : n) + 1;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int img = blockIdx.x * BG_WARPS + warp;
  if (img >= K * NP) return;  // warp-uniform
  const int pi = img / NP, t = img - pi * NP;
  const Prime P = primes[pi];
  const uint32_t p = P.p;
  uint32_t* X = sm + warp * 2 * W;
  uint32_t* Y = X + W;
  const uint32_t* r = res + (size_t)pi * C;
  const uint32_t x = (uint32_t)(t + 1) % p;  // points x_t = t + 1 (x_t < p for every table prime)
  const uint32_t xc = shoup_comp(x, P);
  // y-coefficients of A(x_t, y) and B(x_t, y)
  const int offB = (m + 1) * (dax + 1);
  for (int j = lane; j <= m + n + 1; j += 32) {
    const bool isa = j <= m;
    const int jj = isa ? j : j - m - 1;
    const uint32_t* c = r + (isa ? jj * (dax + 1) : offB + jj * (dbx + 1));
    uint32_t acc = 0u;
    for (int i = degs[j]; i >= 0; --i) acc = add_mod(shoup(acc, x, xc, p), c[i], p);
    (isa ? X : Y)[jj] = acc;
  }
  __syncwarp();
  uint32_t* o = out + (size_t)img * Wo;
  if (X[m] == 0u || Y[n] == 0u) {  // a leading coefficient vanishes at x_t: skip the point
    for (int i = lane; i < Wo; i += 32) o[i] = 0u;
    if (lane == 0) odeg[img] = -2;
    return;
  }
  // Euclid, division-free: A <- lc(B) A - lc(A) y^s B while deg A >= deg B
  uint32_t* A = X;
  uint32_t* B = Y;
  int da = m, db = n;
  while (db >= 0) {
    while (da >= db) {
      const uint32_t la = A[da], lb = B[db];
      const int s = da - db;
      const uint32_t lbc = shoup_comp(lb, P);
      const uint32_t nla = neg_mod(la, p), nlac = shoup_comp(nla, P);
      for (int j = lane; j < da; j += 32) {
        uint32_t v = shoup(A[j], lb, lbc, p);
        if (j >= s) v = add_mod(v, shoup(B[j - s], nla, nlac, p), p);
        A[j] = v;
      }
      __syncwarp();
      // new degree: highest nonzero entry below da (ballot over 32-entry windows)
      int d = da - 1;
      while (d >= 0) {
        const int i = d - lane;
        const unsigned nz = __ballot_sync(0xffffffffu, i >= 0 && A[i] != 0u);
        if (nz) {
          d -= __ffs(nz) - 1;
          break;
        }
        d -= 32;
      }
      da = d < 0 ? -1 : d;
      if (da < 0) break;
    }
    uint32_t* tp = A;
    A = B;
    B = tp;
    const int td = da;
    da = db;
    db = td;
  }
  // A: the gcd (deg da >= 0, A nonzero since B(x_t) has a nonzero lc)
  // Gamma(x_t) / lc(A): Gamma by Horner (lane 0), one inverse
  uint32_t scale = 0u;
  if (lane == 0) {
    const uint32_t* gm = r + offB + (n + 1) * (dbx + 1);
    uint32_t gv = 0u;
    for (int i = dgam; i >= 0; --i) gv = add_mod(shoup(gv, x, xc, p), gm[i], p);
    scale = mul_mod(gv, inv_mod(A[da], P), P);
  }
  scale = __shfl_sync(0xffffffffu, scale, 0);
  const uint32_t sc = shoup_comp(scale, P);
  for (int i = lane; i < Wo; i += 32) o[i] = (i <= da) ? shoup(A[i], scale, sc, p) : 0u;
  if (lane == 0) odeg[img] = da;
}

void launch_biv_gcd_images(const uint32_t* res, int C, const int16_t* degs, int m, int n, int dax, int dbx, int dgam,
                           const Prime* primes, int K, int NP, uint32_t* out, int Wo, int32_t* odeg, cudaStream_t st) {
  const int W = (m > n ? m : n) + 1;
  const size_t smem = (size_t)BG_WARPS * 2 * W * 4;
  const unsigned blocks = (unsigned)(((size_t)K * NP + BG_WARPS - 1) / BG_WARPS);
  k_biv_gcd_images<<<blocks, 32 * BG_WARPS, smem, st>>>(res, C, degs, m, n, dax, dbx, dgam, primes, K, NP, out, Wo,
                                                         odeg);
}

}  // namespace ckb

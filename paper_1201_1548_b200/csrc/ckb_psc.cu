// The modular subresultant degree profile (GeoTop's N^- test)
// on the device: curvekit.modpoly.modular_subres_profile
// (pkg/src/curvekit/modpoly.py:428-474) with its psc values (_psc_det, :477-501)
// taken from ONE remainder sequence per point instead of one dense determinant
// per (point, i):
//
//   k_psc_points  one CTA: the reference's points t = 0, 1, 2, ... that do not
//                 annihilate a leading coefficient (modpoly.py:446-453), the
//                 first `need` of them compacted by a block scan;
//   k_psc_prs     one warp per point: evaluate the y-coefficients at t (:459-460),
//                 run the Euclidean remainder sequence mod p (the reference's own
//                 _zp_rem, :102-112) and read every psc_i off its degrees
//                 n_0 = m > n_1 = n > ... and leading coefficients c_l by the
//                 fundamental theorem of subresultants:
//                   psc_{n_i} = (-1)^tau_i c_i^(n_{i-1} - n_i) prod_{l<i} c_l^(n_{l-1} - n_{l+1}),
//                   tau_i = sum_{l<i} (n_{l-1} - n_i)(n_l - n_i),
//                 and psc_j = 0 for every other j (checked against _psc_det on
//                 random, sparse and common-factor inputs: tests/test_subres.py);
//   interpolation of every psc_i from its first cnt_i points (k_interp_points,
//                 all i in one launch, the shared point list);
//   k_gcd_chain   one CTA: S_0 = rstar mod p, S_i = gcd(S_{i-1}, psc_i) (:464-473)
//                 -- only the degrees are needed, so the gcds run division-free.
#include "ckb_kernels.cuh"

namespace ckb {

constexpr int PSC_WARPS = 4;
constexpr int SEL_THREADS = 1024;

// candidates t = 0 .. ncand-1: t is a point when lc_f(t) lc_g(t) != 0 mod p;
// sel[0..need) = the first `need` points in increasing t, *count = how many exist
__global__ void __launch_bounds__(SEL_THREADS) k_psc_points(const uint32_t* __restrict__ lcf, int dlf,
                                                           const uint32_t* __restrict__ lcg, int dlg, Prime P,
                                                           int ncand, int need, uint32_t* __restrict__ sel,
                                                           int* __restrict__ count) {
  __shared__ int warp_tot[SEL_THREADS / 32];
  __shared__ int base;
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t p = P.p;
  if (tid == 0) base = 0;
  __syncthreads();
  for (int c0 = 0; c0 < ncand; c0 += SEL_THREADS) {
    const int t = c0 + tid;
    bool ok = false;
    if (t < ncand) {
      const uint32_t x = (uint32_t)t % p, xc = shoup_comp(x, P);
      uint32_t a = 0, b = 0;
      for (int e = dlf; e >= 0; --e) a = add_mod(shoup(a, x, xc, p), lcf[e], p);
      for (int e = dlg; e >= 0; --e) b = add_mod(shoup(b, x, xc, p), lcg[e], p);
      ok = a != 0u && b != 0u;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, ok);
    const int before = __popc(bal & ((1u << lane) - 1u));
    if (lane == 0) warp_tot[w] = __popc(bal);
    __syncthreads();
    int off = 0;
    for (int k = 0; k < w; ++k) off += warp_tot[k];
    const int pos = base + off + before;
    if (ok && pos < need) sel[pos] = (uint32_t)t;
    __syncthreads();
    if (tid == 0) {
      int s = 0;
      for (int k = 0; k < SEL_THREADS / 32; ++k) s += warp_tot[k];
      base += s;
    }
    __syncthreads();
  }
  if (tid == 0) *count = base;
}

// remainder of a (len la) by b (len lb, lc nonzero) into r (len la), the
// reference's _zp_rem; returns the trimmed length of r
__device__ int warp_rem(const uint32_t* a, int la, const uint32_t* b, int lb, uint32_t* r, const Prime& P) {
  const int lane = threadIdx.x & 31;
  const uint32_t p = P.p;
  for (int i = lane; i < la; i += 32) r[i] = a[i];
  __syncwarp();
  const uint32_t inv = inv_mod(b[lb - 1], P);
  int lr = la;
  while (lr >= lb) {
    const uint32_t c = mul_mod(r[lr - 1], inv, P);
    __syncwarp();  // every lane has read r[lr - 1] before its owner updates it
    if (c) {
      const int k = lr - lb;
      const uint32_t nc = p - c, ncc = shoup_comp(nc, P);
      for (int j = lane; j < lb; j += 32) r[k + j] = add_mod(r[k + j], shoup(b[j], nc, ncc, p), p);
    }
    __syncwarp();
    --lr;
  }
  while (lr > 0 && r[lr - 1] == 0u) --lr;
  return lr;
}

// psc_1..psc_n at the points (pts, or t = index when pts is null) -> out [n][npts];
// valid (optional) [npts]: 1 where neither leading coefficient vanishes (elsewhere
// the values are 0: the reference never uses such a point)
__global__ void __launch_bounds__(32 * PSC_WARPS) k_psc_prs(const uint32_t* __restrict__ fres,
                                                           const int16_t* __restrict__ fdeg, int m, int dfx,
                                                           const uint32_t* __restrict__ gres,
                                                           const int16_t* __restrict__ gdeg, int n, int dgx, Prime P,
                                                           const uint32_t* __restrict__ pts, int npts,
                                                           uint32_t* __restrict__ out, uint8_t* __restrict__ valid) {
  extern __shared__ uint32_t sm[];
  CKB_SMEM_POISON(sm);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int j = blockIdx.x * PSC_WARPS + w;
  const int stride = 3 * (m + 1) + 2 * (n + 3);
  uint32_t* X = sm + (size_t)w * stride;  // three remainder buffers of m + 1 words
  uint32_t* Y = X + (m + 1);
  uint32_t* Z = Y + (m + 1);
  int* degs = reinterpret_cast<int*>(Z + (m + 1));  // n_0 .. (<= n + 2 entries)
  uint32_t* psc = Z + (m + 1) + (n + 3);            // psc_1 .. psc_n at [1 .. n]
  if (j >= npts) return;
  const uint32_t p = P.p;
  const uint32_t t = (pts ? pts[j] : (uint32_t)j) % p;
  const uint32_t tc = shoup_comp(t, P);
  for (int q = lane; q <= m + n + 1; q += 32) {
    const bool isf = q <= m;
    const int qq = isf ? q : q - m - 1;
    const uint32_t* c = isf ? fres + q * (dfx + 1) : gres + qq * (dgx + 1);
    const int deg = isf ? fdeg[q] : gdeg[qq];
    uint32_t acc = 0;
    for (int e = deg; e >= 0; --e) acc = add_mod(shoup(acc, t, tc, p), c[e], p);
    (isf ? X : Y)[qq] = acc;
  }
  for (int i = lane; i <= n; i += 32) psc[i] = 0u;
  __syncwarp();
  const bool ok = X[m] != 0u && Y[n] != 0u;
  if (valid && lane == 0) valid[j] = ok ? 1 : 0;
  if (ok) {
    // R_0 = X (deg m), R_1 = Y (deg n); acc = prod_{l<i} c_l^(n_{l-1} - n_{l+1})
    uint32_t* Rp = X;
    uint32_t* Rc = Y;
    uint32_t* Rn = Z;
    int lp = m + 1, lc = n + 1;
    if (lane == 0) {
      degs[0] = m;
      degs[1] = n;
    }
    __syncwarp();
    uint32_t acc = 1u % p;
    for (int i = 1;; ++i) {
      const int ni = lc - 1;
      const uint32_t ci = Rc[lc - 1];
      int tau = 0;
      for (int l = 1; l < i; ++l) tau ^= ((degs[l - 1] - ni) * (degs[l] - ni)) & 1;
      uint32_t v = mul_mod(pow_mod(ci, (uint64_t)(degs[i - 1] - ni), P), acc, P);
      if (tau) v = neg_mod(v, p);
      if (ni >= 1 && lane == 0) psc[ni] = v;
      if (ni == 0) break;
      const int lr = warp_rem(Rp, lp, Rc, lc, Rn, P);
      if (lr == 0) break;  // a common factor: every lower psc is 0
      if (lane == 0) degs[i + 1] = lr - 1;
      acc = mul_mod(acc, pow_mod(ci, (uint64_t)(degs[i - 1] - (lr - 1)), P), P);
      uint32_t* tmp = Rp;
      Rp = Rc;
      Rc = Rn;
      Rn = tmp;
      lp = lc;
      lc = lr;
      __syncwarp();
    }
  }
  __syncwarp();
  for (int i = 1 + lane; i <= n; i += 32) out[(size_t)(i - 1) * npts + j] = psc[i];
}

// one CTA: S_0 = rstar mod p (trimmed length must be rlen_int), S_i = gcd(S_{i-1}, sr_i)
// for the interpolated sr_i (rows of `sr`, row i-1 has cnt[i-1] coefficients, stride W);
// chain[0..n] = deg S_i; *status = 2 when S_0 loses degree mod p (UnluckyPrime)
__global__ void __launch_bounds__(1024) k_gcd_chain(const uint32_t* __restrict__ rmod, int rlen, int rlen_int,
                                                   const uint32_t* __restrict__ sr, const int* __restrict__ cnt,
                                                   int W, int n, Prime P, int* __restrict__ chain,
                                                   uint32_t* __restrict__ status) {
  extern __shared__ uint32_t sm[];
  CKB_SMEM_POISON(sm);
  __shared__ int s_len;
  const int tid = threadIdx.x, T = blockDim.x;
  const uint32_t p = P.p;
  const int cap = max(rlen, W);
  uint32_t* A = sm;
  uint32_t* B = sm + cap;
  for (int i = tid; i < rlen; i += T) A[i] = rmod[i];
  __syncthreads();
  if (tid == 0) {
    int l = rlen;
    while (l > 0 && A[l - 1] == 0u) --l;
    s_len = l;
  }
  __syncthreads();
  int la = s_len;
  if (la != rlen_int) {
    if (tid == 0) *status = 2u;
    return;
  }
  if (tid == 0) chain[0] = la - 1;
  for (int i = 1; i <= n; ++i) {
    const int c = cnt[i - 1];
    const uint32_t* row = sr + (size_t)(i - 1) * W;
    for (int k = tid; k < c; k += T) B[k] = row[k];
    __syncthreads();
    if (tid == 0) {
      int l = c;
      while (l > 0 && B[l - 1] == 0u) --l;
      s_len = l;
    }
    __syncthreads();
    int lb = s_len;
    if (lb > 0 && la > 1) {
      // Euclid, division-free: X <- lc(Y) X - lc(X) x^s Y keeps every remainder a
      // nonzero multiple of the reference's, so the gcd's degree is unchanged
      uint32_t* X = A;
      uint32_t* Y = B;
      int lx = la, ly = lb;
      if (lx < ly) {
        uint32_t* tp = X; X = Y; Y = tp;
        const int tl = lx; lx = ly; ly = tl;
      }
      while (ly > 0) {
        // one barrier per step: the update writes X[0 .. lx-2] only, the new
        // leading coefficient and the trim read X[lx'-1 ..] (lx' the new length),
        // so a thread still trimming never reads what the next step writes
        while (lx >= ly) {
          // Montgomery products with the RAW coefficients as multipliers: every
          // term of a step carries the same factor 2^-32 (and so does the next
          // step's), which leaves gcd(X, Y) unchanged -- no conversion or Shoup
          // companion on the per-step critical path
          const uint32_t ca = X[lx - 1], cb = Y[ly - 1];
          const uint32_t nca = neg_mod(ca, p);
          const int s = lx - ly;
          int l;
          if (s >= 1 && ly >= 2) {
            // two elimination steps per barrier: X <- cb^2 X - (cb ca x^s + l1 x^(s-1)) Y,
            // l1 = cb X[lx-2] - ca Y[ly-2] the lc after the first (both leading terms cancel)
            const uint32_t l1 = redc((uint64_t)cb * X[lx - 2] + (uint64_t)nca * Y[ly - 2], P);
            const uint32_t w1 = redc((uint64_t)cb * cb, P), w2 = redc((uint64_t)cb * nca, P);
            const uint32_t w3 = neg_mod(l1, p);
            for (int k = tid; k < lx - 2; k += T) {
              uint64_t t = (uint64_t)X[k] * w1;
              if (k >= s) t += (uint64_t)Y[k - s] * w2;
              if (k >= s - 1) t += (uint64_t)Y[k - s + 1] * w3;
              X[k] = redc(t, P);  // t < 3 p^2 < p 2^32
            }
            l = lx - 2;
          } else {
            for (int k = tid; k < lx - 1; k += T) {
              uint64_t t = (uint64_t)X[k] * cb;
              if (k >= s) t += (uint64_t)Y[k - s] * nca;
              X[k] = redc(t, P);
            }
            l = lx - 1;
          }
          __syncthreads();
          while (l > 0 && X[l - 1] == 0u) --l;  // every thread, the same length
          lx = l;
          if (lx == 0) break;
        }
        uint32_t* tp = X; X = Y; Y = tp;
        const int tl = lx; lx = ly; ly = tl;
      }
      // the gcd is X (length lx); keep it in A
      if (X != A) {
        for (int k = tid; k < lx; k += T) A[k] = X[k];
      }
      la = lx;
      __syncthreads();
    }
    if (tid == 0) chain[i] = la - 1;
    __syncthreads();
  }
}

void launch_psc_points(const uint32_t* lcf, int dlf, const uint32_t* lcg, int dlg, const Prime& P, int ncand,
                       int need, uint32_t* sel, int* count, cudaStream_t st) {
  k_psc_points<<<1, SEL_THREADS, 0, st>>>(lcf, dlf, lcg, dlg, P, ncand, need, sel, count);
}

static size_t psc_smem(int m, int n) { return (size_t)PSC_WARPS * (3 * (m + 1) + 2 * (n + 3)) * 4; }
bool psc_fits(int m, int n) { return psc_smem(m, n) <= 200 * 1024; }

void launch_psc(const uint32_t* fres, const int16_t* fdeg, int m, int dfx, const uint32_t* gres,
                const int16_t* gdeg, int n, int dgx, const Prime& P, const uint32_t* pts, int npts, uint32_t* out,
                uint8_t* valid, cudaStream_t st) {
  const size_t smem = psc_smem(m, n);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_psc_prs, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_psc_prs<<<(npts + PSC_WARPS - 1) / PSC_WARPS, 32 * PSC_WARPS, smem, st>>>(fres, fdeg, m, dfx, gres, gdeg, n, dgx,
                                                                              P, pts, npts, out, valid);
}

bool gcd_chain_fits(int rlen, int W) { return (size_t)2 * (rlen > W ? rlen : W) * 4 <= 200 * 1024; }

void launch_gcd_chain(const uint32_t* rmod, int rlen, int rlen_int, const uint32_t* sr, const int* cnt, int W, int n,
                      const Prime& P, int* chain, uint32_t* status, cudaStream_t st) {
  const size_t smem = (size_t)2 * (rlen > W ? rlen : W) * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_gcd_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_gcd_chain<<<1, 1024, smem, st>>>(rmod, rlen, rlen_int, sr, cnt, W, n, P, chain, status);
}

}  // namespace ckb

// The per-prime point scale c (modpoly.py:380-390 skips the points where a
// leading coefficient vanishes; here the whole progression x = w^j c y_u is
// shifted by c = 1, 2, ... instead, keeping the cached plan valid).  One CTA
// per prime (any blockDim); lcf / lcg are the residues of the two leading
// coefficients (x-polynomials of degree lcf_deg / lcg_deg).  Shared by
// k_choose_c (ckb_plan.cu) and the merged K1 kernel (ckb_images.cu).
#pragma once
#include "ckb_kernels.cuh"

namespace ckb {

__device__ __forceinline__ void choose_c_prime(const Prime& P, int pi, const InterpPlan& plan,
                                               const uint32_t* lcf, int lcf_deg, const uint32_t* lcg, int lcg_deg,
                                               uint32_t* __restrict__ cval, uint32_t* status) {
  const int tid = threadIdx.x, T = blockDim.x, N = plan.N;
  const uint32_t p = P.p;
  if (lcf_deg <= 0 && lcg_deg <= 0) {  // constant leading coefficients
    if (tid == 0) {
      cval[pi] = 1u;
      if (lcf[0] == 0u || lcg[0] == 0u) atomicOr(status, 1u);
    }
    return;
  }
  // image points x = w^j c y_u, j < S, u < N (polyphase cosets)
  const int S = plan.S;
  const uint32_t* yq = plan.yq + (size_t)pi * N;
  const uint32_t* om = plan.om + (size_t)pi * 4 * S;
  for (int attempt = 0; attempt < 64; ++attempt) {
    const uint32_t c = (uint32_t)(attempt + 1) % p;
    const uint32_t cc = shoup_comp(c, P);
    int bad = 0;
    if (S == 8) {
      // one thread per coset: with x = c y_u every point is w^j x and (w^j x)^8 = x^8, so
      // lc(w^j x) = sum_r w^(jr) x^r A_r(x^8), A_r(z) = sum_q a_(8q+r) z^q: eight short
      // Horner chains in z, then an 8-point transform (~120 products for 8 points, not 8 deg)
      for (int u = tid; u < N; u += T) {
        const uint32_t x = shoup(yq[u], c, cc, p);
        const uint32_t x2 = mul_mod(x, x, P), x4 = mul_mod(x2, x2, P), z = mul_mod(x4, x4, P);
        const uint32_t zc = shoup_comp(z, P);
        for (int side = 0; side < 2; ++side) {
          const uint32_t* lc = side ? lcg : lcf;
          const int dl = side ? lcg_deg : lcf_deg;
          uint32_t B[8];
          uint32_t xr = 1u % p;
#pragma unroll
          for (int r = 0; r < 8; ++r) {
            uint32_t a = 0u;
            for (int e = r + 8 * ((dl - r) >= 0 ? (dl - r) / 8 : -1); e >= r; e -= 8)
              a = add_mod(shoup(a, z, zc, p), lc[e], p);
            B[r] = mul_mod(a, xr, P);  // x^r A_r(x^8)
            xr = mul_mod(xr, x, P);
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            uint32_t v = 0u;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
              const int k = (j * r) & 7;
              v = add_mod(v, k ? shoup(B[r], om[k], om[S + k], p) : B[r], p);
            }
            if (v == 0u) bad = 1;
          }
        }
      }
    } else {
      for (int t = tid; t < N * S; t += T) {
        const int u = t / S, j = t % S;
        const uint32_t x = shoup(shoup(yq[u], om[j], om[S + j], p), c, cc, p);
        const uint32_t xc = shoup_comp(x, P);
        uint32_t vf = 0, vg = 0;
        for (int i = lcf_deg; i >= 0; --i) vf = add_mod(shoup(vf, x, xc, p), lcf[i], p);
        for (int i = lcg_deg; i >= 0; --i) vg = add_mod(shoup(vg, x, xc, p), lcg[i], p);
        if (vf == 0u || vg == 0u) bad = 1;
      }
    }
    bad = __syncthreads_or(bad);
    if (!bad) {
      if (tid == 0) cval[pi] = c;
      return;
    }
  }
  if (tid == 0) {
    cval[pi] = 1u;
    atomicOr(status, 1u);
  }
}

}  // namespace ckb

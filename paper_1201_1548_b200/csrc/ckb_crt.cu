// K5: Chinese remaindering of every coefficient and the symmetric lift to
// two's-complement 32-bit limbs.
//
// Reference: curvekit.modpoly._CrtAccumulator.add / symmetric
// (pkg/src/curvekit/modpoly.py:278-300) and crt_reconstruct (:264-275):
// incremental Garner, then x - M if 2x > M.  The result is the unique
// representative of the residues in (-M/2, M/2]; this kernel computes the
// same integer by the *explicit* CRT, which has no sequential recurrence:
//     y_i = r_i * (M/p_i)^-1 mod p_i                     (one Shoup product)
//     X   = sum_i y_i * (M/p_i)                           (an N x K x LW integer
//                                                          product: K2 below)
//     q   = round(sum_i y_i / p_i)                       (FP64)
//     x   = X - q M
// X/M = q + x/M exactly; the planner guarantees M > 4 * bound, so |x/M| < 1/4
// and the FP64 sum (error < K^2 2^-52) always rounds to the right q.
#include "ckb_kernels.cuh"

namespace ckb {

constexpr int TN = 64;   // coefficients per CTA tile
constexpr int TL = 32;   // limbs per CTA tile
constexpr int TI = 32;   // primes per k-step
constexpr int CRT_THREADS = 256;

// K2: S[k][l] = sum_i y_i(k) * (M/p_i)[l] as 96-bit (lo64, hi32) column sums.
// Thread micro-tile: 2 coefficients x 4 limbs.
__global__ void __launch_bounds__(CRT_THREADS) k_crt_gemm(CrtTables T, const uint32_t* __restrict__ r, int N,
                                                          uint32_t* __restrict__ S) {
  __shared__ uint32_t sy[TI][TN];
  __shared__ uint32_t sm[TI][TL];
  const int K = T.K, LW = T.LW;
  const int k0 = blockIdx.x * TN, l0 = blockIdx.y * TL;
  const int tid = threadIdx.x;
  const int tk = (tid % 32) * 2;        // coefficient offset (0..62)
  const int tl = (tid / 32) * 4;        // limb offset (0..28)
  uint64_t lo[2][4] = {};
  uint32_t hi[2][4] = {};
  for (int i0 = 0; i0 < K; i0 += TI) {
    // stage y (computed on the fly from the residues) and the M/p_i limbs
    for (int e = tid; e < TI * TN; e += CRT_THREADS) {
      const int ii = e / TN, kk = e % TN;
      const int i = i0 + ii, k = k0 + kk;
      uint32_t y = 0;
      if (i < K && k < N) {
        const uint32_t p = T.p[i];
        y = red1(shoup_lazy(r[(size_t)i * N + k], T.c[i], T.cc[i], p), p);
      }
      sy[ii][kk] = y;
    }
    for (int e = tid; e < TI * TL; e += CRT_THREADS) {
      const int ii = e / TL, ll = e % TL;
      const int i = i0 + ii, l = l0 + ll;
      sm[ii][ll] = (i < K && l < LW) ? T.Mi[(size_t)i * LW + l] : 0u;
    }
    __syncthreads();
#pragma unroll 4
    for (int ii = 0; ii < TI; ++ii) {
      const uint2 yv = *reinterpret_cast<const uint2*>(&sy[ii][tk]);
      const uint4 mv = *reinterpret_cast<const uint4*>(&sm[ii][tl]);
      const uint32_t ys[2] = {yv.x, yv.y};
      const uint32_t ms[4] = {mv.x, mv.y, mv.z, mv.w};
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint64_t pr = (uint64_t)ys[a] * ms[b];
          const uint64_t s = lo[a][b] + pr;
          hi[a][b] += (s < pr);
          lo[a][b] = s;
        }
    }
    __syncthreads();
  }
  // limb-major layout S[l][0..2][k]: the carry pass reads it coalesced
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int k = k0 + tk + a, l = l0 + tl + b;
      if (k < N && l < LW) {
        uint32_t* o = S + (size_t)l * 3 * N + k;
        o[0] = (uint32_t)lo[a][b];
        o[N] = (uint32_t)(lo[a][b] >> 32);
        o[2 * N] = hi[a][b];
      }
    }
}

// K3: per coefficient, q = round(sum y_i / p_i), then x = S - q M with a
// signed carry chain over the limbs -> two's complement out[k][0..LW).
__global__ void __launch_bounds__(128) k_crt_carry(CrtTables T, const uint32_t* __restrict__ r, int N,
                                                   const uint32_t* __restrict__ S, uint32_t* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  __shared__ uint32_t stage[128][33];
  const int tid = threadIdx.x, k0 = blockIdx.x * blockDim.x;
  const bool act = k < N;
  const int K = T.K, LW = T.LW;
  double s = 0.0;
  if (act) {
#pragma unroll 8
    for (int i = 0; i < K; ++i) {
      const uint32_t p = T.p[i];
      const uint32_t y = red1(shoup_lazy(r[(size_t)i * N + k], T.c[i], T.cc[i], p), p);
      s = fma((double)y, T.pinvd[i], s);
    }
  }
  const uint64_t q = (uint64_t)llrint(s);
  // carry = (c_hi:c_lo) signed 128-bit; value at limb l = S_l - q M_l + carry
  long long c_hi = 0;
  unsigned long long c_lo = 0;
  for (int l0 = 0; l0 < LW; l0 += 32) {
    if (act) {
      // issue every load of the chunk before the (sequential) carry chain
      uint32_t v0[32], v1[32], v2[32], ml[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int l = l0 + j;
        const bool in = l < LW;
        const uint32_t* Sl = S + (size_t)(in ? l : 0) * 3 * N + k;
        v0[j] = in ? Sl[0] : 0u;
        v1[j] = in ? Sl[N] : 0u;
        v2[j] = in ? Sl[2 * N] : 0u;
        ml[j] = in ? T.Ml[l] : 0u;
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const unsigned long long s_lo = (unsigned long long)v0[j] | ((unsigned long long)v1[j] << 32);
        const long long s_hi = v2[j];
        const unsigned long long qm = q * (unsigned long long)ml[j];  // < 2^44
        unsigned long long t_lo = s_lo - qm;  // t = s - qm + carry
        long long t_hi = s_hi - (long long)(s_lo < qm);
        const unsigned long long u = t_lo + c_lo;
        t_hi += c_hi + (long long)(u < t_lo);
        t_lo = u;
        stage[tid][j] = (uint32_t)t_lo;
        c_lo = (t_lo >> 32) | ((unsigned long long)t_hi << 32);  // carry = t >> 32
        c_hi = t_hi >> 32;
      }
    }
    __syncthreads();
    for (int e = tid; e < 128 * 32; e += blockDim.x) {  // coalesced rows
      const int rr = e >> 5, j = e & 31;
      if (k0 + rr < N && l0 + j < LW) out[(size_t)(k0 + rr) * LW + l0 + j] = stage[rr][j];
    }
    __syncthreads();
  }
  if (!act) return;
  uint32_t* ok = out + (size_t)k * LW;
  // Exactness guard for callers without the 4x margin (crt_reconstruct on
  // arbitrary residues): if s was near a half-integer, q may be off by one;
  // fold x into [-floor(M/2), floor(M/2)] exactly.  Never taken when M > 4 bound.
  const double fr = s - floor(s);
  if (fabs(fr - 0.5) < 1e-3) {
    // d = x - H - 1 ; if d >= 0 then x -= M
    long long br = 0;
    for (int l = 0; l < LW; ++l) {
      const long long v = (long long)ok[l] - (long long)T.Mh[l] - (l == 0 ? 1 : 0) + br;
      br = v >> 32;
    }
    const bool x_top_neg = (int32_t)ok[LW - 1] < 0;
    // the sign of d is the sign of the full-width result: x (signed) - H - 1
    const bool gt = !x_top_neg && br >= 0;
    // e = x + H ; if e < 0 then x += M
    long long cr = 0;
    for (int l = 0; l < LW; ++l) {
      const long long v = (long long)ok[l] + (long long)T.Mh[l] + cr;
      cr = v >> 32;
    }
    const bool lt = x_top_neg && cr == 0;  // x + H did not carry out of a negative x: still negative
    if (gt || lt) {
      long long c = 0;
      for (int l = 0; l < LW; ++l) {
        const long long v = (long long)ok[l] + (gt ? -(long long)T.Ml[l] : (long long)T.Ml[l]) + c;
        ok[l] = (uint32_t)v;
        c = v >> 32;
      }
    }
  }
}

void launch_crt(const CrtTables& t, const uint32_t* coeffs, int N, uint32_t* out, uint32_t* scratch,
                cudaStream_t st) {
  dim3 g1((N + TN - 1) / TN, (t.LW + TL - 1) / TL);
  k_crt_gemm<<<g1, CRT_THREADS, 0, st>>>(t, coeffs, N, scratch);
  k_crt_carry<<<(N + 127) / 128, 128, 0, st>>>(t, coeffs, N, scratch, out);
}

}  // namespace ckb

// K5: mixed-radix (Garner) CRT of every coefficient and the symmetric lift to
// two's-complement 32-bit limbs, one warp per coefficient.
//
// Reference: curvekit.modpoly._CrtAccumulator.add / symmetric
// (pkg/src/curvekit/modpoly.py:278-300) and crt_reconstruct (:264-275):
//   x_{i+1} = x_i + M_i * ((r_i - x_i) * M_i^-1 mod p_i),  M_i = prod_{l<i} p_l
//   result  = x - M if 2x > M else x.
// Here the digits a_i = ((r_i - x_i) M_i^-1 mod p_i) are computed for all i
// at once (column-updated residues, Montgomery table of M_j mod p_i), the sign
// is decided on the digits (2x > M  <=>  digits > ((p_i - 1)/2)_i lexicographic
// from the top, M being odd), and the magnitude sum_i b_i M_i is formed as
// 32-bit column sums with a ballot carry-lookahead, so only bytes leave the GPU.
#include "ckb_kernels.cuh"

namespace ckb {

constexpr int CRT_WARPS = 4;

__global__ void __launch_bounds__(CRT_WARPS * 32) k_crt(CrtTables T, const uint32_t* __restrict__ coeffs, int N,
                                                       uint32_t* __restrict__ out) {
  extern __shared__ uint32_t sm[];
  const int K = T.K, LW = T.LW;
  uint32_t* sp = sm;            // [K] primes
  uint32_t* spinv = sm + K;     // [K] p^-1 mod 2^32
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* dig = sm + 2 * K + warp * K;
  for (int i = threadIdx.x; i < K; i += blockDim.x) {
    sp[i] = T.primes[i].p;
    spinv[i] = T.primes[i].pinv;
  }
  __syncthreads();
  const int k = blockIdx.x * CRT_WARPS + warp;
  if (k >= N) return;
  const unsigned FULL = 0xffffffffu;

  for (int i = lane; i < K; i += 32) dig[i] = coeffs[(size_t)i * N + k];
  __syncwarp();
  // Garner digits
  for (int j = 0; j < K; ++j) {
    uint32_t aj = 0;
    if (lane == (j & 31)) {
      Prime Pj;
      Pj.p = sp[j];
      Pj.pinv = spinv[j];
      aj = redc((uint64_t)dig[j] * T.invm[j], Pj);
      dig[j] = aj;
    }
    aj = __shfl_sync(FULL, aj, j & 31);
    const uint32_t* Wrow = T.Wm + (size_t)j * K;
    for (int i = j + 1 + lane; i < K; i += 32) {
      Prime Pi;
      Pi.p = sp[i];
      Pi.pinv = spinv[i];
      const uint32_t tt = redc((uint64_t)aj * Wrow[i], Pi);
      dig[i] = sub_mod(dig[i], tt, Pi.p);
    }
    __syncwarp();
  }
  // sign: x > (M-1)/2 ?
  bool neg = false;
  for (int s = (K - 1) >> 5; s >= 0; --s) {
    const int i = (s << 5) + lane;
    const bool d = (i < K) && (dig[i] != ((sp[i] - 1) >> 1));
    const unsigned b = __ballot_sync(FULL, d);
    if (b) {
      const int il = (s << 5) + (31 - __clz(b));
      neg = dig[il] > ((sp[il] - 1) >> 1);
      break;
    }
  }
  if (neg) {  // |x - M| = (M - 1 - x) + 1, digits p_i - 1 - a_i
    for (int i = lane; i < K; i += 32) dig[i] = sp[i] - 1 - dig[i];
  }
  __syncwarp();

  // column sums S_l = sum_j b_j * M_j[l] (+1 at l = 0 if neg), carry-resolved
  uint32_t prev_a1 = 0, prev_a2_30 = 0, prev_a2_31 = 0, prev_t1 = 0, cin = 0, ncin = 1;
  uint32_t* orow = out + (size_t)k * LW;
  for (int l0 = 0; l0 < LW; l0 += 32) {
    const int l = l0 + lane;
    uint64_t lo = 0;
    uint32_t hi = 0;
    if (l < LW) {
      for (int j = l0; j < K; ++j) {  // M_j has no limb at index >= j (j >= 1)
        const uint64_t pr = (uint64_t)dig[j] * T.Pl[(size_t)j * LW + l];
        lo += pr;
        hi += (lo < pr);
      }
      if (l0 == 0 && lane == 0) {  // j = 0 term handled above only if l0 == 0; add the +1
        if (neg) {
          lo += 1;
          hi += (lo == 0);
        }
      }
    }
    const uint32_t a0 = (uint32_t)lo, a1 = (uint32_t)(lo >> 32), a2 = hi;
    uint32_t a1m = __shfl_up_sync(FULL, a1, 1);
    uint32_t a2m = __shfl_up_sync(FULL, a2, 2);
    if (lane == 0) a1m = prev_a1;
    if (lane == 0) a2m = prev_a2_30;
    if (lane == 1) a2m = prev_a2_31;
    const uint64_t Tsum = (uint64_t)a0 + a1m + a2m;
    const uint32_t t0 = (uint32_t)Tsum, t1 = (uint32_t)(Tsum >> 32);
    uint32_t t1m = __shfl_up_sync(FULL, t1, 1);
    if (lane == 0) t1m = prev_t1;
    const uint64_t y = (uint64_t)t0 + t1m;  // <= 2^32 + 1
    const bool G = y >= 0x100000000ull;
    const bool Pp = (uint32_t)y == 0xffffffffu && !G;
    const unsigned X = __ballot_sync(FULL, G || Pp), Y = __ballot_sync(FULL, G);
    const uint64_t sum = (uint64_t)X + Y + cin;
    const uint32_t carries = (uint32_t)(sum ^ X ^ Y);
    uint32_t mag = (uint32_t)y + ((carries >> lane) & 1u);
    // spill to the next chunk
    prev_a1 = __shfl_sync(FULL, a1, 31);
    prev_a2_30 = __shfl_sync(FULL, a2, 30);
    prev_a2_31 = __shfl_sync(FULL, a2, 31);
    prev_t1 = __shfl_sync(FULL, t1, 31);
    cin = (uint32_t)(sum >> 32);
    if (neg) {  // two's complement: ~mag + 1
      const uint32_t ym = ~mag;
      const unsigned Pn = __ballot_sync(FULL, ym == 0xffffffffu);
      const uint64_t sn = (uint64_t)Pn + ncin;
      const uint32_t cn = (uint32_t)(sn ^ Pn);
      mag = ym + ((cn >> lane) & 1u);
      ncin = (uint32_t)(sn >> 32);
    }
    if (l < LW) orow[l] = mag;
  }
}

void launch_crt(const CrtTables& t, const uint32_t* coeffs, int N, uint32_t* out, cudaStream_t st) {
  const size_t smem = (size_t)(2 + CRT_WARPS) * t.K * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_crt, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_crt<<<(N + CRT_WARPS - 1) / CRT_WARPS, CRT_WARPS * 32, smem, st>>>(t, coeffs, N, out);
}

}  // namespace ckb

// Number-theoretic transforms of length L = 2^logL <= 2^14 in shared memory,
// one CTA per transform (p = 1 mod 2^14, p < 2^30).
//
// Forward: decimation in frequency (natural order in, bit-reversed out);
// inverse: decimation in time (bit-reversed in, natural out, NO 1/L factor),
// so a cyclic convolution is DIF(a) .* DIF(b) -> DIT without any permutation.
// Values stay lazily in [0, 2p) (Harvey's butterflies): a sum is folded with
// one conditional subtraction of 2p, a difference is offset by 2p and fed to
// a Shoup product, which accepts any 32-bit input.
#pragma once
#include "ckb_modarith.cuh"

namespace ckb {

__device__ __forceinline__ uint32_t red2p(uint32_t x, uint32_t p2) { return min(x, x - p2); }

// W/Wc: twiddles w^j and Shoup companions, j < L/2 (w a primitive L-th root)
__device__ __forceinline__ void ntt_dif(uint32_t* buf, int logL, const uint32_t* __restrict__ W,
                                        const uint32_t* __restrict__ Wc, uint32_t p) {
  const int L = 1 << logL, half = L >> 1;
  const uint32_t p2 = 2u * p;
  for (int lh = logL - 1; lh >= 0; --lh) {  // h = 2^lh
    const int h = 1 << lh, sh = logL - 1 - lh;  // twiddle stride L/(2h) = 2^sh
    for (int idx = threadIdx.x; idx < half; idx += blockDim.x) {
      const int j = idx & (h - 1);
      const int i0 = ((idx >> lh) << (lh + 1)) + j, i1 = i0 + h;
      const uint32_t x = buf[i0], y = buf[i1];
      const int w = j << sh;
      buf[i0] = red2p(x + y, p2);
      buf[i1] = shoup_lazy(x - y + p2, W[w], Wc[w], p);
    }
    __syncthreads();
  }
}

// Wi/Wic: inverse twiddles w^-j
__device__ __forceinline__ void ntt_dit(uint32_t* buf, int logL, const uint32_t* __restrict__ Wi,
                                        const uint32_t* __restrict__ Wic, uint32_t p) {
  const int L = 1 << logL, half = L >> 1;
  const uint32_t p2 = 2u * p;
  for (int lh = 0; lh < logL; ++lh) {
    const int h = 1 << lh, sh = logL - 1 - lh;
    for (int idx = threadIdx.x; idx < half; idx += blockDim.x) {
      const int j = idx & (h - 1);
      const int i0 = ((idx >> lh) << (lh + 1)) + j, i1 = i0 + h;
      const int w = j << sh;
      const uint32_t x = buf[i0];
      const uint32_t y = shoup_lazy(buf[i1], Wi[w], Wic[w], p);
      buf[i0] = red2p(x + y, p2);
      buf[i1] = red2p(x - y + p2, p2);
    }
    __syncthreads();
  }
}

}  // namespace ckb

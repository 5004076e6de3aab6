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

// Shared-memory index with one pad word per 8 (PAD = true): the radix-8
// passes read 8 words at stride h/4 per lane; unpadded, the lanes of a warp
// collide 4-8 ways on the banks for h <= 32 (ncu: 60% of the shared wavefronts
// of k_interp_poly were conflicts).  i + i/8 makes stride-8 and the
// (8-group x 8-lane) patterns conflict-free.
template <bool PAD>
__device__ __forceinline__ int sidx(int i) { return PAD ? i + (i >> 3) : i; }
// words a padded buffer of n entries occupies
__host__ __device__ __forceinline__ int padded_words(int n) { return n + (n >> 3) + 1; }

// ---- register-blocked radix-8 passes (same transforms, 3 stages per pass) ----
// DIF stage with half-size h on the pair (a, b) at in-block position pos:
//   a <- a + b,  b <- (a - b) w^(pos L / 2h)
__device__ __forceinline__ void bf_dif(uint32_t& a, uint32_t& b, int widx, const uint32_t* W, const uint32_t* Wc,
                                       uint32_t p, uint32_t p2) {
  const uint32_t x = a, y = b;
  a = red2p(x + y, p2);
  b = shoup_lazy(x - y + p2, W[widx], Wc[widx], p);
}
// DIT stage: b <- b w^-(pos L / 2h);  a <- a + b,  b <- a - b
__device__ __forceinline__ void bf_dit(uint32_t& a, uint32_t& b, int widx, const uint32_t* Wi, const uint32_t* Wic,
                                       uint32_t p, uint32_t p2) {
  const uint32_t x = a, y = shoup_lazy(b, Wi[widx], Wic[widx], p);
  a = red2p(x + y, p2);
  b = red2p(x - y + p2, p2);
}

// forward DIF: passes of three stages (h, h/2, h/4) on 8 registers, then a
// radix-4 or radix-2 tail; T = blockDim.x (a power of two)
template <int T, bool PAD = false>
__device__ __forceinline__ void ntt_dif8(uint32_t* buf, int logL, const uint32_t* W, const uint32_t* Wc, uint32_t p) {
  const int L = 1 << logL;
  const uint32_t p2 = 2u * p;
  int lh = logL - 1;  // current stage: half = 2^lh
  for (; lh >= 2; lh -= 3) {
    const int h = 1 << lh, q4 = h >> 2;
    for (int g = threadIdx.x; g < (L >> 3); g += T) {
      const int j = g & (q4 - 1), base = (g >> (lh - 2)) << (lh + 1);
      uint32_t x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = buf[sidx<PAD>(base + j + k * q4)];
      const int s0 = logL - 1 - lh;  // twiddle stride L/(2h)
#pragma unroll
      for (int k = 0; k < 4; ++k) bf_dif(x[k], x[k + 4], (j + k * q4) << s0, W, Wc, p, p2);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        bf_dif(x[k], x[k + 2], (j + k * q4) << (s0 + 1), W, Wc, p, p2);
        bf_dif(x[k + 4], x[k + 6], (j + k * q4) << (s0 + 1), W, Wc, p, p2);
      }
#pragma unroll
      for (int k = 0; k < 8; k += 2) bf_dif(x[k], x[k + 1], j << (s0 + 2), W, Wc, p, p2);
#pragma unroll
      for (int k = 0; k < 8; ++k) buf[sidx<PAD>(base + j + k * q4)] = x[k];
    }
    __syncthreads();
  }
  // remaining stages lh = 1 (radix-4: h = 2, 1) or lh = 0 (radix-2: h = 1)
  if (lh == 1) {
    for (int g = threadIdx.x; g < (L >> 2); g += T) {
      const int base = g << 2;
      uint32_t x0 = buf[sidx<PAD>(base)], x1 = buf[sidx<PAD>(base + 1)], x2 = buf[sidx<PAD>(base + 2)], x3 = buf[sidx<PAD>(base + 3)];
      const int s0 = logL - 2;
      bf_dif(x0, x2, 0, W, Wc, p, p2);
      bf_dif(x1, x3, 1 << s0, W, Wc, p, p2);
      bf_dif(x0, x1, 0, W, Wc, p, p2);
      bf_dif(x2, x3, 0, W, Wc, p, p2);
      buf[sidx<PAD>(base)] = x0; buf[sidx<PAD>(base + 1)] = x1; buf[sidx<PAD>(base + 2)] = x2; buf[sidx<PAD>(base + 3)] = x3;
    }
    __syncthreads();
  } else if (lh == 0) {
    for (int g = threadIdx.x; g < (L >> 1); g += T) {
      uint32_t x0 = buf[sidx<PAD>(2 * g)], x1 = buf[sidx<PAD>(2 * g + 1)];
      bf_dif(x0, x1, 0, W, Wc, p, p2);
      buf[sidx<PAD>(2 * g)] = x0; buf[sidx<PAD>(2 * g + 1)] = x1;
    }
    __syncthreads();
  }
}

// inverse DIT (no 1/L): a radix-2 or radix-4 head, then passes of three
// stages (h, 2h, 4h) on 8 registers
template <int T, bool PAD = false>
__device__ __forceinline__ void ntt_dit8(uint32_t* buf, int logL, const uint32_t* Wi, const uint32_t* Wic, uint32_t p) {
  const int L = 1 << logL;
  const uint32_t p2 = 2u * p;
  int lh = 0;
  const int head = logL % 3;
  if (head == 1) {
    for (int g = threadIdx.x; g < (L >> 1); g += T) {
      uint32_t x0 = buf[sidx<PAD>(2 * g)], x1 = buf[sidx<PAD>(2 * g + 1)];
      bf_dit(x0, x1, 0, Wi, Wic, p, p2);
      buf[sidx<PAD>(2 * g)] = x0; buf[sidx<PAD>(2 * g + 1)] = x1;
    }
    __syncthreads();
    lh = 1;
  } else if (head == 2) {
    for (int g = threadIdx.x; g < (L >> 2); g += T) {
      const int base = g << 2;
      uint32_t x0 = buf[sidx<PAD>(base)], x1 = buf[sidx<PAD>(base + 1)], x2 = buf[sidx<PAD>(base + 2)], x3 = buf[sidx<PAD>(base + 3)];
      const int s1 = logL - 2;
      bf_dit(x0, x1, 0, Wi, Wic, p, p2);
      bf_dit(x2, x3, 0, Wi, Wic, p, p2);
      bf_dit(x0, x2, 0, Wi, Wic, p, p2);
      bf_dit(x1, x3, 1 << s1, Wi, Wic, p, p2);
      buf[sidx<PAD>(base)] = x0; buf[sidx<PAD>(base + 1)] = x1; buf[sidx<PAD>(base + 2)] = x2; buf[sidx<PAD>(base + 3)] = x3;
    }
    __syncthreads();
    lh = 2;
  }
  for (; lh + 3 <= logL; lh += 3) {
    // stages lh, lh+1, lh+2 with halves h = 2^lh, 2h, 4h; block size 8h
    const int h = 1 << lh;
    for (int g = threadIdx.x; g < (L >> 3); g += T) {
      const int j = g & (h - 1), base = (g >> lh) << (lh + 3);
      uint32_t x[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = buf[sidx<PAD>(base + j + k * h)];
      const int s0 = logL - 1 - lh;  // stride for half h
#pragma unroll
      for (int k = 0; k < 8; k += 2) bf_dit(x[k], x[k + 1], j << s0, Wi, Wic, p, p2);
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        bf_dit(x[k], x[k + 2], (j + k * h) << (s0 - 1), Wi, Wic, p, p2);
        bf_dit(x[k + 4], x[k + 6], (j + k * h) << (s0 - 1), Wi, Wic, p, p2);
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) bf_dit(x[k], x[k + 4], (j + k * h) << (s0 - 2), Wi, Wic, p, p2);
#pragma unroll
      for (int k = 0; k < 8; ++k) buf[sidx<PAD>(base + j + k * h)] = x[k];
    }
    __syncthreads();
  }
}

}  // namespace ckb

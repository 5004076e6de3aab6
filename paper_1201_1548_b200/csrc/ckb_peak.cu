// Roofline denominators for the integer-multiply-bound kernels, measured live.
//
// The images and interpolation kernels are bound by the fma-heavy pipe's
// high-half multiplies (IMAD.HI / IMAD.WIDE run at ~1/3 the IMAD rate on
// B200, tools/imad_peak.cu).  Their unit of work is one modular product; the
// densest form in the kernels is the Shoup pair of the elimination step
//     red(red(x*w - hi(x*w')p) + red(y*v - hi(y*v')p))      (2 products)
// so the peak is that op in 8 independent chains per thread on every SM; the
// fused remainders use a three-product Montgomery update, measured the same
// way.  Also reports raw IMAD / IMAD.HI / IMAD.WIDE rates for reference.
#include <cuda_runtime.h>

#include "../../include/curvekit_b200.h"
#include "ckb_modarith.cuh"

using namespace ckb;

namespace {

constexpr int CH = 8, IT = 2048;

__global__ void k_pk_imad(uint32_t* out, uint32_t s) {
  uint32_t x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = s + threadIdx.x * 7 + c;
  const uint32_t m = s | 1u;
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = x[c] * m + x[(c + 1) % CH];
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) r ^= x[c];
  if (r == 0x9e3779b9u) out[threadIdx.x] = r;
}

__global__ void k_pk_hi(uint32_t* out, uint32_t s) {
  uint32_t x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = s + threadIdx.x * 7 + c;
  const uint32_t m = s | 0x80000001u;
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = __umulhi(x[c], m) + x[c];
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) r ^= x[c];
  if (r == 0x9e3779b9u) out[threadIdx.x] = r;
}

__global__ void k_pk_wide(uint32_t* out, uint32_t s) {
  uint64_t x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = s + threadIdx.x * 7 + c;
  const uint32_t m = s | 1u;
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = (uint64_t)(uint32_t)x[c] * m + x[c];
  uint64_t r = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) r ^= x[c];
  if (r == 0x9e3779b9ull) out[threadIdx.x] = (uint32_t)r;
}

__global__ void k_pk_shoup2(uint32_t* out, uint32_t p, uint32_t w, uint32_t wc, uint32_t v, uint32_t vc) {
  uint32_t x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = (threadIdx.x * 7 + c) % p;
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      uint32_t a = red1(shoup_lazy(x[c], w, wc, p), p);
      uint32_t b = red1(shoup_lazy(x[(c + 1) % CH], v, vc, p), p);
      x[c] = red1(a + b, p);
    }
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) r ^= x[c];
  if (r == 0x9e3779b9u) out[threadIdx.x] = r;
}

// the fused remainder's update: three products summed in 64 bits, one
// signed Montgomery reduction (ckb_resultant.cuh mont3)
__global__ void k_pk_mont3(uint32_t* out, uint32_t p, uint32_t pinv, uint32_t a, uint32_t b, uint32_t c) {
  uint32_t x[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) x[k] = (threadIdx.x * 7 + k) % p;
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int k = 0; k < CH; ++k) {
      const uint64_t t = (uint64_t)x[k] * a + (uint64_t)x[(k + 1) % CH] * b + (uint64_t)x[(k + 2) % CH] * c;
      x[k] = (uint32_t)(t >> 32) - __umulhi((uint32_t)t * pinv, p) + p;
    }
  uint32_t r = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) r ^= x[k];
  if (r == 0x9e3779b9u) out[threadIdx.x] = r;
}

}  // namespace

extern "C" int ckb_measure_peak(float* out, int n) {
  // out[0..n): IMAD, IMAD.HI, IMAD.WIDE (T ops/s), Shoup-pair modular products,
  // three-product Montgomery modular products (T products/s)
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess) return -1;
  const int threads = 256, blocks = prop.multiProcessorCount * 8;
  uint32_t* buf = nullptr;
  if (cudaMalloc(&buf, 4096) != cudaSuccess) return -1;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const double per = (double)threads * blocks * IT * CH;
  const uint32_t p = 1073692673u;  // PRIMES30[0]
  const uint64_t w = 123456789u % p, v = 987654321u % p;
  const uint32_t wc = (uint32_t)((w << 32) / p), vc = (uint32_t)((v << 32) / p);
  uint32_t pinv = p;
  for (int i = 0; i < 5; ++i) pinv *= 2u - p * pinv;
  float ms[5] = {0, 0, 0, 0, 0};
  for (int k = 0; k < 5; ++k) {
    for (int rep = 0; rep < 2; ++rep) {  // first launch warms up
      cudaEventRecord(a);
      if (k == 0) k_pk_imad<<<blocks, threads>>>(buf, 3);
      if (k == 1) k_pk_hi<<<blocks, threads>>>(buf, 3);
      if (k == 2) k_pk_wide<<<blocks, threads>>>(buf, 3);
      if (k == 3) k_pk_shoup2<<<blocks, threads>>>(buf, p, (uint32_t)w, wc, (uint32_t)v, vc);
      if (k == 4) k_pk_mont3<<<blocks, threads>>>(buf, p, pinv, (uint32_t)w, (uint32_t)v, 55555555u % p);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms[k], a, b);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  if (e != cudaSuccess) return -1;
  float v5[5];
  for (int k = 0; k < 3; ++k) v5[k] = (float)(per / (ms[k] * 1e-3) / 1e12);
  v5[3] = (float)(2.0 * per / (ms[3] * 1e-3) / 1e12);
  v5[4] = (float)(3.0 * per / (ms[4] * 1e-3) / 1e12);
  for (int k = 0; k < n && k < 5; ++k) out[k] = v5[k];
  return 0;
}

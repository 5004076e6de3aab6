// Roofline denominators for the integer-multiply-bound kernels, measured live.
//
// The images and interpolation kernels are bound by the fma-heavy pipe's
// high-half multiplies (IMAD.HI / IMAD.WIDE run at ~1/3 the IMAD rate on
// B200, tools/imad_peak.cu).  Their unit of work is one modular product; the
// densest form in the kernels is the Shoup pair of the elimination step
//     red(red(x*w - hi(x*w')p) + red(y*v - hi(y*v')p))      (2 products)
// so the peak is that op on every SM at 64 warps per SM, the best of 1, 2 or 8
// independent chains per thread; the fused remainders use a three-product
// Montgomery update, measured the same way.  Also reports raw IMAD / IMAD.HI /
// IMAD.WIDE rates (8 chains) for reference.
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

template <int NC>
__global__ void k_pk_shoup2(uint32_t* out, uint32_t p, uint32_t w, uint32_t wc, uint32_t v, uint32_t vc) {
  uint32_t x[NC + 1];
#pragma unroll
  for (int c = 0; c <= NC; ++c) x[c] = (threadIdx.x * 7 + c) % p;
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      uint32_t a = red1(shoup_lazy(x[c], w, wc, p), p);
      uint32_t b = red1(shoup_lazy(x[c + 1], v, vc, p), p);
      x[c] = red1(a + b, p);
    }
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c <= NC; ++c) r ^= x[c];
  if (r == 0x9e3779b9u) out[threadIdx.x] = r;
}

// the fused remainder's update: three products summed in 64 bits, one
// signed Montgomery reduction (ckb_resultant.cuh mont3)
template <int NC>
__global__ void k_pk_mont3(uint32_t* out, uint32_t p, uint32_t pinv, uint32_t a, uint32_t b, uint32_t c) {
  uint32_t x[NC + 2];
#pragma unroll
  for (int k = 0; k < NC + 2; ++k) x[k] = (threadIdx.x * 7 + k) % p;
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int k = 0; k < NC; ++k) {
      const uint64_t t = (uint64_t)x[k] * a + (uint64_t)x[k + 1] * b + (uint64_t)x[k + 2] * c;
      x[k] = (uint32_t)(t >> 32) - __umulhi((uint32_t)t * pinv, p) + p;
    }
  uint32_t r = 0;
#pragma unroll
  for (int k = 0; k < NC + 2; ++k) r ^= x[k];
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
  // the modular-product peaks take the best of 1, 2 and 8 independent chains
  // per thread at 64 warps per SM (measured: fewer chains, more warps win)
  float ms[5] = {0, 0, 0, 0, 0};
  auto timed = [&](auto launch) {
    float best = 1e30f;
    for (int rep = 0; rep < 2; ++rep) {  // first launch warms up
      cudaEventRecord(a);
      launch();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float t = 0;
      cudaEventElapsedTime(&t, a, b);
      if (rep) best = t;
    }
    return best;
  };
  ms[0] = timed([&] { k_pk_imad<<<blocks, threads>>>(buf, 3); });
  ms[1] = timed([&] { k_pk_hi<<<blocks, threads>>>(buf, 3); });
  ms[2] = timed([&] { k_pk_wide<<<blocks, threads>>>(buf, 3); });
  const uint32_t v3 = 55555555u % p;
  // per-thread op counts differ with the chain count: normalise to ops per ms
  double shoup_rate = 0, mont_rate = 0;
  {
    const double t1 = timed([&] { k_pk_shoup2<1><<<blocks, threads>>>(buf, p, (uint32_t)w, wc, (uint32_t)v, vc); });
    const double t2 = timed([&] { k_pk_shoup2<2><<<blocks, threads>>>(buf, p, (uint32_t)w, wc, (uint32_t)v, vc); });
    const double t8 = timed([&] { k_pk_shoup2<8><<<blocks, threads>>>(buf, p, (uint32_t)w, wc, (uint32_t)v, vc); });
    shoup_rate = fmax(fmax(1.0 / t1, 2.0 / t2), 8.0 / t8);
  }
  {
    const double t1 = timed([&] { k_pk_mont3<1><<<blocks, threads>>>(buf, p, pinv, (uint32_t)w, (uint32_t)v, v3); });
    const double t2 = timed([&] { k_pk_mont3<2><<<blocks, threads>>>(buf, p, pinv, (uint32_t)w, (uint32_t)v, v3); });
    const double t8 = timed([&] { k_pk_mont3<8><<<blocks, threads>>>(buf, p, pinv, (uint32_t)w, (uint32_t)v, v3); });
    mont_rate = fmax(fmax(1.0 / t1, 2.0 / t2), 8.0 / t8);
  }
  cudaError_t e = cudaDeviceSynchronize();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  if (e != cudaSuccess) return -1;
  float v5[5];
  for (int k = 0; k < 3; ++k) v5[k] = (float)(per / (ms[k] * 1e-3) / 1e12);
  const double per1 = (double)threads * blocks * IT;  // ops per launch per chain
  v5[3] = (float)(2.0 * per1 * shoup_rate * 1e3 / 1e12);
  v5[4] = (float)(3.0 * per1 * mont_rate * 1e3 / 1e12);
  for (int k = 0; k < n && k < 5; ++k) out[k] = v5[k];
  return 0;
}

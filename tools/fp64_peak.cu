// Microbenchmark: can the FP64 pipe carry modular products next to (or instead
// of) the integer multiplier?  B200 runs FP64 FMA on its own pipe; the images
// kernel's fused update is bound by IMAD.WIDE / IMAD.HI on the fma-heavy pipe.
//
//   k_dfma      8 independent DFMA chains per thread (raw FP64 FMA rate)
//   k_fp3<NC>   the fused three-product update on doubles, signed-centred:
//               t = x0 a + x1 b + x2 c (exact, |t| < 2^53 for p < 2^26.5),
//               q = rint(t / p) via (t pinv + 1.5 2^52) - 1.5 2^52, r = t - q p
//   k_mont3<NC> the current integer update (ckb_resultant.cuh mont3)
//   k_mixed     even warps run mont3, odd warps fp3 (both pipes at once)
//
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/fp64_peak tools/fp64_peak.cu
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

constexpr int IT = 2048;

__global__ void k_dfma(double* out, double s) {
  double x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = s + threadIdx.x + c;
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = fma(x[c], 0.999999, 1e-7);
  double r = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) r += x[c];
  if (r == 1.2345) out[threadIdx.x] = r;
}

__global__ void k_imad(uint32_t* out, uint32_t s) {
  uint32_t x[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = s + threadIdx.x * 7 + c;
  const uint32_t m = s | 1u;
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) x[c] = x[c] * m + x[(c + 1) % 8];
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) r ^= x[c];
  if (r == 0x9e3779b9u) out[threadIdx.x] = r;
}

__device__ __forceinline__ double fp3(double x0, double a, double x1, double b, double x2, double c, double p,
                                      double pinv) {
  const double M = 6755399441055744.0;  // 1.5 * 2^52
  const double t = fma(x0, a, fma(x1, b, x2 * c));
  const double q = fma(t, pinv, M) - M;
  return fma(-q, p, t);
}

template <int NC>
__device__ __forceinline__ void fp3_loop(double* out, double p, double a, double b, double c) {
  const double pinv = 1.0 / p;
  double x[NC + 2];
#pragma unroll
  for (int k = 0; k < NC + 2; ++k) x[k] = (double)((threadIdx.x * 7 + k) % 1000) - 500.0;
  for (int i = 0; i < IT; ++i)
#pragma unroll
    for (int k = 0; k < NC; ++k) x[k] = fp3(x[k], a, x[k + 1], b, x[k + 2], c, p, pinv);
  double r = 0;
#pragma unroll
  for (int k = 0; k < NC + 2; ++k) r += x[k];
  if (r == 1.2345) out[threadIdx.x] = r;
}

template <int NC>
__global__ void k_fp3(double* out, double p, double a, double b, double c) {
  fp3_loop<NC>(out, p, a, b, c);
}

template <int NC>
__device__ __forceinline__ void mont3_loop(uint32_t* out, uint32_t p, uint32_t pinv, uint32_t a, uint32_t b,
                                           uint32_t c) {
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

template <int NC>
__global__ void k_mont3(uint32_t* out, uint32_t p, uint32_t pinv, uint32_t a, uint32_t b, uint32_t c) {
  mont3_loop<NC>(out, p, pinv, a, b, c);
}

template <int NC>
__global__ void k_mixed(uint32_t* out, uint32_t p, uint32_t pinv, uint32_t a, uint32_t b, uint32_t c, double pd,
                        double ad, double bd, double cd, int fp_every) {
  // warp w runs the FP64 update when w % fp_every == 0, else the integer one
  if (((threadIdx.x >> 5) % fp_every) == 0)
    fp3_loop<NC>((double*)out, pd, ad, bd, cd);
  else
    mont3_loop<NC>(out, p, pinv, a, b, c);
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  const int sms = prop.multiProcessorCount;
  void* buf;
  cudaMalloc(&buf, 1 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timed = [&](auto launch) {
    float best = 1e30f;
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float t;
      cudaEventElapsedTime(&t, e0, e1);
      if (r && t < best) best = t;
    }
    return (double)best;
  };
  const uint32_t p = 1073692673u;
  uint32_t pinv = p;
  for (int i = 0; i < 5; ++i) pinv *= 2u - p * pinv;
  const double pd = 67043329.0;  // < 2^26
  for (int threads : {256, 512}) {
    for (int bps : {2, 4, 8}) {
      const int blocks = sms * bps;
      const double lanes = (double)threads * blocks;
      double t = timed([&] { k_dfma<<<blocks, threads>>>((double*)buf, 1.0); });
      printf("threads %d blocks/SM %d: DFMA %.2f T/s (%.1f lanes/clk/SM @1965)\n", threads, bps,
             lanes * IT * 8 / t / 1e9, lanes * IT * 8 / (t * 1e-3) / sms / 1.965e9);
      t = timed([&] { k_imad<<<blocks, threads>>>((uint32_t*)buf, 3); });
      printf("   IMAD %.2f T/s\n", lanes * IT * 8 / t / 1e9);
#define RUNNC(NC)                                                                                                 \
  {                                                                                                               \
    double tf = timed([&] { k_fp3<NC><<<blocks, threads>>>((double*)buf, pd, 1234567.0, -7654321.0, 3333.0); }); \
    double ti = timed([&] { k_mont3<NC><<<blocks, threads>>>((uint32_t*)buf, p, pinv, 123456789u, 98765432u, 5555u); }); \
    double tm2 = timed([&] {                                                                                      \
      k_mixed<NC><<<blocks, threads>>>((uint32_t*)buf, p, pinv, 123456789u, 98765432u, 5555u, pd, 1234567.0,       \
                                       -7654321.0, 3333.0, 2);                                                    \
    });                                                                                                           \
    double tm3 = timed([&] {                                                                                      \
      k_mixed<NC><<<blocks, threads>>>((uint32_t*)buf, p, pinv, 123456789u, 98765432u, 5555u, pd, 1234567.0,       \
                                       -7654321.0, 3333.0, 3);                                                    \
    });                                                                                                           \
    const double outs = lanes * IT * NC;                                                                          \
    printf("   NC=%d fp3 %.2f T out/s | mont3 %.2f T out/s | mixed 1:1 %.2f | mixed 1fp:2int %.2f\n", NC,        \
           outs / tf / 1e9, outs / ti / 1e9, outs / tm2 / 1e9, outs / tm3 / 1e9);                                 \
  }
      RUNNC(1) RUNNC(2) RUNNC(4) RUNNC(8)
    }
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(err));
  return 0;
}

// Integer multiply-pipe microbenchmark for the roofline denominator.
//
// Measures, on the box it runs on, the sustained chip-wide rate of
//   imad     : IMAD (32x32 -> low 32)
//   imadwide : IMAD.WIDE.U32 (32x32 -> 64, with 64-bit addend)
//   imadhi   : IMAD.HI.U32
//   mont     : one 31-bit signed-Montgomery mulmod (the product kernels' unit)
//   mont2    : lazy two-product Montgomery (a*b + c*d) mod p, the PRS update
// using 8 independent dependency chains per thread, 148*k CTAs, CUDA events.
// Prints one JSON line.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CHAINS 8
#define ITERS 4096

__global__ void k_imad(uint32_t* out, uint32_t seed) {
  uint32_t x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = seed + threadIdx.x * 7 + c;
  const uint32_t m = seed | 1u;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = x[c] * m + (uint32_t)c;
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s ^= x[c];
  if (s == 0x12345678u) out[threadIdx.x] = s;
}

__global__ void k_imadwide(uint32_t* out, uint32_t seed) {
  uint64_t x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = seed + threadIdx.x * 7 + c;
  const uint32_t m = seed | 1u;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = (uint64_t)(uint32_t)x[c] * m + x[c];
  }
  uint64_t s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s ^= x[c];
  if (s == 0x12345678ull) out[threadIdx.x] = (uint32_t)s;
}

__global__ void k_imadhi(uint32_t* out, uint32_t seed) {
  uint32_t x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = seed + threadIdx.x * 7 + c;
  const uint32_t m = seed | 0x80000001u;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = __umulhi(x[c], m) + x[c];
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s ^= x[c];
  if (s == 0x12345678u) out[threadIdx.x] = s;
}

__device__ __forceinline__ uint32_t redc(uint64_t t, uint32_t p, uint32_t pinv) {
  uint32_t m = (uint32_t)t * pinv;
  int32_t u = (int32_t)((uint32_t)(t >> 32) - __umulhi(m, p));
  return (uint32_t)(u + ((u >> 31) & (int32_t)p));
}

__global__ void k_mont(uint32_t* out, uint32_t p, uint32_t pinv) {
  uint32_t x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = (threadIdx.x * 7 + c) % p;
  const uint32_t m = 123456789u % p;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = redc((uint64_t)x[c] * m, p, pinv);
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s ^= x[c];
  if (s == 0x12345678u) out[threadIdx.x] = s;
}

__global__ void k_mont2(uint32_t* out, uint32_t p, uint32_t pinv) {
  uint32_t x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = (threadIdx.x * 7 + c) % p;
  const uint32_t a = 123456789u % p, b = 987654321u % p;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      uint64_t t = (uint64_t)x[c] * a + (uint64_t)x[(c + 1) % CHAINS] * b;
      x[c] = redc(t, p, pinv);
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s ^= x[c];
  if (s == 0x12345678u) out[threadIdx.x] = s;
}


__global__ void k_dfma(uint32_t* out, double seed) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = seed + threadIdx.x * 7 + c;
  const double m = 0.999999, a = 1e-9;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], m, a);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 1.2345) out[threadIdx.x] = 1;
}

// balanced FP64 three-product modular update (p < 2^25, |values| <= p/2):
// t = a x + b y + c z exact (< 2^50), q = rint(t / p) via the 1.5 * 2^52 trick
__global__ void k_dmod3(uint32_t* out, double p, double pinv) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = (double)((threadIdx.x * 7 + c) % 1000) - 500.0;
  const double a = 12345.0, b = -54321.0, cc = 777777.0, magic = 6755399441055744.0;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      double t = x[c] * a;
      t = fma(x[(c + 1) % CHAINS], b, t);
      t = fma(x[(c + 2) % CHAINS], cc, t);
      const double q = fma(t, pinv, magic) - magic;
      x[c] = fma(-q, p, t);
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 1.2345) out[threadIdx.x] = 1;
}

// integer Montgomery three-product update (p < 2^30, values in [0, 4p))
__global__ void k_mont3(uint32_t* out, uint32_t p, uint32_t pinv) {
  uint32_t x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = (threadIdx.x * 7 + c) % p;
  const uint32_t a = 123456789u % p, b = 987654321u % p, cc = 55555555u % p;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) {
      uint64_t t = (uint64_t)x[c] * a + (uint64_t)x[(c + 1) % CHAINS] * b + (uint64_t)x[(c + 2) % CHAINS] * cc;
      x[c] = (uint32_t)(t >> 32) - __umulhi((uint32_t)t * pinv, p) + p;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s ^= x[c];
  if (s == 0x12345678u) out[threadIdx.x] = s;
}

// both at once: half the chains integer, half FP64 (do the pipes overlap?)
__global__ void k_mixed3(uint32_t* out, uint32_t p, uint32_t pinv, double pd, double pdinv) {
  uint32_t x[CHAINS / 2];
  double y[CHAINS / 2];
#pragma unroll
  for (int c = 0; c < CHAINS / 2; ++c) {
    x[c] = (threadIdx.x * 7 + c) % p;
    y[c] = (double)((threadIdx.x * 7 + c) % 1000) - 500.0;
  }
  const uint32_t a = 123456789u % p, b = 987654321u % p, cc = 55555555u % p;
  const double da = 12345.0, db = -54321.0, dc = 777777.0, magic = 6755399441055744.0;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS / 2; ++c) {
      uint64_t t = (uint64_t)x[c] * a + (uint64_t)x[(c + 1) % (CHAINS / 2)] * b +
                   (uint64_t)x[(c + 2) % (CHAINS / 2)] * cc;
      x[c] = (uint32_t)(t >> 32) - __umulhi((uint32_t)t * pinv, p) + p;
      double u = y[c] * da;
      u = fma(y[(c + 1) % (CHAINS / 2)], db, u);
      u = fma(y[(c + 2) % (CHAINS / 2)], dc, u);
      const double q = fma(u, pdinv, magic) - magic;
      y[c] = fma(-q, pd, u);
    }
  }
  uint32_t s = 0;
  double z = 0;
#pragma unroll
  for (int c = 0; c < CHAINS / 2; ++c) {
    s ^= x[c];
    z += y[c];
  }
  if (s == 0x12345678u || z == 1.2345) out[threadIdx.x] = s;
}

template <typename F>
static float time_kernel(F launch, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < reps; ++r) launch();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, 0);
  int sms = prop.multiProcessorCount;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  uint32_t* out;
  cudaMalloc(&out, 4096);
  const int threads = 256, blocks = sms * 8;
  const double nthreads = (double)threads * blocks;
  const uint32_t p = 2147483629u;  // < 2^31, prime
  uint32_t pinv = 1;               // p^-1 mod 2^32 by Newton
  for (int i = 0; i < 5; ++i) pinv *= 2u - p * pinv;
  const double ops = nthreads * ITERS * CHAINS;
  float t1 = time_kernel([&] { k_imad<<<blocks, threads>>>(out, 3); }, 5);
  float t2 = time_kernel([&] { k_imadwide<<<blocks, threads>>>(out, 3); }, 5);
  float t3 = time_kernel([&] { k_imadhi<<<blocks, threads>>>(out, 3); }, 5);
  float t4 = time_kernel([&] { k_mont<<<blocks, threads>>>(out, p, pinv); }, 5);
  float t5 = time_kernel([&] { k_mont2<<<blocks, threads>>>(out, p, pinv); }, 5);
  const uint32_t p30 = 1073692673u;  // < 2^30
  uint32_t pinv30 = 1;
  for (int i = 0; i < 5; ++i) pinv30 *= 2u - p30 * pinv30;
  const double pd = 33292289.0;       // prime < 2^25
  float t6 = time_kernel([&] { k_dfma<<<blocks, threads>>>(out, 1.0); }, 5);
  float t7 = time_kernel([&] { k_dmod3<<<blocks, threads>>>(out, pd, 1.0 / pd); }, 5);
  float t8 = time_kernel([&] { k_mont3<<<blocks, threads>>>(out, p30, pinv30); }, 5);
  float t9 = time_kernel([&] { k_mixed3<<<blocks, threads>>>(out, p30, pinv30, pd, 1.0 / pd); }, 5);
  cudaError_t e = cudaDeviceSynchronize();
  printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"err\": \"%s\", "
         "\"imad_tops\": %.3f, \"imadwide_tops\": %.3f, \"imadhi_tops\": %.3f, "
         "\"mont_mulmod_tops\": %.3f, \"mont2_tops\": %.3f, \"dfma_tops\": %.3f, "
         "\"dmod3_updates_t\": %.3f, \"mont3_updates_t\": %.3f, \"mixed3_updates_t\": %.3f}\n",
         sms, clk_khz / 1e3, cudaGetErrorString(e), ops / t1 / 1e9, ops / t2 / 1e9,
         ops / t3 / 1e9, ops / t4 / 1e9, ops / t5 / 1e9, ops / t6 / 1e9, ops / t7 / 1e9, ops / t8 / 1e9,
         ops / t9 / 1e9);
  return 0;
}

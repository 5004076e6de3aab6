// How does the three-product Montgomery update rate depend on warps per
// scheduler and independent chains per thread?  (the images kernel runs 4
// warps per scheduler with ~2 chains in flight)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int CH>
__global__ void k_mont3(uint32_t* out, uint32_t p, uint32_t pinv, int iters) {
  uint32_t x[CH + 2];
#pragma unroll
  for (int c = 0; c < CH + 2; ++c) x[c] = (threadIdx.x * 7 + c) % p;
  const uint32_t a = 123456789u % p, b = 987654321u % p, cc = 55555555u % p;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      uint64_t t = (uint64_t)x[c] * a + (uint64_t)x[c + 1] * b + (uint64_t)x[c + 2] * cc;
      x[c] = (uint32_t)(t >> 32) - __umulhi((uint32_t)t * pinv, p) + p;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH + 2; ++c) s ^= x[c];
  if (s == 0x12345678u) out[threadIdx.x] = s;
}

template <int CH>
void run(int warps_per_sm, uint32_t* out) {
  const uint32_t p = 1073692673u;
  uint32_t pinv = p;
  for (int i = 0; i < 5; ++i) pinv *= 2u - p * pinv;
  const int threads = 128, blocks = 148 * warps_per_sm / 4;
  const int iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_mont3<CH><<<blocks, threads>>>(out, p, pinv, iters);
  cudaEventRecord(e0);
  k_mont3<CH><<<blocks, threads>>>(out, p, pinv, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double upd = (double)blocks * threads * iters * CH;
  printf("{\"warps_per_sm\": %d, \"chains\": %d, \"T_updates_per_s\": %.3f}\n", warps_per_sm, CH, upd / ms / 1e9);
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 4096);
  for (int w : {8, 16, 32, 64}) {
    run<1>(w, out);
    run<2>(w, out);
    run<4>(w, out);
    run<8>(w, out);
  }
  return 0;
}

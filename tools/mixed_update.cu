// Three-product modular update on the integer pipe, on the FP64 pipe with
// uint32 storage (magic-number conversions), and both interleaved, at the
// images kernel's occupancy (16 warps per SM).  Does the FP64 pipe add
// throughput for register-resident uint32 operands?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t upd_int(uint32_t x, uint32_t y, uint32_t z, uint32_t a, uint32_t b, uint32_t c,
                                            uint32_t pinv, uint32_t p) {
  const uint64_t t = (uint64_t)x * a + (uint64_t)y * b + (uint64_t)z * c;
  return (uint32_t)(t >> 32) - __umulhi((uint32_t)t * pinv, p) + p;
}
// p < 2^25; x,y,z in [0, 2p) as uint32; multipliers a,b,c balanced doubles (|.| <= p/2)
__device__ __forceinline__ uint32_t upd_fp(uint32_t x, uint32_t y, uint32_t z, double a, double b, double c, double pd,
                                           double pinvd) {
  const double M52 = 4503599627370496.0;  // 2^52
  const double dx = __hiloint2double(0x43300000, (int)x) - M52;
  const double dy = __hiloint2double(0x43300000, (int)y) - M52;
  const double dz = __hiloint2double(0x43300000, (int)z) - M52;
  double t = dx * a;
  t = fma(dy, b, t);
  t = fma(dz, c, t);
  const double magic = 6755399441055744.0;  // 1.5 * 2^52
  const double q = fma(t, pinvd, magic) - magic;
  const double r = fma(-q, pd, t);              // |r| <= ~p/2
  const double rr = r + magic;                  // low word = r as int32
  return (uint32_t)__double2loint(rr) + (uint32_t)pd;  // [p/2, 3p/2)
}

template <int MODE, int CH>
__global__ void k(uint32_t* out, uint32_t p, uint32_t pinv, int iters) {
  uint32_t x[CH + 2];
#pragma unroll
  for (int c = 0; c < CH + 2; ++c) x[c] = (threadIdx.x * 7 + c) % p;
  const uint32_t a = 1234567u % p, b = 7654321u % p, c3 = 5555555u % p;
  const double pd = (double)p, pinvd = 1.0 / pd;
  const double da = (double)(int)(a % p) - (a > p / 2 ? pd : 0), db = -12345.0, dc = 77777.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (MODE == 0 || (MODE == 2 && (c & 1) == 0))
        x[c] = upd_int(x[c], x[c + 1], x[c + 2], a, b, c3, pinv, p);
      else
        x[c] = upd_fp(x[c], x[c + 1], x[c + 2], da, db, dc, pd, pinvd);
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < CH + 2; ++c) s ^= x[c];
  if (s == 0x12345678u) out[threadIdx.x] = s;
}

template <int MODE, int CH>
void run(const char* name, int warps_per_sm, uint32_t* out, uint32_t p, uint32_t pinv) {
  const int threads = 128, blocks = 148 * warps_per_sm / 4, iters = 2048;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<MODE, CH><<<blocks, threads>>>(out, p, pinv, iters);
  cudaEventRecord(e0);
  k<MODE, CH><<<blocks, threads>>>(out, p, pinv, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"mode\": \"%s\", \"warps_per_sm\": %d, \"chains\": %d, \"T_updates_per_s\": %.3f}\n", name, warps_per_sm,
         CH, (double)blocks * threads * iters * CH / ms / 1e9);
}

int main() {
  uint32_t* out;
  cudaMalloc(&out, 4096);
  const uint32_t p = 33292289u;  // prime < 2^25
  uint32_t pinv = p;
  for (int i = 0; i < 5; ++i) pinv *= 2u - p * pinv;
  for (int w : {16, 32}) {
    run<0, 2>("int", w, out, p, pinv);
    run<0, 4>("int", w, out, p, pinv);
    run<1, 2>("fp64", w, out, p, pinv);
    run<1, 4>("fp64", w, out, p, pinv);
    run<2, 2>("mixed", w, out, p, pinv);
    run<2, 4>("mixed", w, out, p, pinv);
  }
  printf("{\"err\": \"%s\"}\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}

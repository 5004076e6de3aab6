// K4: interpolation of each prime's image values at the planned geometric
// points x_t = c q^t.  Replaces the reference's Newton divided differences
// with a Fermat inverse inside the O(N^2) loop (pkg/src/curvekit/
// modpoly.py:164-185) by the Lagrange form with closed-form weights:
//   P~(y) = sum_t u_t M~(y)/(y - q^t),  M~(y) = prod_t (y - q^t),  u_t = v_t / M~'(q^t)
//   P~_k  = sum_{l>k} M~_l S_{l-k-1},   S_e = sum_t u_t q^(t e)
//   q^(t e) = q^C(t+e,2) q^-C(t,2) q^-C(e,2)   (chirp identity)
// so both O(N^2) stages are structured (Hankel, then triangular Toeplitz)
// products against per-prime plan tables, fully parallel over the output
// index, with no inverse anywhere.  P_k = P~_k c^-k undoes the scaling.
#include "ckb_kernels.cuh"

namespace ckb {

constexpr int INT_THREADS = 128;

// acc < p * 2^32  ->  acc mod p
__device__ __forceinline__ uint32_t mod64(uint64_t acc, const Prime& P) {
  return redc((uint64_t)redc(acc, P) * P.r2, P);
}

// a_t = v_t * z_t, with its Shoup companion
__global__ void k_interp_prologue(InterpPlan plan, const Prime* __restrict__ primes,
                                  const uint32_t* __restrict__ values, uint32_t* __restrict__ a,
                                  uint32_t* __restrict__ ac) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x, pi = blockIdx.y, N = plan.N;
  if (t >= N) return;
  const Prime P = primes[pi];
  const size_t o = (size_t)pi * N + t;
  const uint32_t v = mul_mod(values[o], plan.z[o], P);
  a[o] = v;
  ac[o] = shoup_comp(v, P);
}

// S_e = q^-C(e,2) * sum_t a_t q^C(t+e,2)
__global__ void __launch_bounds__(INT_THREADS) k_interp_hankel(InterpPlan plan, const Prime* __restrict__ primes,
                                                               const uint32_t* __restrict__ a,
                                                               const uint32_t* __restrict__ ac,
                                                               uint32_t* __restrict__ S) {
  extern __shared__ uint32_t sm[];
  const int N = plan.N, pi = blockIdx.y, e0 = blockIdx.x * INT_THREADS;
  uint32_t* sa = sm;
  uint32_t* sac = sm + N;
  uint32_t* sh = sm + 2 * N;  // hC[e0 .. e0 + INT_THREADS + N - 1)
  const size_t oN = (size_t)pi * N, o2N = (size_t)pi * 2 * N;
  for (int i = threadIdx.x; i < N; i += INT_THREADS) {
    sa[i] = a[oN + i];
    sac[i] = ac[oN + i];
  }
  const int hn = min(INT_THREADS + N, 2 * N - e0);
  for (int i = threadIdx.x; i < hn; i += INT_THREADS) sh[i] = plan.hC[o2N + e0 + i];
  __syncthreads();
  const int e = e0 + threadIdx.x;
  if (e >= N) return;
  const Prime P = primes[pi];
  const uint32_t p = P.p;
  uint64_t acc = 0;
  const uint32_t* hh = sh + threadIdx.x;
#pragma unroll 4
  for (int t = 0; t < N; ++t) acc += shoup_lazy(hh[t], sa[t], sac[t], p);
  S[oN + e] = mul_mod(mod64(acc, P), plan.hCinv[oN + e], P);
}

// P_k = c^-k * sum_{l=k+1..N} M~_l S_{l-k-1}
__global__ void __launch_bounds__(INT_THREADS) k_interp_toeplitz(InterpPlan plan, const Prime* __restrict__ primes,
                                                                 const uint32_t* __restrict__ S,
                                                                 uint32_t* __restrict__ coeffs) {
  extern __shared__ uint32_t sm[];
  const int N = plan.N, pi = blockIdx.y;
  uint32_t* sS = sm;
  uint32_t* sM = sm + N;
  uint32_t* sMc = sm + 2 * N + 1;
  const size_t oN = (size_t)pi * N, oN1 = (size_t)pi * (N + 1);
  for (int i = threadIdx.x; i < N; i += INT_THREADS) sS[i] = S[oN + i];
  for (int i = threadIdx.x; i <= N; i += INT_THREADS) {
    sM[i] = plan.Mt[oN1 + i];
    sMc[i] = plan.Mtc[oN1 + i];
  }
  __syncthreads();
  const int k = blockIdx.x * INT_THREADS + threadIdx.x;
  if (k >= N) return;
  const Prime P = primes[pi];
  const uint32_t p = P.p;
  uint64_t acc = 0;
#pragma unroll 4
  for (int l = k + 1; l <= N; ++l) acc += shoup_lazy(sS[l - k - 1], sM[l], sMc[l], p);
  coeffs[oN + k] = mul_mod(mod64(acc, P), plan.cinv[oN + k], P);
}

void launch_interp(const InterpPlan& plan, const Prime* primes, const uint32_t* values, uint32_t* coeffs,
                   uint32_t* a, uint32_t* ac, uint32_t* S, cudaStream_t st) {
  const int N = plan.N, K = plan.K;
  k_interp_prologue<<<dim3((N + 255) / 256, K), 256, 0, st>>>(plan, primes, values, a, ac);
  const dim3 grid((N + INT_THREADS - 1) / INT_THREADS, K);
  const size_t sm1 = (size_t)(3 * N + INT_THREADS) * 4;
  const size_t sm2 = (size_t)(3 * N + 2) * 4;
  if (sm1 > 48 * 1024) cudaFuncSetAttribute(k_interp_hankel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1);
  if (sm2 > 48 * 1024) cudaFuncSetAttribute(k_interp_toeplitz, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2);
  k_interp_hankel<<<grid, INT_THREADS, sm1, st>>>(plan, primes, a, ac, S);
  k_interp_toeplitz<<<grid, INT_THREADS, sm2, st>>>(plan, primes, S, coeffs);
}

}  // namespace ckb

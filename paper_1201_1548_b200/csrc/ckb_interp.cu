// K4: interpolation of each prime's image values at the planned geometric
// points x_t = c q^t.  Replaces the reference's Newton divided differences
// with a Fermat inverse inside the O(N^2) loop (pkg/src/curvekit/
// modpoly.py:164-185) by the Lagrange form with closed-form weights:
//   P~(y) = sum_t u_t M~(y)/(y - q^t),  M~(y) = prod_t (y - q^t),  u_t = v_t / M~'(q^t)
//   P~_k  = sum_{j} S_j M~_{k+1+j},     S_e = sum_t u_t q^(t e)
//   q^(t e) = q^C(t+e,2) q^-C(t,2) q^-C(e,2)             (chirp identity)
// Both sums are correlations with per-(prime, N) constant sequences, done as
// cyclic convolutions of length L = 2^ceil(log2(2N-1)) with NTTs (our primes
// are 1 mod 2^14): 4 transforms of length L per prime instead of 1.5 N^2
// products.  The transforms of the constant operands live in the cached plan.
// P_k = P~_k c^-k undoes the point scale.
#include "ckb_kernels.cuh"
#include "ckb_ntt.cuh"

namespace ckb {

constexpr int NTT_THREADS = 512;
constexpr int MAX_PER_THREAD = 16;  // N <= 16 * 512

// plan, part 1: twiddles, 1/L, and the Shoup companions of the pointwise tables
__global__ void __launch_bounds__(NTT_THREADS) k_plan_twiddles(const Prime* __restrict__ primes,
                                                               const uint32_t* __restrict__ gens, InterpPlan plan) {
  const int pi = blockIdx.x, tid = threadIdx.x, T = blockDim.x;
  const Prime P = primes[pi];
  const uint32_t p = P.p;
  const int N = plan.N, L = plan.L, half = L >> 1;
  const uint32_t w = pow_mod(gens[pi] % p, (uint64_t)(p - 1) >> plan.logL, P);  // primitive L-th root
  const uint32_t wi = inv_mod(w, P);
  const uint32_t wc = shoup_comp(w, P), wic = shoup_comp(wi, P);
  const size_t oH = (size_t)pi * half, oN = (size_t)pi * N;
  const int seg = (half + T - 1) / T;
  const int s0 = min(half, tid * seg), s1 = min(half, s0 + seg);
  if (s0 < s1) {
    uint32_t a = pow_mod(w, s0, P), b = pow_mod(wi, s0, P);
    for (int j = s0; j < s1; ++j) {
      plan.W[oH + j] = a;
      plan.Wc[oH + j] = shoup_comp(a, P);
      plan.Wi[oH + j] = b;
      plan.Wic[oH + j] = shoup_comp(b, P);
      a = shoup(a, w, wc, p);
      b = shoup(b, wi, wic, p);
    }
  }
  const uint32_t linv = inv_mod((uint32_t)L % p, P);
  if (tid == 0) plan.Linv[pi] = linv;
  for (int e = tid; e < N; e += T) {
    const uint32_t s = mul_mod(plan.hCinv[oN + e], linv, P);
    plan.sS[oN + e] = s;
    plan.sSc[oN + e] = shoup_comp(s, P);
    plan.zc[oN + e] = shoup_comp(plan.z[oN + e], P);
  }
}

// plan, part 2: DIF transforms of the chirp q^C(m,2) (m < 2N-1) and of M~_{u+1} (u < N)
__global__ void __launch_bounds__(NTT_THREADS) k_plan_transforms(const Prime* __restrict__ primes, InterpPlan plan) {
  extern __shared__ uint32_t buf[];
  CKB_SMEM_POISON(buf);
  const int pi = blockIdx.x, tid = threadIdx.x, T = blockDim.x;
  const Prime P = primes[pi];
  const uint32_t p = P.p;
  const int N = plan.N, L = plan.L;
  const size_t oL = (size_t)pi * L, oH = (size_t)pi * (L >> 1);
  const size_t o2N = (size_t)pi * 2 * N, oN1 = (size_t)pi * (N + 1);
  const uint32_t* W = plan.W + oH;
  const uint32_t* Wc = plan.Wc + oH;
  for (int m = tid; m < L; m += T) buf[m] = (m < 2 * N - 1) ? plan.hC[o2N + m] : 0u;
  __syncthreads();
  ntt_dif(buf, plan.logL, W, Wc, p);
  for (int u = tid; u < L; u += T) {
    const uint32_t v = red1(buf[u], p);
    plan.Hf[oL + u] = v;
    plan.Hfc[oL + u] = shoup_comp(v, P);
  }
  __syncthreads();
  for (int u = tid; u < L; u += T) buf[u] = (u < N) ? plan.Mt[oN1 + u + 1] : 0u;
  __syncthreads();
  ntt_dif(buf, plan.logL, W, Wc, p);
  for (int u = tid; u < L; u += T) {
    const uint32_t v = red1(buf[u], p);
    plan.Mf[oL + u] = v;
    plan.Mfc[oL + u] = shoup_comp(v, P);
  }
}

// polyphase input weights zr[pi][r][t] = (1/S) y_t^-r z_t: the per-element
// factor of the phase-r interpolation, tabled once per plan
__global__ void k_plan_zr(const Prime* __restrict__ primes, InterpPlan plan) {
  const int pi = blockIdx.y, r = blockIdx.z, S = plan.S, M = plan.N;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= M) return;
  const Prime P = primes[pi];
  const uint32_t invS = inv_mod((uint32_t)S % P.p, P);
  const size_t o = (size_t)pi * M + t;
  const uint32_t w = mul_mod(mul_mod(invS, pow_mod(plan.yqi[o], (uint64_t)r, P), P), plan.z[o], P);
  const size_t q = ((size_t)pi * S + r) * M + t;
  plan.zr[q] = w;
  plan.zrc[q] = shoup_comp(w, P);
}

void launch_plan_ntt(const Prime* primes, const uint32_t* gens, const InterpPlan& plan, cudaStream_t st) {
  if (plan.S > 1) k_plan_zr<<<dim3((plan.N + 127) / 128, plan.K, plan.S), 128, 0, st>>>(primes, plan);
  k_plan_twiddles<<<plan.K, NTT_THREADS, 0, st>>>(primes, gens, plan);
  const size_t smem = (size_t)plan.L * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_plan_transforms, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_plan_transforms<<<plan.K, NTT_THREADS, smem, st>>>(primes, plan);
}

// per call: values -> coefficients, one CTA per prime, everything in shared memory
__global__ void __launch_bounds__(NTT_THREADS) k_interp(InterpPlan plan, const Prime* __restrict__ primes,
                                                        const uint32_t* __restrict__ values,
                                                        const uint32_t* __restrict__ cval,
                                                        uint32_t* __restrict__ coeffs) {
  extern __shared__ uint32_t buf[];  // [L] data, then 4 x [L/2] twiddle tables
  CKB_SMEM_POISON(buf);
  const int pi = blockIdx.x, tid = threadIdx.x, T = blockDim.x;
  const Prime P = primes[pi];
  const uint32_t p = P.p;
  const int N = plan.N, L = plan.L, logL = plan.logL, half = L >> 1;
  const size_t oN = (size_t)pi * N, oL = (size_t)pi * L, oH = (size_t)pi * half;
  uint32_t *W = buf + L, *Wc = W + half, *Wi = Wc + half, *Wic = Wi + half;
  for (int j = tid; j < half; j += T) {  // stage the twiddles once (no global loads in the stages)
    W[j] = plan.W[oH + j];
    Wc[j] = plan.Wc[oH + j];
    Wi[j] = plan.Wi[oH + j];
    Wic[j] = plan.Wic[oH + j];
  }
  const uint32_t *Hf = plan.Hf + oL, *Hfc = plan.Hfc + oL, *Mf = plan.Mf + oL, *Mfc = plan.Mfc + oL;
  const uint32_t* v = values + oN;
  // a'_s = u_{N-1-s} q^-C(N-1-s,2) = v_t z_t with t = N-1-s
  for (int s = tid; s < L; s += T) {
    uint32_t a = 0u;
    if (s < N) {
      const int t = N - 1 - s;
      a = shoup_lazy(v[t], plan.z[oN + t], plan.zc[oN + t], p);
    }
    buf[s] = a;
  }
  __syncthreads();
  ntt_dif8<NTT_THREADS>(buf, logL, W, Wc, p);
  for (int u = tid; u < L; u += T) buf[u] = shoup_lazy(buf[u], Hf[u], Hfc[u], p);
  __syncthreads();
  ntt_dit8<NTT_THREADS>(buf, logL, Wi, Wic, p);
  // S_e = conv[N-1+e] q^-C(e,2) / L, then s'_u = S_{N-1-u}
  uint32_t sv[MAX_PER_THREAD];
#pragma unroll
  for (int r = 0; r < MAX_PER_THREAD; ++r) {
    const int e = tid + r * T;
    sv[r] = (e < N) ? shoup_lazy(buf[N - 1 + e], plan.sS[oN + e], plan.sSc[oN + e], p) : 0u;
  }
  __syncthreads();
  for (int u = tid; u < L; u += T) buf[u] = 0u;
  __syncthreads();
#pragma unroll
  for (int r = 0; r < MAX_PER_THREAD; ++r) {
    const int e = tid + r * T;
    if (e < N) buf[N - 1 - e] = sv[r];
  }
  __syncthreads();
  ntt_dif8<NTT_THREADS>(buf, logL, W, Wc, p);
  for (int u = tid; u < L; u += T) buf[u] = shoup_lazy(buf[u], Mf[u], Mfc[u], p);
  __syncthreads();
  ntt_dit8<NTT_THREADS>(buf, logL, Wi, Wic, p);
  // P_k = conv[N-1+k] / L * c^-k
  const uint32_t linv = plan.Linv[pi];
  const uint32_t linvc = shoup_comp(linv, P);
  const uint32_t c = cval[pi];
  const uint32_t cinv = (c == 1u) ? 1u : inv_mod(c, P);
  for (int k = tid; k < N; k += T) {
    uint32_t r = shoup(buf[N - 1 + k], linv, linvc, p);
    if (c != 1u) r = mul_mod(r, pow_mod(cinv, (uint64_t)k, P), P);
    coeffs[oN + k] = r;
  }
}

// Polyphase plan (S > 1): images v[u S + j] at x = w^j y_u, y_u = c g^u.  With
// P(x) = sum_{r<S} x^r P_r(x^S):  P_r(z_u) = (1/S) y_u^-r sum_j w^-jr v[u S + j],
// z_u = y_u^S = c^S q^u (q = g^S) -- S independent geometric interpolations of
// size M, one CTA per (prime, r), interleaved into P_{S k + r}.
// threads per CTA = the radix-8 passes' L/8 groups, clamped to [32, 256]

// cp.async (LDGSTS) copies global -> shared without a register round trip, so
// every constant table of a CTA is requested at once at kernel entry and lands
// while the input gather runs (one L2 latency instead of one per table)
__device__ __forceinline__ void cp_async16(uint32_t* sdst, const uint32_t* gsrc) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t* sdst, const uint32_t* gsrc) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
// n words (n % 4 == 0, both pointers 16-byte aligned) by the CTA
__device__ __forceinline__ void stage16(uint32_t* sdst, const uint32_t* gsrc, int n, int tid, int T) {
  for (int i = 4 * tid; i < n; i += 4 * T) cp_async16(sdst + i, gsrc + i);
}

// STAGE: the pointwise tables (Hf, Hfc, Mf, Mfc, sS, sSc — each element read once
// per CTA) are staged in shared memory with the twiddles; by default they are
// read from global memory (L2) where used, which keeps shared memory to the data
// and twiddles (staging them cost occupancy: 3 CTAs per SM at L = 2048)
template <int POLY_THREADS, bool STAGE = true>
__global__ void __launch_bounds__(POLY_THREADS) k_interp_poly(InterpPlan plan, const Prime* __restrict__ primes,
                                                              const uint32_t* __restrict__ values,
                                                              const uint32_t* __restrict__ cval,
                                                              uint32_t* __restrict__ coeffs,
                                                              const uint32_t* __restrict__ crt_c,
                                                              const uint32_t* __restrict__ crt_cc, PeerOut po) {
  // shared: [L] data (one pad word per 8, sidx) | W, Wc, Wi, Wic [L/2 each] | Hf, Hfc, Mf, Mfc [L each] | sS, sSc [Mp each]
  extern __shared__ __align__(16) uint32_t buf[];
  CKB_SMEM_POISON(buf);
  const int S = plan.S;
  const int pi = blockIdx.x / S, r = blockIdx.x % S, tid = threadIdx.x, T = blockDim.x;
  const Prime P = primes[pi];
  const uint32_t p = P.p;
  const int M = plan.N, L = plan.L, logL = plan.logL, half = L >> 1, Nfull = plan.Nfull;
  const int Mp = (M + 3) & ~3, Lp = (L + 3) & ~3, hp = (half + 3) & ~3;  // 16-byte aligned regions
  const size_t oM = (size_t)pi * M, oL = (size_t)pi * L, oH = (size_t)pi * half;
  uint32_t *W = buf + ((padded_words(L) + 3) & ~3), *Wc = W + hp, *Wi = Wc + hp, *Wic = Wi + hp;
  uint32_t *sHf = Wic + hp, *sHfc = sHf + Lp, *sMf = sHfc + Lp, *sMfc = sMf + Lp;
  uint32_t *ssS = sMfc + Lp, *ssSc = ssS + Mp;
  const uint32_t* Hf = STAGE ? sHf : plan.Hf + oL;
  const uint32_t* Hfc = STAGE ? sHfc : plan.Hfc + oL;
  const uint32_t* Mf = STAGE ? sMf : plan.Mf + oL;
  const uint32_t* Mfc = STAGE ? sMfc : plan.Mfc + oL;
  const uint32_t* sS = STAGE ? ssS : plan.sS + oM;
  const uint32_t* sSc = STAGE ? ssSc : plan.sSc + oM;
  // every per-plan constant this CTA needs, requested up front (16-byte copies
  // when the per-prime table offsets are 16-byte aligned: L >= 8)
  if (L >= 8) {
    stage16(W, plan.W + oH, half, tid, T);
    stage16(Wc, plan.Wc + oH, half, tid, T);
    stage16(Wi, plan.Wi + oH, half, tid, T);
    stage16(Wic, plan.Wic + oH, half, tid, T);
    if (STAGE) {
      stage16(sHf, plan.Hf + oL, L, tid, T);
      stage16(sHfc, plan.Hfc + oL, L, tid, T);
      stage16(sMf, plan.Mf + oL, L, tid, T);
      stage16(sMfc, plan.Mfc + oL, L, tid, T);
    }
  } else {
    for (int j = tid; j < half; j += T) {
      cp_async4(W + j, plan.W + oH + j);
      cp_async4(Wc + j, plan.Wc + oH + j);
      cp_async4(Wi + j, plan.Wi + oH + j);
      cp_async4(Wic + j, plan.Wic + oH + j);
    }
    for (int j = tid; j < L && STAGE; j += T) {
      cp_async4(sHf + j, plan.Hf + oL + j);
      cp_async4(sHfc + j, plan.Hfc + oL + j);
      cp_async4(sMf + j, plan.Mf + oL + j);
      cp_async4(sMfc + j, plan.Mfc + oL + j);
    }
  }
  for (int e = tid; e < M && STAGE; e += T) {
    cp_async4(ssS + e, plan.sS + oM + e);
    cp_async4(ssSc + e, plan.sSc + oM + e);
  }
  // pdl_launch();  (implicit at exit: measured better)
  pdl_wait();  // the images kernels' values and k_choose_c's point scales from here on
  const uint32_t* om = plan.om + (size_t)pi * 4 * S;
  const uint32_t c = cval[pi];
  // c^-r (the shifted point set; 1 almost always)
  const uint32_t cr = (c == 1u) ? 1u : pow_mod(inv_mod(c, P), (uint64_t)r, P);
  const uint32_t crc = shoup_comp(cr, P);
  const uint32_t* zr = plan.zr + ((size_t)pi * S + r) * M;
  const uint32_t* zrc = plan.zrc + ((size_t)pi * S + r) * M;
  const uint32_t* v = values + (size_t)pi * M * S;
  // a'_s = P_r(z_t) * zweight_t with t = M-1-s (global loads overlap the copies above)
  for (int s = tid; s < L; s += T) {
    uint32_t a = 0u;
    if (s < M) {
      const int t = M - 1 - s;
      uint32_t g = 0u;
#pragma unroll 8
      for (int j = 0; j < S; ++j) {
        const int k = (j * r) & (S - 1);
        g = add_mod(g, shoup(v[(size_t)t * S + j], om[2 * S + k], om[3 * S + k], p), p);
      }
      if (c != 1u) g = shoup(g, cr, crc, p);
      a = shoup_lazy(g, zr[t], zrc[t], p);  // (1/S) y_t^-r z_t
    }
    buf[sidx<true>(s)] = a;
  }
  cp_async_wait_all();
  __syncthreads();
  ntt_dif8<POLY_THREADS, true>(buf, logL, W, Wc, p);
  for (int u = tid; u < L; u += T) buf[sidx<true>(u)] = shoup_lazy(buf[sidx<true>(u)], Hf[u], Hfc[u], p);
  __syncthreads();
  ntt_dit8<POLY_THREADS, true>(buf, logL, Wi, Wic, p);
  uint32_t sv[MAX_PER_THREAD];
#pragma unroll
  for (int q = 0; q < MAX_PER_THREAD; ++q) {
    const int e = tid + q * T;
    sv[q] = (e < M) ? shoup_lazy(buf[sidx<true>(M - 1 + e)], sS[e], sSc[e], p) : 0u;
  }
  __syncthreads();
  for (int u = tid; u < L; u += T) buf[sidx<true>(u)] = 0u;
  __syncthreads();
#pragma unroll
  for (int q = 0; q < MAX_PER_THREAD; ++q) {
    const int e = tid + q * T;
    if (e < M) buf[sidx<true>(M - 1 - e)] = sv[q];
  }
  __syncthreads();
  ntt_dif8<POLY_THREADS, true>(buf, logL, W, Wc, p);
  for (int u = tid; u < L; u += T) buf[sidx<true>(u)] = shoup_lazy(buf[sidx<true>(u)], Mf[u], Mfc[u], p);
  __syncthreads();
  ntt_dit8<POLY_THREADS, true>(buf, logL, Wi, Wic, p);
  // P_r[k] = conv[M-1+k] / L * (c^S)^-k  ->  coefficient S k + r
  const uint32_t linv = plan.Linv[pi];
  const uint32_t linvc = shoup_comp(linv, P);
  const uint32_t cS = (c == 1u) ? 1u : pow_mod(inv_mod(c, P), (uint64_t)S, P);
  // optional CRT pre-multiplication y = coeff (M/p)^-1 mod p (ckb_crt.cu), so
  // the CRT needs no separate pass over the residues
  uint32_t fin = linv, finc = linvc;
  if (crt_c) {
    fin = shoup(crt_c[pi], linv, linvc, p);
    finc = shoup_comp(fin, P);
  }
  uint32_t* out = coeffs + (size_t)pi * Nfull;
  const int KC = (plan.K + 31) / 32;
  for (int k = tid; k < M; k += T) {
    const int idx = S * k + r;
    if (idx >= Nfull) continue;
    uint32_t res = shoup(buf[sidx<true>(M - 1 + k)], fin, finc, p);
    if (c != 1u) res = mul_mod(res, pow_mod(cS, (uint64_t)k, P), P);
    if (crt_c)
      store_y(coeffs, po, pi, idx, KC, res);  // straight into the CRT GEMM's A layout (peer contexts' with po)
    else
      out[idx] = res;
  }
  (void)crt_cc;
}

void launch_interp(const InterpPlan& plan, const Prime* primes, const uint32_t* values, const uint32_t* cval,
                   uint32_t* coeffs, cudaStream_t st, const uint32_t* crt_c, const uint32_t* crt_cc,
                   const PeerOut* po) {
  if (plan.S > 1 && plan.Ab) {  // the tensor-core product with the plan's inverse Vandermonde
    launch_interp_mma(plan, primes, values, cval, coeffs, st, crt_c, po);
    return;
  }
  PeerOut pv = po ? *po : PeerOut{};
  if (!po) pv.G = 0;
  size_t smem = (size_t)plan.L * 4 * 3;  // data + 4 twiddle tables of L/2
  if (plan.S == 1) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_interp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_interp<<<plan.K, NTT_THREADS, smem, st>>>(plan, primes, values, cval, coeffs);
  } else {
    const size_t Lp = (plan.L + 3) & ~3, hp = (plan.L / 2 + 3) & ~3, Mp = (plan.N + 3) & ~3;
    const size_t Dp = ((size_t)padded_words(plan.L) + 3) & ~(size_t)3;
    // pointwise tables straight from L2 (measured: cfg4 28.3 -> 26.1 us, cfg2 13.7 -> 13.1 us, cfg5
    // 617 -> 544 us against staging them; CKB_INTERP_STAGE=1 stages them)
    static int force = -2;
    if (force == -2) {
      const char* e = getenv("CKB_INTERP_STAGE");
      force = e ? atoi(e) : -1;
    }
    const bool stage = force == 1;
    smem = (Dp + 4 * hp + (stage ? 4 * Lp + 2 * Mp : 0)) * 4;  // padded data, twiddles[, staged tables]
    const int want = plan.L / 8;
#define POLY_LAUNCH(TT)                                                                                       \
  if ((TT == 32 && want <= 32) || (TT == 64 && want == 64) || (TT == 128 && want == 128) ||                 \
      (TT == 256 && want >= 256)) {                                                                           \
    if (stage) {                                                                                              \
      if (smem > 48 * 1024)                                                                                   \
        cudaFuncSetAttribute(k_interp_poly<TT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      launch_pdl(k_interp_poly<TT, true>, dim3(plan.K * plan.S), dim3(TT), smem, st, plan, primes, values, cval,  \
                 coeffs, crt_c, crt_cc, pv);                                                                  \
    } else {                                                                                                  \
      if (smem > 48 * 1024)                                                                                   \
        cudaFuncSetAttribute(k_interp_poly<TT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
      launch_pdl(k_interp_poly<TT, false>, dim3(plan.K * plan.S), dim3(TT), smem, st, plan, primes, values, cval, \
                 coeffs, crt_c, crt_cc, pv);                                                                  \
    }                                                                                                         \
  }
    POLY_LAUNCH(32) POLY_LAUNCH(64) POLY_LAUNCH(128) POLY_LAUNCH(256)
#undef POLY_LAUNCH
  }
}

}  // namespace ckb

// Descartes sign-variation test of real-root isolation on the GPU.
//
// Reference: curvekit.upoly._variations_on (pkg/src/curvekit/upoly.py:338-346),
// the inner test of descartes_isolate (:358-408):
//     r = compose_linear(p, a, w, ld)      = 2^(n ld) p((a + w x) / 2^ld)   (:202-212)
//     c = taylor_shift(reversed(r), 1)     = (x + 1)^n r(1 / (x + 1))      (:193-199)
//     v = sign_variations(c)                                               (:215-224)
// Both steps are linear maps of the coefficients with binomial structure, so
// modulo a word prime each is one correlation:
//     r_k = w^k / k! * sum_i (p_i 2^(ld (n-i)) i!) (a^(i-k) / (i-k)!)
//     c_k = 1 / k!   * sum_i (i! r_{n-i})          (1 / (i-k)!)
// done with NTTs of length L >= 2n+1 (one CTA per prime, factorials, inverse
// factorials, twiddles and the transform of 1/j! cached per (primes, n)).  The
// exact integers c_k come back through the tensor-core CRT (their bound is
// planned on the host), and one CTA counts the sign variations.  The host keeps
// the reference's subdivision loop, so the isolating intervals are identical.
#include "ckb_kernels.cuh"
#include "ckb_ntt.cuh"

namespace ckb {

constexpr int DT = 256;  // threads per CTA

// inclusive multiplicative scan of buf[0..n) by one CTA (reverse: suffix)
__device__ void desc_scan_mul(uint32_t* buf, int n, const Prime& P, uint32_t* sh) {
  const int T = blockDim.x, tid = threadIdx.x;
  const int seg = (n + T - 1) / T;
  const int s0 = min(n, tid * seg), s1 = min(n, s0 + seg);
  uint32_t acc = 1u % P.p;
  for (int i = s0; i < s1; ++i) {
    acc = mul_mod(acc, buf[i], P);
    buf[i] = acc;
  }
  sh[tid] = acc;
  __syncthreads();
  for (int off = 1; off < T; off <<= 1) {
    const uint32_t v = (tid >= off) ? sh[tid - off] : 1u % P.p;
    __syncthreads();
    if (tid >= off) sh[tid] = mul_mod(sh[tid], v, P);
    __syncthreads();
  }
  const uint32_t pre = tid ? sh[tid - 1] : 1u % P.p;
  __syncthreads();
  if (tid)
    for (int i = s0; i < s1; ++i) buf[i] = mul_mod(buf[i], pre, P);
  __syncthreads();
}

// plan per prime: i!, 1/i! (i <= n), twiddles of length L, 1/L, and the DIF
// transform of the zero-padded 1/j! (the fixed operand of the second correlation)
__global__ void __launch_bounds__(DT) k_desc_plan(const Prime* __restrict__ primes, const uint32_t* __restrict__ gens,
                                                  DescPlan pl) {
  extern __shared__ uint32_t sm[];  // [L] work, [DT] scan scratch
  uint32_t* buf = sm;
  uint32_t* sh = sm + pl.L;
  const int pi = blockIdx.x, tid = threadIdx.x, T = blockDim.x, n = pl.n, L = pl.L, half = L >> 1;
  const Prime P = primes[pi];
  const uint32_t p = P.p;
  uint32_t* fact = pl.fact + (size_t)pi * (n + 1);
  uint32_t* ifact = pl.ifact + (size_t)pi * (n + 1);
  // factorials: prefix products of 1, 1, 2, ..., n
  for (int i = tid; i <= n; i += T) buf[i] = i ? (uint32_t)i % p : 1u % p;
  __syncthreads();
  desc_scan_mul(buf, n + 1, P, sh);
  for (int i = tid; i <= n; i += T) fact[i] = buf[i];
  __syncthreads();
  // inverse factorials: 1/n!, then suffix products of (n, n-1, ..., 1): 1/i! = (1/n!) * prod_{j>i} j
  const uint32_t inv_nf = inv_mod(buf[n], P);
  __syncthreads();
  for (int i = tid; i <= n; i += T) buf[i] = (i == 0) ? inv_nf : (uint32_t)(n - i + 1) % p;
  __syncthreads();
  desc_scan_mul(buf, n + 1, P, sh);  // buf[m] = (1/n!) * n (n-1) ... (n-m+1) = 1/(n-m)!
  for (int i = tid; i <= n; i += T) ifact[n - i] = buf[i];
  __syncthreads();
  // twiddles
  const uint32_t w = pow_mod(gens[pi] % p, (uint64_t)(p - 1) >> pl.logL, P);
  const uint32_t wi = inv_mod(w, P);
  const uint32_t wc = shoup_comp(w, P), wic = shoup_comp(wi, P);
  const size_t oH = (size_t)pi * half;
  const int seg = (half + T - 1) / T;
  const int s0 = min(half, tid * seg), s1 = min(half, s0 + seg);
  if (s0 < s1) {
    uint32_t a = pow_mod(w, s0, P), b = pow_mod(wi, s0, P);
    for (int j = s0; j < s1; ++j) {
      pl.W[oH + j] = a;
      pl.Wc[oH + j] = shoup_comp(a, P);
      pl.Wi[oH + j] = b;
      pl.Wic[oH + j] = shoup_comp(b, P);
      a = shoup(a, w, wc, p);
      b = shoup(b, wi, wic, p);
    }
  }
  if (tid == 0) pl.Linv[pi] = inv_mod((uint32_t)L % p, P);
  __syncthreads();
  // DIF of (1/0!, ..., 1/n!, 0, ...), twiddles read from global
  for (int i = tid; i < L; i += T) buf[i] = i <= n ? ifact[i] : 0u;
  __syncthreads();
  ntt_dif(buf, pl.logL, pl.W + oH, pl.Wc + oH, p);
  for (int i = tid; i < L; i += T) {
    const uint32_t v = red1(buf[i], p);
    pl.Vf[(size_t)pi * L + i] = v;
    pl.Vfc[(size_t)pi * L + i] = shoup_comp(v, P);
  }
}

void launch_desc_plan(const Prime* primes, const uint32_t* gens, const DescPlan& pl, cudaStream_t st) {
  const size_t smem = ((size_t)pl.L + DT) * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_desc_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_desc_plan<<<pl.K, DT, smem, st>>>(primes, gens, pl);
}

// c_k mod p for every prime and every interval b (grid.y): res [K][n+1]
// residues of p; aw [B][2][AL] limbs of a, w; lds [B]; out [K][B (n+1)]
// (interval b's coefficients at columns b (n+1) + k: one CRT lifts them all)
__global__ void __launch_bounds__(DT) k_desc_shift(const Prime* __restrict__ primes, DescPlan pl,
                                                   const uint32_t* __restrict__ res, const uint32_t* __restrict__ aws,
                                                   int AL, const int32_t* __restrict__ lds,
                                                   uint32_t* __restrict__ outs) {
  extern __shared__ uint32_t sm[];  // X [L], Y [L], twiddles 4 x [L/2]
  const int pi = blockIdx.x, tid = threadIdx.x, T = blockDim.x, n = pl.n, L = pl.L, half = L >> 1;
  const int b = blockIdx.y, B = gridDim.y;
  const uint32_t* aw = aws + (size_t)b * 2 * AL;
  const int ld = lds[b];
  const Prime P = primes[pi];
  const uint32_t p = P.p;
  uint32_t* X = sm;
  uint32_t* Y = sm + L;
  uint32_t *W = sm + 2 * L, *Wc = W + half, *Wi = Wc + half, *Wic = Wi + half;
  const size_t oH = (size_t)pi * half;
  for (int j = tid; j < half; j += T) {
    W[j] = pl.W[oH + j];
    Wc[j] = pl.Wc[oH + j];
    Wi[j] = pl.Wi[oH + j];
    Wic[j] = pl.Wic[oH + j];
  }
  const uint32_t* fact = pl.fact + (size_t)pi * (n + 1);
  const uint32_t* ifact = pl.ifact + (size_t)pi * (n + 1);
  const uint32_t* rp = res + (size_t)pi * (n + 1);
  // scalars: a, w mod p (two's-complement limbs), s = 2^ld mod p
  const uint32_t a = limbs_mod(aw, AL, P), wv = limbs_mod(aw + AL, AL, P);
  const uint32_t s = pow_mod(2u % p, (uint64_t)ld, P);
  // X'_m = u_{n-m} = p_{n-m} s^m (n-m)!   (m <= n);   Y_j = a^j / j!
  {
    uint32_t sm_ = pow_mod(s, (uint64_t)tid, P), aj = pow_mod(a, (uint64_t)tid, P);
    const uint32_t sT = pow_mod(s, (uint64_t)T, P), aT = pow_mod(a, (uint64_t)T, P);
    const uint32_t sTc = shoup_comp(sT, P), aTc = shoup_comp(aT, P);
    for (int m = tid; m < L; m += T) {
      if (m <= n) {
        X[m] = mul_mod(mul_mod(rp[n - m], sm_, P), fact[n - m], P);
        Y[m] = mul_mod(aj, ifact[m], P);
      } else {
        X[m] = 0u;
        Y[m] = 0u;
      }
      sm_ = shoup(sm_, sT, sTc, p);
      aj = shoup(aj, aT, aTc, p);
    }
  }
  __syncthreads();
  ntt_dif8<DT>(X, pl.logL, W, Wc, p);
  ntt_dif8<DT>(Y, pl.logL, W, Wc, p);
  for (int i = tid; i < L; i += T) X[i] = mul_mod(red1(X[i], p), red1(Y[i], p), P);
  __syncthreads();
  ntt_dit8<DT>(X, pl.logL, Wi, Wic, p);
  // t_k = X[n-k] / L;  r_k = w^k / k! t_k;  second operand X2'_m = (n-m)! r'_{n-m} = (n-m)! r_m
  const uint32_t linv = pl.Linv[pi];
  {
    uint32_t wk = pow_mod(wv, (uint64_t)tid, P);
    const uint32_t wT = pow_mod(wv, (uint64_t)T, P), wTc = shoup_comp(wT, P);
    for (int m = tid; m < L; m += T) {
      uint32_t v = 0u;
      if (m <= n) {
        const uint32_t t = mul_mod(red1(X[n - m], p), linv, P);  // t_m
        const uint32_t r = mul_mod(mul_mod(t, wk, P), ifact[m], P);
        v = mul_mod(r, fact[n - m], P);
      }
      Y[m] = v;  // Y is free after the pointwise product
      wk = shoup(wk, wT, wTc, p);
    }
  }
  __syncthreads();
  ntt_dif8<DT>(Y, pl.logL, W, Wc, p);
  const uint32_t* Vf = pl.Vf + (size_t)pi * L;
  const uint32_t* Vfc = pl.Vfc + (size_t)pi * L;
  for (int i = tid; i < L; i += T) Y[i] = shoup_lazy(Y[i], Vf[i], Vfc[i], p);
  __syncthreads();
  ntt_dit8<DT>(Y, pl.logL, Wi, Wic, p);
  // c_k = 1/k! * conv[n-k] / L
  uint32_t* out = outs + (size_t)pi * B * (n + 1) + (size_t)b * (n + 1);
  for (int k = tid; k <= n; k += T) out[k] = mul_mod(mul_mod(red1(Y[n - k], p), linv, P), ifact[k], P);
}

void launch_desc_shift(const Prime* primes, const DescPlan& pl, const uint32_t* res, const uint32_t* aw, int AL,
                       const int32_t* ld, int B, uint32_t* out, cudaStream_t st) {
  const size_t smem = (size_t)pl.L * 4 * 4;  // X, Y, 4 half-length twiddle tables
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_desc_shift, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_desc_shift<<<dim3(pl.K, B), DT, smem, st>>>(primes, pl, res, aw, AL, ld, out);
}

// sign variations of the lifted coefficients limbs [N][LW] (two's complement),
// upoly.sign_variations (:215-224): zeros are skipped, count sign changes; one
// CTA per interval (rows b N .. b N + N - 1)
__global__ void __launch_bounds__(1024) k_desc_signs(const uint32_t* __restrict__ limbs_all, int N, int LW,
                                                     int32_t* __restrict__ results) {
  const uint32_t* limbs = limbs_all + (size_t)blockIdx.x * N * LW;
  int32_t* result = results + blockIdx.x;
  __shared__ int cnt[1024];
  __shared__ int8_t sg[16384];
  const int tid = threadIdx.x, T = blockDim.x;
  for (int k = tid; k < N; k += T) {
    const uint32_t* c = limbs + (size_t)k * LW;
    int8_t s = 0;
    if ((int32_t)c[LW - 1] < 0) {
      s = -1;
    } else {
      for (int l = LW - 1; l >= 0; --l)
        if (c[l]) {
          s = 1;
          break;
        }
    }
    sg[k] = s;
  }
  __syncthreads();
  // each thread: a contiguous segment; count changes inside, remember first/last nonzero sign
  const int seg = (N + T - 1) / T;
  const int s0 = min(N, tid * seg), s1 = min(N, s0 + seg);
  int first = 0, last = 0, c = 0;
  for (int k = s0; k < s1; ++k) {
    const int s = sg[k];
    if (!s) continue;
    if (!first) first = s;
    if (last && s != last) ++c;
    last = s;
  }
  __shared__ int8_t fs[1024], ls[1024];
  fs[tid] = (int8_t)first;
  ls[tid] = (int8_t)last;
  cnt[tid] = c;
  __syncthreads();
  if (tid == 0) {
    int total = 0, prev = 0;
    for (int t = 0; t < T; ++t) {
      total += cnt[t];
      if (fs[t]) {
        if (prev && fs[t] != prev) ++total;
        prev = ls[t];
      }
    }
    *result = total;
  }
}

void launch_desc_signs(const uint32_t* limbs, int N, int LW, int B, int32_t* result, cudaStream_t st) {
  k_desc_signs<<<B, 1024, 0, st>>>(limbs, N, LW, result);
}

}  // namespace ckb

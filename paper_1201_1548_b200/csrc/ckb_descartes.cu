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
  CKB_SMEM_POISON(sm);
  const int pi = blockIdx.x, tid = threadIdx.x, T = blockDim.x, n = pl.n, L = pl.L, half = L >> 1;
  // direct mode (degrees beyond the NTT): the scans run in a global slice
  uint32_t* buf = pl.direct ? pl.Vf + (size_t)pi * (n + 1) : sm;
  uint32_t* sh = pl.direct ? sm : sm + pl.L;
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
  if (pl.direct) return;  // the direct correlations need only the factorials
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
  const size_t smem = ((pl.direct ? 0 : (size_t)pl.L) + DT) * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_desc_plan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_desc_plan<<<pl.K, DT, smem, st>>>(primes, gens, pl);
}

// c_k mod p for every prime and every interval b (grid.y): res [K][n+1]
// residues of p; aw [B][2][AL] limbs of a, w; lds [B]; out [K][B (n+1)]
// (interval b's coefficients at columns b (n+1) + k: one CRT lifts them all)
// TWS: the four twiddle tables staged in shared memory (L <= 2^13); at L = 2^14
// X and Y alone take 128 KB, so the twiddles are read from global memory (L2)
template <bool TWS>
__global__ void __launch_bounds__(DT) k_desc_shift(const Prime* __restrict__ primes, DescPlan pl,
                                                   const uint32_t* __restrict__ res, const uint32_t* __restrict__ aws,
                                                   int AL, const int32_t* __restrict__ lds,
                                                   uint32_t* __restrict__ outs) {
  extern __shared__ uint32_t sm[];  // X [L], Y [L], (TWS) twiddles 4 x [L/2]
  CKB_SMEM_POISON(sm);
  const int pi = blockIdx.x, tid = threadIdx.x, T = blockDim.x, n = pl.n, L = pl.L, half = L >> 1;
  const int b = blockIdx.y, B = gridDim.y;
  const uint32_t* aw = aws + (size_t)b * 2 * AL;
  const int ld = lds[b];
  const Prime P = primes[pi];
  const uint32_t p = P.p;
  uint32_t* X = sm;
  uint32_t* Y = sm + L;
  const size_t oH = (size_t)pi * half;
  const uint32_t *W = pl.W + oH, *Wc = pl.Wc + oH, *Wi = pl.Wi + oH, *Wic = pl.Wic + oH;
  if (TWS) {
    uint32_t *sW = sm + 2 * L, *sWc = sW + half, *sWi = sWc + half, *sWic = sWi + half;
    for (int j = tid; j < half; j += T) {
      sW[j] = W[j];
      sWc[j] = Wc[j];
      sWi[j] = Wi[j];
      sWic[j] = Wic[j];
    }
    W = sW, Wc = sWc, Wi = sWi, Wic = sWic;
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

// ---- direct mode: degrees whose NTT length exceeds the primes' 2^14 -------------
// the same two correlations as k_desc_shift, each output an O(n) dot product
// (thread per output, operands in a global slice per (prime, interval)):
//   conv1[i] = sum_{j <= i} X'_{i-j} Y_j,   conv2[i] = sum_{j <= i} Y2_{i-j} / j!
__device__ __forceinline__ uint32_t desc_dot(const uint32_t* __restrict__ u, const uint32_t* __restrict__ v, int i,
                                             const Prime& P) {
  // sum_{j=0}^{i} u[i-j] v[j]: products < 2^60 (p < 2^30), 16 of them summed in 64 bits
  // before one reduction to [0, p) by REDC (result carries R^-1, the caller compensates)
  const uint32_t p = P.p;
  uint32_t acc = 0u;
  int j = 0;
  while (j <= i) {
    const int e = min(i + 1, j + 15);
    uint64_t t = 0;
    for (; j < e; ++j) t += (uint64_t)u[i - j] * v[j];
    t = t % ((uint64_t)p << 32);  // keep t < p 2^32 for the REDC (16 * 2^60 < 2^64)
    acc = add_mod(acc, redc(t, P), p);
  }
  return acc;
}

__global__ void __launch_bounds__(DT) k_desc_direct_prep(const Prime* __restrict__ primes, DescPlan pl,
                                                         const uint32_t* __restrict__ res,
                                                         const uint32_t* __restrict__ aws, int AL,
                                                         const int32_t* __restrict__ lds, uint32_t* __restrict__ scr) {
  const int pi = blockIdx.y, b = blockIdx.z, B = gridDim.z, n = pl.n;
  const int m = blockIdx.x * DT + threadIdx.x;
  if (m > n) return;
  const Prime P = primes[pi];
  const uint32_t* aw = aws + (size_t)b * 2 * AL;
  const uint32_t a = limbs_mod(aw, AL, P);
  const uint32_t s = pow_mod(2u % P.p, (uint64_t)lds[b], P);
  const uint32_t* fact = pl.fact + (size_t)pi * (n + 1);
  const uint32_t* ifact = pl.ifact + (size_t)pi * (n + 1);
  uint32_t* X = scr + ((size_t)pi * B + b) * 3 * (n + 1);
  uint32_t* Y = X + (n + 1);
  X[m] = mul_mod(mul_mod(res[(size_t)pi * (n + 1) + n - m], pow_mod(s, (uint64_t)m, P), P), fact[n - m], P);
  Y[m] = mul_mod(pow_mod(a, (uint64_t)m, P), ifact[m], P);
}

// conv1 -> Y2 (a third region of the slice: conv1 reads all of X and Y)
__global__ void __launch_bounds__(DT) k_desc_direct_conv1(const Prime* __restrict__ primes, DescPlan pl,
                                                          const uint32_t* __restrict__ aws, int AL,
                                                          uint32_t* __restrict__ scr) {
  const int pi = blockIdx.y, b = blockIdx.z, B = gridDim.z, n = pl.n;
  const int m = blockIdx.x * DT + threadIdx.x;
  if (m > n) return;
  const Prime P = primes[pi];
  const uint32_t wv = limbs_mod(aws + (size_t)b * 2 * AL + AL, AL, P);
  uint32_t* X = scr + ((size_t)pi * B + b) * 3 * (n + 1);
  const uint32_t R1 = redc((uint64_t)P.r2, P);  // 2^32 mod p: undoes desc_dot's R^-1
  const uint32_t t = mul_mod(desc_dot(X, X + (n + 1), n - m, P), R1, P);
  // r_m = t_m w^m / m!;  Y2_m = (n-m)! r_m
  const uint32_t r = mul_mod(mul_mod(t, pow_mod(wv, (uint64_t)m, P), P), pl.ifact[(size_t)pi * (n + 1) + m], P);
  X[2 * (n + 1) + m] = mul_mod(r, pl.fact[(size_t)pi * (n + 1) + n - m], P);
}

__global__ void __launch_bounds__(DT) k_desc_direct_conv2(const Prime* __restrict__ primes, DescPlan pl,
                                                          const uint32_t* __restrict__ scr, uint32_t* __restrict__ outs) {
  const int pi = blockIdx.y, b = blockIdx.z, B = gridDim.z, n = pl.n;
  const int k = blockIdx.x * DT + threadIdx.x;
  if (k > n) return;
  const Prime P = primes[pi];
  const uint32_t* ifact = pl.ifact + (size_t)pi * (n + 1);
  const uint32_t* Y2 = scr + ((size_t)pi * B + b) * 3 * (n + 1) + 2 * (n + 1);
  const uint32_t v = mul_mod(desc_dot(Y2, ifact, n - k, P), redc((uint64_t)P.r2, P), P);
  outs[(size_t)pi * B * (n + 1) + (size_t)b * (n + 1) + k] = mul_mod(v, ifact[k], P);  // c_k = conv2[n-k] / k!
}

void launch_desc_shift(const Prime* primes, const DescPlan& pl, const uint32_t* res, const uint32_t* aw, int AL,
                       const int32_t* ld, int B, uint32_t* out, uint32_t* scratch, cudaStream_t st) {
  if (pl.direct) {
    const dim3 grid((unsigned)((pl.n + DT) / DT), (unsigned)pl.K, (unsigned)B);
    k_desc_direct_prep<<<grid, DT, 0, st>>>(primes, pl, res, aw, AL, ld, scratch);
    k_desc_direct_conv1<<<grid, DT, 0, st>>>(primes, pl, aw, AL, scratch);
    k_desc_direct_conv2<<<grid, DT, 0, st>>>(primes, pl, scratch, out);
    return;
  }
  const size_t full = (size_t)pl.L * 4 * 4;  // X, Y, 4 half-length twiddle tables
  if (full <= 200 * 1024) {
    if (full > 48 * 1024) cudaFuncSetAttribute(k_desc_shift<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)full);
    k_desc_shift<true><<<dim3(pl.K, B), DT, full, st>>>(primes, pl, res, aw, AL, ld, out);
  } else {
    const size_t smem = (size_t)pl.L * 2 * 4;  // X, Y (128 KB at L = 2^14)
    cudaError_t e = cudaFuncSetAttribute(k_desc_shift<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return;  // surfaces through cudaGetLastError in the caller
    k_desc_shift<false><<<dim3(pl.K, B), DT, smem, st>>>(primes, pl, res, aw, AL, ld, out);
  }
}

// sign variations of the lifted coefficients limbs [N][LW] (two's complement),
// upoly.sign_variations (:215-224): zeros are skipped, count sign changes; one
// CTA per interval (rows b N .. b N + N - 1)
__global__ void __launch_bounds__(1024) k_desc_signs(const uint32_t* __restrict__ limbs_all, int N, int LW,
                                                     int32_t* __restrict__ results) {
  const uint32_t* limbs = limbs_all + (size_t)blockIdx.x * N * LW;
  int32_t* result = results + blockIdx.x;
  __shared__ int cnt[1024];
  const int tid = threadIdx.x, T = blockDim.x;
  // each thread: a contiguous segment (signs read straight from the limbs, any N);
  // count changes inside, remember the first/last nonzero sign
  const int seg = (N + T - 1) / T;
  const int s0 = min(N, tid * seg), s1 = min(N, s0 + seg);
  int first = 0, last = 0, c = 0;
  for (int k = s0; k < s1; ++k) {
    const uint32_t* w = limbs + (size_t)k * LW;
    int s = 0;
    if ((int32_t)w[LW - 1] < 0) {
      s = -1;
    } else {
      for (int l = LW - 1; l >= 0; --l)
        if (w[l]) {
          s = 1;
          break;
        }
    }
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

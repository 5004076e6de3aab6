// K5: Chinese remaindering of every coefficient and the symmetric lift to
// two's-complement 32-bit limbs.
//
// Reference: curvekit.modpoly._CrtAccumulator.add / symmetric
// (pkg/src/curvekit/modpoly.py:278-300) and crt_reconstruct (:264-275):
// incremental Garner, then x - M if 2x > M.  The result is the unique
// representative of the residues in (-M/2, M/2]; this computes the same
// integer by the *explicit* CRT, which has no sequential recurrence:
//     y_i = r_i * (M/p_i)^-1 mod p_i                     (k_crt_ymul, or fused
//                                                          into the interpolation)
//     X   = sum_i y_i * (M/p_i)                           (k_crt_mma: an N x K x LW
//                                                          product on the tensor cores)
//     q   = round(sum_i y_i / p_i)                       (k_crt_carry, FP64)
//     x   = X - q M                                      (k_crt_carry: signed carries)
// X/M = q + x/M exactly; the planner guarantees M > 4 * bound, so |x/M| < 1/4
// and the FP64 sum (error < K^2 2^-52) always rounds to the right q.  Callers
// without that margin (crt_reconstruct on arbitrary residues) get an exact
// fold when the sum lands near a half-integer.
#include "ckb_kernels.cuh"

namespace ckb {

// ---------------------------------------------------------------------------
// CRT tables per prime set (built once, cached): thread i divides M = prod p
// (LW limbs) by p_i — 64/32-bit quotient digits from a 64-bit reciprocal, at
// most two corrections — writing M/p_i, and accumulates (M/p_i) mod p_i from
// the quotient digits (Horner in 2^32) for c_i = (M/p_i)^-1 mod p_i.  (The
// host loop it replaces spent K LW hardware divisions plus K^2 modular
// products: 10-60 ms per table at the Descartes test's 500-1,500 primes.)
// ---------------------------------------------------------------------------
__global__ void k_crt_tables(const uint32_t* __restrict__ primes, int K, const uint32_t* __restrict__ M, int LW,
                             uint32_t* __restrict__ Mi, uint32_t* __restrict__ c, uint32_t* __restrict__ cc,
                             uint32_t* __restrict__ bad) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K) return;
  const uint32_t p = primes[i];
  const Prime P = make_prime(p);
  const uint64_t m = ~0ull / p;  // floor((2^64 - 1) / p)
  const uint32_t R1 = redc(P.r2, P), R1c = shoup_comp(R1, P), onec = shoup_comp(1u % p, P);
  uint64_t rem = 0;
  uint32_t mod = 0;
  for (int l = LW - 1; l >= 0; --l) {
    const uint64_t cur = (rem << 32) | M[l];  // < p 2^32: the quotient digit fits 32 bits
    uint64_t q = __umul64hi(cur, m);
    uint64_t r = cur - q * p;
    while (r >= p) {
      r -= p;
      ++q;
    }
    Mi[(size_t)i * LW + l] = (uint32_t)q;
    rem = r;
    mod = add_mod(shoup(mod, R1, R1c, p), mod_word((uint32_t)q, onec, p), p);
  }
  if (mod == 0u) {  // p_i divides M / p_i: the primes are not pairwise distinct
    atomicOr(bad, 1u);
    return;
  }
  const uint32_t inv = inv_mod(mod, P);
  c[i] = inv;
  cc[i] = shoup_comp(inv, P);
}

void launch_crt_tables(const uint32_t* primes, int K, const uint32_t* M, int LW, uint32_t* Mi, uint32_t* c,
                       uint32_t* cc, uint32_t* bad, cudaStream_t st) {
  k_crt_tables<<<(K + 127) / 128, 128, 0, st>>>(primes, K, M, LW, Mi, c, cc, bad);
}

// ---------------------------------------------------------------------------
// y[i][k] = r[i][k] (M/p_i)^-1 mod p_i (standalone API path; the pipeline's
// interpolation kernel writes y directly)
// ---------------------------------------------------------------------------
__global__ void k_crt_ymul(CrtTables T, const uint32_t* __restrict__ r, int N, uint32_t* __restrict__ y) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
  // pdl_launch();  (implicit at exit: measured better)
  pdl_wait();
  if (k >= N) return;
  const uint32_t p = T.p[i];
  y[crt_a_word(i, k, (T.K + 31) / 32)] = red1(shoup_lazy(r[(size_t)i * N + k], T.c[i], T.cc[i], p), p);
}

// ---------------------------------------------------------------------------
// carry: one warp per coefficient, 8 limbs per lane per 256-limb chunk.
// Each lane carries through its 8 limbs with carry-in 0, then the true
// carry-ins run along the lanes (32 cheap sequential steps: adding a carry-in
// below 2^63 to a segment changes its carry-out by -1, 0 or +1, decided by the
// segment's low 64 bits and whether its upper limbs are all ones / all zeros),
// then each lane applies its carry-in.
// ---------------------------------------------------------------------------
struct I128 {
  long long hi;
  unsigned long long lo;
};
__device__ __forceinline__ I128 add128(I128 a, long long bhi, unsigned long long blo) {
  I128 r;
  r.lo = a.lo + blo;
  r.hi = a.hi + bhi + (long long)(r.lo < a.lo);
  return r;
}

// S: the tensor-core limb sums (u64 [N][LWp], ckb_crt_mma.cu); y in the A layout.
// out may be page-locked host memory (mapped): the limbs then travel to the host
// as the kernel writes them, each warp store one contiguous 128-byte run.
// status_src -> status_dst (optional): the pipeline's status word, final once
// the grids this one waits on have completed.
__global__ void __launch_bounds__(128) k_crt_carry(CrtTables T, int N, const unsigned long long* __restrict__ S,
                                                   const uint32_t* __restrict__ y, int LWp,
                                                   uint32_t* __restrict__ out, const uint32_t* status_src,
                                                   uint32_t* status_dst) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.x * 4 + warp;
  __shared__ uint32_t stage[4][256];
  uint32_t* so = stage[warp];
  // pdl_launch();  (implicit at exit: measured better)
  pdl_wait();
  if (status_dst && blockIdx.x == 0 && threadIdx.x == 0) *status_dst = *status_src;
  if (k >= N) return;
  const unsigned FULL = 0xffffffffu;
  const int LW = T.LW;
  const unsigned long long* Sk = S + (size_t)k * LWp;
  // the first chunk's limb sums and modulus limbs are loaded before q is known
  // (their latency overlaps the q reduction)
  unsigned long long pre_s[8];
  uint32_t pre_m[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int l = lane * 8 + j;
    pre_s[j] = l < LW ? Sk[l] : 0ull;
    pre_m[j] = l < LW ? T.Ml[l] : 0u;
  }
  // q = round(sum_i y_i / p_i); lane 0's value is broadcast so every lane agrees bitwise
  const int KC = (T.K + 31) / 32;
  double qs = 0.0;
  for (int i = lane; i < T.K; i += 32) qs = fma((double)y[crt_a_word(i, k, KC)], T.pinvd[i], qs);
#pragma unroll
  for (int o = 16; o; o >>= 1) qs += __shfl_xor_sync(FULL, qs, o);
  qs = __shfl_sync(FULL, qs, 0);
  const unsigned long long q = (unsigned long long)llrint(qs);
  const bool ambk = fabs((qs - floor(qs)) - 0.5) < 1e-3;  // near a half-integer: exact fold needed
  uint32_t* ok = out + (size_t)k * LW;
  long long cin_hi = 0;            // carry into the chunk (signed 128-bit, fits in hi:lo)
  unsigned long long cin_lo = 0;
  for (int c0 = 0; c0 < LW; c0 += 256) {
    const int l0 = c0 + lane * 8;
    uint32_t o[8];
    I128 c = {0, 0};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int l = l0 + j;
      unsigned long long s_lo = 0, qm = 0;
      long long s_hi = 0;
      if (l < LW) {
        s_lo = c0 == 0 ? pre_s[j] : Sk[l];
        qm = q * (unsigned long long)(c0 == 0 ? pre_m[j] : T.Ml[l]);
      }
      I128 t;
      t.lo = s_lo - qm;
      t.hi = s_hi - (long long)(s_lo < qm);
      t = add128(t, c.hi, c.lo);
      o[j] = (uint32_t)t.lo;
      c.lo = (t.lo >> 32) | ((unsigned long long)t.hi << 32);  // t >> 32
      c.hi = t.hi >> 32;
    }
    // segment summary for the carry-in transfer
    const unsigned long long seg_lo = (unsigned long long)o[0] | ((unsigned long long)o[1] << 32);
    bool ones = true, zeros = true;
#pragma unroll
    for (int j = 2; j < 8; ++j) {
      ones &= (o[j] == 0xffffffffu);
      zeros &= (o[j] == 0u);
    }
    // carry-ins along the lanes: lane s's carry-out is c + delta_s(cin_s), delta in
    // {-1, 0, 1} (nonzero only when the carry-in overflows the low 64 bits AND
    // limbs 2..7 are all ones / all zeros).  Fixed-point iteration from lane 0's
    // known carry-in: after t rounds lanes 0..t-1 are exact, and a round in
    // which nothing changes is exact everywhere (the chain is anchored at lane
    // 0); typically 1-3 rounds instead of 32 sequential steps.
    long long my_cin = 0;
    long long co = (long long)c.lo;  // this lane's carry-out, current estimate
    for (int it = 0; it < 33; ++it) {
      const long long up = __shfl_up_sync(FULL, co, 1);
      const long long cin = (lane == 0) ? (long long)cin_lo : up;
      const unsigned long long u = seg_lo + (unsigned long long)cin;
      const long long kappa = (cin >= 0) ? (long long)(u < seg_lo) : -(long long)(u > seg_lo);
      long long delta = 0;
      if (kappa == 1 && ones) delta = 1;
      if (kappa == -1 && zeros) delta = -1;
      const long long nco = (long long)c.lo + delta;
      const bool changed = nco != co;
      co = nco;
      my_cin = cin;
      if (!__any_sync(FULL, changed)) break;
    }
    const long long run = __shfl_sync(FULL, co, 31);  // carry out of lane 31 = into the next chunk
    // apply the carry-in
    {
      const unsigned long long u = seg_lo + (unsigned long long)my_cin;
      long long kappa = (my_cin >= 0) ? (long long)(u < seg_lo) : -(long long)(u > seg_lo);
      o[0] = (uint32_t)u;
      o[1] = (uint32_t)(u >> 32);
#pragma unroll
      for (int j = 2; j < 8; ++j) {
        const long long v = (long long)o[j] + kappa;
        o[j] = (uint32_t)v;
        kappa = v >> 32;
      }
    }
    // through shared memory: lane-contiguous stores instead of a stride of 8 limbs
#pragma unroll
    for (int j = 0; j < 8; ++j) so[lane * 8 + j] = o[j];
    __syncwarp();
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (c0 + j * 32 + lane < LW) ok[c0 + j * 32 + lane] = so[j * 32 + lane];
    __syncwarp();
    cin_lo = (unsigned long long)run;  // carry out of lane 31 = into the next chunk
  }
  // Exactness guard (never taken when M > 4 bound): fold x into
  // [-floor(M/2), floor(M/2)] if q came from a sum near a half-integer.
  if (ambk) {
    __syncwarp();
    __threadfence_block();
    if (lane == 0) {
      long long br = 0;  // d = x - H - 1 >= 0  <=>  x > H
      for (int l = 0; l < LW; ++l) {
        const long long v = (long long)ok[l] - (long long)T.Mh[l] - (l == 0 ? 1 : 0) + br;
        br = v >> 32;
      }
      const bool x_top_neg = (int32_t)ok[LW - 1] < 0;
      const bool gt = !x_top_neg && br >= 0;
      long long cr = 0;  // e = x + H < 0  <=>  x < -H
      for (int l = 0; l < LW; ++l) {
        const long long v = (long long)ok[l] + (long long)T.Mh[l] + cr;
        cr = v >> 32;
      }
      const bool lt = x_top_neg && cr == 0;
      if (gt || lt) {
        long long cc = 0;
        for (int l = 0; l < LW; ++l) {
          const long long v = (long long)ok[l] + (gt ? -(long long)T.Ml[l] : (long long)T.Ml[l]) + cc;
          ok[l] = (uint32_t)v;
          cc = v >> 32;
        }
      }
    }
  }
}

int launch_crt(const CrtTables& t, const uint32_t* coeffs, int N, uint32_t* out, uint32_t* scratch,
               cudaStream_t st, bool input_is_y, const uint32_t* status_src, uint32_t* status_dst) {
  // scratch (cudaMalloc-aligned): S [N][LWp] u64 | y (A layout)
  const int LWp = (t.LW + 31) / 32 * 32;
  unsigned long long* S = reinterpret_cast<unsigned long long*>(scratch);
  const uint32_t* y = coeffs;
  if (!input_is_y) {
    uint32_t* yb = scratch + (size_t)2 * N * LWp;
    launch_pdl(k_crt_ymul, dim3((N + 255) / 256, t.K), dim3(256), 0, st, t, coeffs, N, yb);
    y = yb;
  }
  launch_crt_mma(t, y, N, S, st);
  launch_pdl(k_crt_carry, dim3((N + 3) / 4), dim3(128), 0, st, t, N, S, y, LWp, out, status_src, status_dst);
  return input_is_y ? 2 : 3;
}

size_t crt_scratch_words(int K, int N, int LW) {
  const size_t LWp = (size_t)(LW + 31) / 32 * 32;
  return 2 * LWp * N + crt_a_words(K, N) + 32;
}

}  // namespace ckb

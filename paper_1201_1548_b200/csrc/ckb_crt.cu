// K5: Chinese remaindering of every coefficient and the symmetric lift to
// two's-complement 32-bit limbs.
//
// Reference: curvekit.modpoly._CrtAccumulator.add / symmetric
// (pkg/src/curvekit/modpoly.py:278-300) and crt_reconstruct (:264-275):
// incremental Garner, then x - M if 2x > M.  The result is the unique
// representative of the residues in (-M/2, M/2]; this computes the same
// integer by the *explicit* CRT, which has no sequential recurrence:
//     y_i = r_i * (M/p_i)^-1 mod p_i                     (k_crt_prep)
//     q   = round(sum_i y_i / p_i)                       (k_crt_prep, FP64)
//     X   = sum_i y_i * (M/p_i)                           (k_crt_gemm: an N x K x LW
//                                                          integer product, 96-bit sums)
//     x   = X - q M                                      (k_crt_carry: signed carries)
// X/M = q + x/M exactly; the planner guarantees M > 4 * bound, so |x/M| < 1/4
// and the FP64 sum (error < K^2 2^-52) always rounds to the right q.  Callers
// without that margin (crt_reconstruct on arbitrary residues) get an exact
// fold when the sum lands near a half-integer.
#include "ckb_kernels.cuh"

namespace ckb {

constexpr int TN = 64;   // coefficients per CTA tile
constexpr int TL = 32;   // limbs per CTA tile
constexpr int TI = 32;   // primes per k-step
constexpr int CRT_THREADS = 256;

// ---------------------------------------------------------------------------
// y[i][k] = r[i][k] (M/p_i)^-1 mod p_i (standalone API path; the pipeline's
// interpolation kernel writes y directly)
// ---------------------------------------------------------------------------
__global__ void k_crt_ymul(CrtTables T, const uint32_t* __restrict__ r, int N, uint32_t* __restrict__ y) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y;
  if (k >= N) return;
  const uint32_t p = T.p[i];
  y[(size_t)i * N + k] = red1(shoup_lazy(r[(size_t)i * N + k], T.c[i], T.cc[i], p), p);
}

// ---------------------------------------------------------------------------
// gemm: S[k][l] = sum_i y_i(k) * (M/p_i)[l] as 96-bit (lo64, hi32) column sums,
// coefficient-major S[k][l][3].  Thread micro-tile: 2 coefficients x 4 limbs;
// products of 30-bit y and 32-bit limbs accumulate 4 at a time in 64 bits.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(CRT_THREADS) k_crt_gemm(CrtTables T, const uint32_t* __restrict__ y, int N,
                                                          uint32_t* __restrict__ S, int64_t* __restrict__ qk,
                                                          uint32_t* __restrict__ amb) {
  __shared__ uint32_t sy[2][TI][TN];
  __shared__ uint32_t sm[2][TI][TL];
  const int K = T.K, LW = T.LW;
  const int k0 = blockIdx.x * TN, l0 = blockIdx.y * TL;
  const int tid = threadIdx.x;
  const int tk = (tid % 32) * 2;        // coefficient offset (0..62)
  const int tl = (tid / 32) * 4;        // limb offset (0..28)
  uint64_t lo[2][4] = {};
  uint32_t hi[2][4] = {};
  // asynchronous global -> shared copies (LDGSTS; src-size 0 zero-fills out
  // of range), so the next tile streams in while this one is multiplied
  auto cp4 = [](uint32_t* dst, const uint32_t* src, bool ok) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(sa), "l"(src), "r"(ok ? 4 : 0));
  };
  auto stage = [&](int buf, int i0) {
    for (int e = tid; e < TI * TN; e += CRT_THREADS) {
      const int ii = e / TN, kk = e % TN;
      const int i = i0 + ii, k = k0 + kk;
      const bool ok = i < K && k < N;
      cp4(&sy[buf][ii][kk], ok ? y + (size_t)i * N + k : y, ok);
    }
    for (int e = tid; e < TI * TL; e += CRT_THREADS) {
      const int ii = e / TL, ll = e % TL;
      const int i = i0 + ii, l = l0 + ll;
      const bool ok = i < K && l < LW;
      cp4(&sm[buf][ii][ll], ok ? T.Mi + (size_t)i * LW + l : T.Mi, ok);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  stage(0, 0);
  asm volatile("cp.async.wait_group 0;\n" ::);
  __syncthreads();
  int buf = 0;
  const bool qrow = blockIdx.y == 0 && tid < TN;  // these threads also form q = round(sum y_i / p_i)
  double qs = 0.0;
  for (int i0 = 0; i0 < K; i0 += TI) {
    if (i0 + TI < K) stage(buf ^ 1, i0 + TI);  // prefetch the next tile while computing this one
    if (qrow)
      for (int ii = 0; ii < TI && i0 + ii < K; ++ii) qs = fma((double)sy[buf][ii][tid], T.pinvd[i0 + ii], qs);
#pragma unroll
    for (int i4 = 0; i4 < TI; i4 += 2) {
      uint64_t acc[2][4] = {};  // 2 products of y < 2^31 and a 32-bit limb stay below 2^64
#pragma unroll
      for (int ii = i4; ii < i4 + 2; ++ii) {
        const uint2 yv = *reinterpret_cast<const uint2*>(&sy[buf][ii][tk]);
        const uint4 mv = *reinterpret_cast<const uint4*>(&sm[buf][ii][tl]);
        const uint32_t ys[2] = {yv.x, yv.y};
        const uint32_t ms[4] = {mv.x, mv.y, mv.z, mv.w};
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] += (uint64_t)ys[a] * ms[b];  // 4 products < 2^64
      }
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const uint64_t s = lo[a][b] + acc[a][b];
          hi[a][b] += (s < acc[a][b]);
          lo[a][b] = s;
        }
    }
    asm volatile("cp.async.wait_group 0;\n" ::);
    __syncthreads();
    buf ^= 1;
  }
  if (qrow && k0 + tid < N) {
    qk[k0 + tid] = llrint(qs);
    amb[k0 + tid] = fabs((qs - floor(qs)) - 0.5) < 1e-3;  // near a half-integer: exact fold needed
  }
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int k = k0 + tk + a;
    if (k >= N) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int l = l0 + tl + b;
      if (l < LW) {
        uint32_t* o = S + ((size_t)k * LW + l) * 3;
        o[0] = (uint32_t)lo[a][b];
        o[1] = (uint32_t)(lo[a][b] >> 32);
        o[2] = hi[a][b];
      }
    }
  }
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

__global__ void __launch_bounds__(128) k_crt_carry(CrtTables T, int N, const uint32_t* __restrict__ S,
                                                   const int64_t* __restrict__ qk, const uint32_t* __restrict__ amb,
                                                   uint32_t* __restrict__ out) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = blockIdx.x * 4 + warp;
  if (k >= N) return;
  const unsigned FULL = 0xffffffffu;
  const int LW = T.LW;
  const unsigned long long q = (unsigned long long)qk[k];
  const uint32_t* Sk = S + (size_t)k * LW * 3;
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
        s_lo = (unsigned long long)Sk[3 * l] | ((unsigned long long)Sk[3 * l + 1] << 32);
        s_hi = Sk[3 * l + 2];
        qm = q * (unsigned long long)T.Ml[l];
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
    // sequential carry-ins along the lanes (c is small: |c| < 2^63)
    long long my_cin = 0;  // carry into this lane's segment (fits in 64 bits)
    long long run = (long long)cin_lo;  // carry entering lane 0 (|.| < 2^63)
    (void)cin_hi;
    for (int s = 0; s < 32; ++s) {
      if (lane == s) {
        my_cin = run;
        // value added to limbs 0..1: seg_lo + run (signed); carry kappa into limb 2
        const unsigned long long u = seg_lo + (unsigned long long)run;
        long long kappa = (run >= 0) ? (long long)(u < seg_lo) : -(long long)(u > seg_lo);
        long long delta = 0;
        if (kappa == 1 && ones) delta = 1;
        if (kappa == -1 && zeros) delta = -1;
        run = (long long)c.lo + delta;  // this lane's carry-out
      }
      run = __shfl_sync(FULL, run, s);
    }
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
#pragma unroll
    for (int j = 0; j < 8; ++j)
      if (l0 + j < LW) ok[l0 + j] = o[j];
    cin_lo = (unsigned long long)run;  // carry out of lane 31 = into the next chunk
  }
  // Exactness guard (never taken when M > 4 bound): fold x into
  // [-floor(M/2), floor(M/2)] if q came from a sum near a half-integer.
  if (amb[k]) {
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

void launch_crt(const CrtTables& t, const uint32_t* coeffs, int N, uint32_t* out, uint32_t* scratch,
                cudaStream_t st, bool input_is_y) {
  // scratch (cudaMalloc-aligned): q [N] (int64) | amb [N] | S [N][LW][3] | y [K][N]
  int64_t* qk = reinterpret_cast<int64_t*>(scratch);
  uint32_t* amb = reinterpret_cast<uint32_t*>(qk + N);
  uint32_t* S = amb + N;
  const uint32_t* y = coeffs;
  if (!input_is_y) {
    uint32_t* yb = S + (size_t)3 * N * t.LW;
    k_crt_ymul<<<dim3((N + 255) / 256, t.K), 256, 0, st>>>(t, coeffs, N, yb);
    y = yb;
  }
  dim3 g1((N + TN - 1) / TN, (t.LW + TL - 1) / TL);
  k_crt_gemm<<<g1, CRT_THREADS, 0, st>>>(t, y, N, S, qk, amb);
  k_crt_carry<<<(N + 3) / 4, 128, 0, st>>>(t, N, S, qk, amb, out);
}

size_t crt_scratch_words(int K, int N, int LW) {
  return (size_t)3 * N * LW + (size_t)K * N + 2 + (size_t)2 * N + N + 16;
}

}  // namespace ckb

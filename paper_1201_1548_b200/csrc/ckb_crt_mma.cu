// The tensor-core stages (tcgen05 kind::i8, s32 accumulators in TMEM):
//   * K5, the explicit-CRT product X = sum_i y_i (M/p_i) as an unsigned 8-bit GEMM;
//   * K4, the interpolation as a product with the plan's inverse Vandermonde
//     (k_interp_mma, second half of this file).
//
// Reference: _CrtAccumulator / crt_reconstruct (pkg/src/curvekit/modpoly.py:264-300);
// see ckb_crt.cu for the explicit-CRT identity this evaluates.
//
// Split both factors into bytes: y_i = sum_a y_{i,a} 2^{8a},  M/p_i = sum_s m_{i,s} 2^{8s}.
// Then X = sum_t D[t] 2^{8t} with
//     D[k][t] = sum_{i,a} y_{i,a}(k) * m_{i, t-a}
// an  N x (4K) x (4 LW)  GEMM whose B operand B[t][(i,a)] = m_{i,t-a} is a
// shifted (Toeplitz) copy of the M/p_i bytes, fixed per prime set and built
// once (k_crt_btable).  Every D < 4K * 255^2 < 2^31, so s32 accumulation is
// exact for K < 8250 primes.  The epilogue folds four byte columns into one
// 64-bit limb sum S_l = sum_{j<4} D[4l+j] 2^{8j} (< 2^54); k_crt_carry then
// subtracts q M and propagates the carries.
//
// Tile: 128 coefficients x 128 byte positions, K streamed in 128-byte chunks
// (32 primes).  Both operands sit in global memory already in the canonical
// no-swizzle K-major layout (A written so by the interpolation kernel, see
// crt_a_word; B pre-tiled), so each chunk is two 16 KB bulk (TMA-engine)
// copies into a 4-deep ring.  One thread issues four 128x128x32 MMAs per chunk;
// tcgen05.commit releases the stage.  Padding rows / primes of A hold
// arbitrary words: the matching B rows are zero and padded D rows are dropped.
#include "ckb_kernels.cuh"

namespace ckb {

namespace {
constexpr int BM = 128;           // coefficients per tile (TMEM lanes)
constexpr int BN = 128;           // byte positions per tile (TMEM columns)
constexpr int BK = 128;           // K bytes per chunk = 32 primes
constexpr int CHUNK = BM * BK;    // 16 KB per operand chunk
constexpr int STAGES = 4;
constexpr int THREADS = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred P;\n mbarrier.try_wait.parity.shared::cta.b64 P, [%1], %2;\n selp.u32 %0, 1, 0, P;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
// no-swizzle K-major matrix descriptor: core matrices of 8 rows x 16 bytes,
// LBO = 128 B between core matrices along K, SBO = 1024 B between 8-row groups
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t addr) {
  const uint64_t lo = ((addr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16);
  const uint64_t hi = (uint64_t)(1024 >> 4) | (1ull << 14);  // version 1 (Blackwell), layout SWIZZLE_NONE
  return lo | (hi << 32);
}
// instruction descriptor: kind::i8, A/B unsigned 8-bit, K-major, D s32, M=128, N=128
constexpr uint32_t IDESC = (2u << 4) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar) : "memory");
}

#define CKB_LD32(r, addr)                                                                                          \
  asm volatile(                                                                                                    \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18," \
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"                                              \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),            \
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),      \
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),    \
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])     \
      : "r"(addr))
}  // namespace

// Byte table B, pre-tiled: [NT][KC][CHUNK] with element (row n, K byte kb) of
// tile (nt, kc) at (n/8)*1024 + (kb/16)*128 + (n%8)*16 + kb%16 and value
// m_{i, t-a} for t = 128 nt + n, i = 32 kc + kb/4, a = kb%4 (0 outside).
__global__ void k_crt_btable(int K, int LW, const uint32_t* __restrict__ Mi, int KC, uint32_t* __restrict__ Bt,
                             size_t words) {
  const size_t w = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= words) return;
  const size_t tile = w / (CHUNK / 4);
  const int nt = (int)(tile / KC), kc = (int)(tile % KC);
  const int r = (int)(w % (CHUNK / 4));
  const int n8 = r / 256, kc16 = (r % 256) / 32, n7 = (r % 32) / 4, wq = r % 4;
  const int n = n8 * 8 + n7, kb = kc16 * 16 + wq * 4;
  const int i = kc * 32 + kb / 4, t = nt * BN + n;
  uint32_t v = 0;
  if (i < K) {
    for (int a = 0; a < 4; ++a) {
      const int s = t - a;
      if (s >= 0 && s < 4 * LW) v |= ((Mi[(size_t)i * LW + s / 4] >> (8 * (s % 4))) & 0xFFu) << (8 * a);
    }
  }
  Bt[w] = v;
}

size_t crt_btable_bytes(int K, int LW) {
  const size_t NT = (size_t)(LW + 31) / 32, KC = (size_t)(K + 31) / 32;
  return NT * KC * CHUNK;
}

void launch_crt_btable(int K, int LW, const uint32_t* Mi, uint32_t* Bt, cudaStream_t st) {
  const size_t words = crt_btable_bytes(K, LW) / 4;
  k_crt_btable<<<(unsigned)((words + 255) / 256), 256, 0, st>>>(K, LW, Mi, (K + 31) / 32, Bt, words);
}

// y in the A layout (crt_a_word), Bt as above -> S [N][LWp] u64 limb sums,
// LWp = 32 * NT.  Thread 0 is the producer (bulk copies of both operands into a
// STAGES-deep ring) and the MMA issuer; the four warps run the epilogue.
__global__ void __launch_bounds__(THREADS, 1) k_crt_mma(int N, int KC, const uint8_t* __restrict__ yA,
                                                        const uint8_t* __restrict__ Bt, int LWp,
                                                        unsigned long long* __restrict__ S) {
  extern __shared__ __align__(1024) uint8_t smem[];
  CKB_SMEM_POISON(smem);
  uint8_t* sA = smem;                      // [STAGES][CHUNK]
  uint8_t* sB = smem + STAGES * CHUNK;     // [STAGES][CHUNK]
  // full[STAGES], done[STAGES], then `fin` (one phase: every MMA of the tile retired)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * STAGES * CHUNK);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mt = blockIdx.x, nt = blockIdx.y, k0 = mt * BM;
  const uint32_t full0 = smem_u32(bars), done0 = smem_u32(bars + STAGES), fin = smem_u32(bars + 2 * STAGES);

  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(done0 + 8 * s, 1);
    }
    mbar_init(fin, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "n"(BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // pdl_launch();  (implicit at exit: measured better)
  pdl_wait();  // y (the interpolation's output) from here on

  if (tid == 0) {
    const uint8_t* gA = yA + (size_t)mt * KC * CHUNK;
    const uint8_t* gB = Bt + (size_t)nt * KC * CHUNK;
    auto issue = [&](int c) {
      const int s = c % STAGES;
      mbar_expect_tx(full0 + 8 * s, 2 * CHUNK);
      bulk_g2s(smem_u32(sA + s * CHUNK), gA + (size_t)c * CHUNK, CHUNK, full0 + 8 * s);
      bulk_g2s(smem_u32(sB + s * CHUNK), gB + (size_t)c * CHUNK, CHUNK, full0 + 8 * s);
    };
    for (int c = 0; c < STAGES && c < KC; ++c) issue(c);
    for (int kc = 0; kc < KC; ++kc) {
      const int s = kc % STAGES;
      mbar_wait(full0 + 8 * s, (kc / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t abase = smem_u32(sA + s * CHUNK), bbase = smem_u32(sB + s * CHUNK);
#pragma unroll
      for (int ks = 0; ks < BK / 32; ++ks)
        mma_i8(tmem, desc_kmajor(abase + ks * 256), desc_kmajor(bbase + ks * 256), (kc | ks) != 0);
      mma_commit(done0 + 8 * s);
      // refill the stage the previous chunk's MMAs read (they are queued ahead of this chunk's)
      const int pc = kc - 1;
      if (pc >= 0 && pc + STAGES < KC) {
        mbar_wait(done0 + 8 * (pc % STAGES), (pc / STAGES) & 1);
        issue(pc + STAGES);
      }
    }
    mma_commit(fin);
  }
  __syncwarp();
  // fin has a single phase, so parity 0 is unambiguous for threads that arrive
  // early (a done[] barrier could still be in an earlier phase)
  mbar_wait(fin, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");

  // epilogue: warp w owns TMEM lanes 32w..32w+31 (= coefficients)
  const uint32_t lane_base = tmem + ((uint32_t)(warp * 32) << 16);
  unsigned long long* out = S + (size_t)(k0 + warp * 32 + lane) * LWp + nt * (BN / 4);
  const bool live = k0 + warp * 32 + lane < N;
#pragma unroll
  for (int c0 = 0; c0 < BN; c0 += 32) {
    uint32_t r[32];
    CKB_LD32(r, lane_base + c0);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (live) {
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        const unsigned long long sum = (unsigned long long)r[4 * l] + ((unsigned long long)r[4 * l + 1] << 8) +
                                       ((unsigned long long)r[4 * l + 2] << 16) +
                                       ((unsigned long long)r[4 * l + 3] << 24);
        out[c0 / 4 + l] = sum;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(BN));
}

size_t crt_mma_smem() { return 2 * STAGES * CHUNK + (2 * STAGES + 1) * 8 + 16; }

void launch_crt_mma(const CrtTables& t, const uint32_t* y, int N, unsigned long long* S, cudaStream_t st) {
  static bool attr = false;
  const int smem = (int)crt_mma_smem();
  if (!attr) {
    cudaFuncSetAttribute(k_crt_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  const int NT = (t.LW + 31) / 32, KC = (t.K + 31) / 32;
  dim3 grid((N + BM - 1) / BM, NT);
  launch_pdl(k_crt_mma, grid, dim3(THREADS), smem, st, N, KC, reinterpret_cast<const uint8_t*>(y), t.Bt, NT * 32, S);
}

// ===========================================================================
// Interpolation as a tensor-core product (polyphase plans).
//
// For one prime the 8 coset phases interpolate at the SAME geometric points
// z_u = q^u (u < M), so every phase is one product with the same matrix:
//     P_r[k] = sum_u A[k][u] X_r[u],   A = inverse Vandermonde of the z_u
//     (A[k][u] = coefficient k of the Lagrange basis polynomial L_u),
//     X_r[u] = (1/S) (c y_u)^-r sum_j w^-jr v[u S + j]   (phase separation)
// — the same values the NTT correlations of k_interp_poly produce.  Both
// operands are split into bytes, A[k][u] = sum_a 2^8a A_a and X = sum_b 2^8b
// X_b, so one u8 GEMM with rows (k, a), columns (r, b) and K = u gives
// D[(k,a)][(r,b)] = sum_u A_a X_b < M 255^2 < 2^25, recombined mod p in the
// epilogue.  A is input-independent: built once per plan (bytes in the
// no-swizzle K-major core-matrix layout, like the CRT tables) and streamed by
// the bulk-copy engine; X is built per call in shared memory by each CTA.
// ===========================================================================
namespace {
constexpr uint32_t IDESC_N32 = (2u << 4) | ((uint32_t)(32 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
// K in steps of 32 bytes (one MMA each), so K is padded to a multiple of 32 only:
// per step, 8-row groups of 2 core matrices (SBO 256 B, LBO 128 B)
constexpr int IA_TILE = 128 * 32;  // A bytes per (M-tile, K-step)
constexpr int IB_TILE = 32 * 32;   // B bytes per K-step
__device__ __forceinline__ size_t ia_byte(int row, int u, int KCH) {  // row = 4k + a; KCH = K-steps
  const size_t tile = (size_t)(row >> 7) * KCH + (u >> 5);
  return tile * IA_TILE + ((row & 127) >> 3) * 256 + ((u & 31) >> 4) * 128 + (row & 7) * 16 + (u & 15);
}
__device__ __forceinline__ size_t ib_byte(int n, int u) {  // n = 4r + b
  return (size_t)(u >> 5) * IB_TILE + (n >> 3) * 256 + ((u & 31) >> 4) * 128 + (n & 7) * 16 + (u & 15);
}
__device__ __forceinline__ uint64_t desc_kmajor_s256(uint32_t addr) {  // LBO 128 B, SBO 256 B
  const uint64_t lo = ((addr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16);
  const uint64_t hi = (uint64_t)(256 >> 4) | (1ull << 14);
  return lo | (hi << 32);
}
__device__ __forceinline__ void mma_i8_n32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC_N32), "r"(acc));
}
}  // namespace

// plan: A bytes for every prime (one CTA per prime, one thread per point u):
// L_u = M~(z) / ((z - z_u) M~'(z_u)) by synthetic division
__global__ void k_interp_lagrange(const Prime* __restrict__ primes, InterpPlan plan, int KCH, int MT,
                                  uint8_t* __restrict__ Ab) {
  const int pi = blockIdx.x, M = plan.N;
  const Prime P = primes[pi];
  const uint32_t p = P.p;
  const uint32_t* Mt = plan.Mt + (size_t)pi * (M + 1);  // M~ = prod_u (z - z_u), degree M
  uint8_t* A = Ab + (size_t)pi * MT * KCH * IA_TILE;
  for (int u = threadIdx.x; u < M; u += blockDim.x) {
    const uint32_t x = plan.xq[(size_t)pi * M + u], xc = shoup_comp(x, P);
    // M~'(x) by Horner on the derivative
    uint32_t d = 0u;
    for (int j = M; j >= 1; --j) d = add_mod(shoup(d, x, xc, p), mul_mod(Mt[j], (uint32_t)j % p, P), p);
    const uint32_t inv = inv_mod(d, P), invc = shoup_comp(inv, P);
    // quotient Q = M~ / (z - x): Q_{M-1} = Mt[M], Q_{j-1} = Mt[j] + x Q_j
    uint32_t q = Mt[M];
    for (int k = M - 1; k >= 0; --k) {
      const uint32_t a = shoup(q, inv, invc, p);  // A[k][u] = Q_k / M~'(x)
#pragma unroll
      for (int b = 0; b < 4; ++b) A[ia_byte(4 * k + b, u, KCH)] = (uint8_t)(a >> (8 * b));
      if (k > 0) q = add_mod(Mt[k], shoup(q, x, xc, p), p);
    }
  }
}

// X bytes of one point u of prime pi (phase separation and weights) into B (shared or global)
__device__ __forceinline__ void interp_x_bytes(const Prime& P, int pi, int u, const InterpPlan& plan,
                                               const uint32_t* __restrict__ values, uint32_t c, uint32_t cinv,
                                               uint32_t inv8, uint8_t* B) {
  const int M = plan.N, S = plan.S;
  const uint32_t p = P.p;
  uint32_t X[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
  if (u < M) {
    const uint32_t* om = plan.om + (size_t)pi * 4 * S;  // w^k, companions, w^-k, companions
    const uint32_t* v = values + ((size_t)pi * M + u) * S;
    uint32_t vv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) vv[j] = v[j];
    // weight (1/S) (c y_u)^-r, r = 0..7
    uint32_t step = plan.yqi[(size_t)pi * M + u];
    if (c != 1u) step = mul_mod(step, cinv, P);
    const uint32_t stepc = shoup_comp(step, P);
    // g_r = sum_j w^-jr v_j: radix-2 DIT on the bit-reversed inputs, natural-order outputs
    // (5 twiddle products instead of 64)
    uint32_t x[8];
#pragma unroll
    for (int m = 0; m < 8; ++m) x[m] = vv[((m & 1) << 2) | (m & 2) | ((m >> 2) & 1)];
#pragma unroll
    for (int h = 1; h < 8; h <<= 1) {
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        if (l & h) continue;
        const int e = (l & (h - 1)) * (8 / (2 * h));  // w^-e
        const uint32_t t = e ? shoup(x[l + h], om[2 * S + e], om[3 * S + e], p) : x[l + h];
        const uint32_t a0 = x[l];
        x[l] = add_mod(a0, t, p);
        x[l + h] = sub_mod(a0, t, p);
      }
    }
    uint32_t wr = inv8;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      X[r] = mul_mod(x[r], wr, P);
      wr = shoup(wr, step, stepc, p);
    }
  }
#pragma unroll
  for (int r = 0; r < 8; ++r)
#pragma unroll
    for (int b = 0; b < 4; ++b) B[ib_byte(4 * r + b, u)] = (uint8_t)(X[r] >> (8 * b));
}

__device__ __forceinline__ uint32_t inv8_mod(const Prime& P) {  // ((p + 1) / 2)^3 = 1/8
  const uint32_t h = (P.p + 1u) >> 1;
  return mul_mod(mul_mod(h, h, P), h, P);
}

// per call: the product, one CTA per (M-tile of 32 coefficients, prime); the
// epilogue recombines the bytes mod p and writes the CRT's y layout (or canonical)
__global__ void __launch_bounds__(128, 1) k_interp_mma(const Prime* __restrict__ primes, InterpPlan plan,
                                                       const uint8_t* __restrict__ Ab,
                                                       const uint32_t* __restrict__ values,
                                                       int KCH, int MT, const uint32_t* __restrict__ cval,
                                                       uint32_t* __restrict__ coeffs, const uint32_t* __restrict__ crt_c,
                                                       PeerOut po) {
  extern __shared__ __align__(1024) uint8_t smem[];
  CKB_SMEM_POISON(smem);
  uint8_t* sA = smem;                        // [KCH][16 KB]
  uint8_t* sB = smem + (size_t)KCH * IA_TILE;  // [KCH][4 KB]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB + (size_t)KCH * IB_TILE);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mt = blockIdx.x, pi = blockIdx.y, M = plan.N, S = plan.S, Nfull = plan.Nfull;
  const uint32_t full = smem_u32(bars), fin = smem_u32(bars + 1);
  if (tid == 0) {
    mbar_init(full, 1);
    mbar_init(fin, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                 "n"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // the A tiles (plan constants) stream in while the CTA builds X
  if (tid == 0) {
    mbar_expect_tx(full, (uint32_t)KCH * IA_TILE);
    bulk_g2s(smem_u32(sA), Ab + ((size_t)pi * MT + mt) * KCH * IA_TILE, (uint32_t)KCH * IA_TILE, full);
  }
  pdl_wait();  // the images' values
  {
    // X for every point of this prime, straight into the B operand's shared-memory layout
    const Prime P = primes[pi];
    const uint32_t c = cval[pi];
    const uint32_t cinv = c != 1u ? inv_mod(c, P) : 1u, inv8 = inv8_mod(P);
    for (int u = tid; u < KCH * 32; u += 128) interp_x_bytes(P, pi, u, plan, values, c, cinv, inv8, sB);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic-proxy writes -> tensor-core reads
  __syncthreads();
  if (tid == 0) {
    mbar_wait(full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    for (int ks = 0; ks < KCH; ++ks)
      mma_i8_n32(tmem, desc_kmajor_s256(smem_u32(sA + (size_t)ks * IA_TILE)),
                 desc_kmajor_s256(smem_u32(sB + (size_t)ks * IB_TILE)), ks != 0);
    mma_commit(fin);
  }
  __syncwarp();
  mbar_wait(fin, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  // epilogue: lane = row (k, a) = 4 k_local + a; columns (r, b) = 4 r + b
  uint32_t r32[32];
  CKB_LD32(r32, tmem + ((uint32_t)(warp * 32) << 16));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
  const Prime P = primes[pi];
  const uint32_t p = P.p;
  const uint64_t m64 = ~0ull / p;
  const int a = lane & 3, k = mt * 32 + warp * 8 + (lane >> 2);
  const uint32_t ra = pow_mod(2u % p, (uint64_t)(8 * a), P), rac = shoup_comp(ra, P);  // 2^8a mod p
  uint32_t out[8];
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const uint64_t T = (uint64_t)r32[4 * r] + ((uint64_t)r32[4 * r + 1] << 8) + ((uint64_t)r32[4 * r + 2] << 16) +
                       ((uint64_t)r32[4 * r + 3] << 24);  // < 2^50
    uint64_t q = __umul64hi(T, m64), t = T - q * p;
    while (t >= p) t -= p;
    uint32_t x = shoup((uint32_t)t, ra, rac, p);
    x = add_mod(x, __shfl_xor_sync(0xffffffffu, x, 1), p);
    x = add_mod(x, __shfl_xor_sync(0xffffffffu, x, 2), p);
    out[r] = x;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(32));
  if (a != 0 || k >= M) return;
  const uint32_t c = cval[pi];
  uint32_t sc = 1u;  // (c^S)^-k
  if (c != 1u) sc = pow_mod(pow_mod(inv_mod(c, P), (uint64_t)S, P), (uint64_t)k, P);
  if (crt_c) sc = mul_mod(sc, crt_c[pi], P);
  const uint32_t scc = shoup_comp(sc, P);
  const int KC = (plan.K + 31) / 32;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int idx = S * k + r;
    if (idx >= Nfull) continue;
    const uint32_t res = shoup(out[r], sc, scc, p);
    if (crt_c)
      store_y(coeffs, po, pi, idx, KC, res);  // CRT A layout (peer contexts' inputs with po)
    else
      coeffs[(size_t)pi * Nfull + idx] = res;
  }
}

size_t interp_mma_bytes(int K, int M, int* KCH, int* MT) {
  *KCH = (M + 31) / 32;  // K-steps of 32 bytes
  *MT = (4 * M + 127) / 128;
  return (size_t)K * (*MT) * (*KCH) * IA_TILE;
}

void launch_interp_lagrange(const Prime* primes, const InterpPlan& plan, uint8_t* Ab, cudaStream_t st) {
  int KCH, MT;
  const size_t bytes = interp_mma_bytes(plan.K, plan.N, &KCH, &MT);
  cudaMemsetAsync(Ab, 0, bytes, st);
  k_interp_lagrange<<<plan.K, 128, 0, st>>>(primes, plan, KCH, MT, Ab);
}

void launch_interp_mma(const InterpPlan& plan, const Prime* primes, const uint32_t* values, const uint32_t* cval,
                       uint32_t* coeffs, cudaStream_t st, const uint32_t* crt_c, const PeerOut* po) {
  PeerOut pv = po ? *po : PeerOut{};
  if (!po) pv.G = 0;
  int KCH, MT;
  interp_mma_bytes(plan.K, plan.N, &KCH, &MT);
  const size_t smem = (size_t)KCH * (IA_TILE + IB_TILE) + 64;
  static size_t attr = 0;
  if (smem > attr) {
    cudaFuncSetAttribute(k_interp_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = smem;
  }
  launch_pdl(k_interp_mma, dim3(MT, plan.K), dim3(128), smem, st, primes, plan, (const uint8_t*)plan.Ab, values,
             KCH, MT, cval, coeffs, crt_c, pv);
}

}  // namespace ckb

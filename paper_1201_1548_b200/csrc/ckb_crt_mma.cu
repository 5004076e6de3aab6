// K5 on the tensor cores: the explicit-CRT product X = sum_i y_i (M/p_i) as an
// unsigned 8-bit GEMM on tcgen05 (kind::i8, s32 accumulators in TMEM).
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

}  // namespace ckb

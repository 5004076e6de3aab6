// Kernel declarations shared by the stage files and the C-ABI layer.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "ckb_modarith.cuh"

namespace ckb {

// ---- programmatic dependent launch (PDL) ----------------------------------
// The pipeline kernels run back to back on one stream (inside a CUDA graph when
// replayed).  Each is launched with programmatic stream serialization, so its
// CTAs may start while the previous kernel's last wave drains; every such
// kernel executes pdl_wait() (griddepcontrol.wait: the previous grid has
// completed and its writes are visible) before touching the previous kernels'
// outputs, and before it exits, which makes completion transitive along the
// chain.  pdl_launch() lets the next kernel be scheduled once every CTA of
// this one has started.  Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
extern bool g_pdl;  // CKB_NO_PDL=1 disables the attribute (A/B measurements)

// Checking builds (-DCKB_POISON_SMEM, tools/build_variants.py; compute-sanitizer is closed on
// this GPU pool): every kernel with dynamic shared memory first fills all of it with a poison
// word, so reading a word that no thread and no bulk copy wrote surfaces as a parity failure.
// The proxy fence orders the poison stores before the CTA's own bulk copies / tensor-core reads.
#ifdef CKB_POISON_SMEM
#define CKB_SMEM_POISON(base)                                                                   \
  do {                                                                                          \
    uint32_t nb_;                                                                               \
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(nb_));                               \
    uint32_t* w_ = reinterpret_cast<uint32_t*>(base);                                           \
    const uint32_t t_ = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);    \
    const uint32_t nt_ = blockDim.x * blockDim.y * blockDim.z;                                  \
    for (uint32_t i_ = t_; i_ < nb_ / 4; i_ += nt_) w_[i_] = 0xA5A5A5A5u;                       \
    __syncthreads();                                                                            \
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");                             \
  } while (0)
#else
#define CKB_SMEM_POISON(base) \
  do {                        \
  } while (0)
#endif
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

// ---- K1: coefficient reduction (modpoly.py:376-377) ------------------------
// limbs: [C][L] two's-complement little-endian u32 words; out: [K][C] in [0,p)
void launch_reduce(const uint32_t* limbs, int C, int L, const Prime* primes, int K, uint32_t* out,
                   cudaStream_t st);

// ---- plan: evaluation points + interpolation tables per prime ---------------
// Depends only on (primes, generators, N): built once and cached, like an FFT
// plan.  Points are x_t = c q^t; every table is for c = 1 (the interpolation
// runs in y = x / c and the per-call scale c only enters through c^-k).
struct InterpPlan {
  int N;              // interpolation points per prime (per polyphase component: M = ceil(Nfull / S))
  int K;              // primes
  int S;              // polyphase factor: images at w^j y_u (j < S, u < N), w a primitive S-th root
  int Nfull;          // requested points (coefficients of the result)
  int L, logL;        // NTT length: power of two >= 2N - 1
  uint32_t* yq;       // [K][N]    g^u   (image base points y_u for c = 1)
  uint32_t* yqi;      // [K][N]    g^-u
  uint32_t* om;       // [K][4S]   w^k, companions, w^-k, companions
  uint32_t* xq;       // [K][N]    q^t with q = g^S (the interpolation points z_t)
  uint32_t* hC;       // [K][2N]   q^C(m,2)              (construction scratch)
  uint32_t* hCinv;    // [K][N]    q^-C(e,2)             (construction scratch)
  uint32_t* Mt;       // [K][N+1]  coefficients of M~(y) = prod_t (y - q^t)   (scratch)
  uint32_t* phi;      // [K][N+1]  prod_{i<=j} (q^i - 1)  (scratch)
  uint32_t* iphi;     // [K][N+1]  inverses of phi       (scratch)
  uint32_t* z;        // [K][N]    1/M~'(q^t) * q^-C(t,2)   and companions zc
  uint32_t* zc;
  uint32_t* sS;       // [K][N]    q^-C(e,2) / L           and companions sSc
  uint32_t* sSc;
  uint32_t* W;        // [K][L/2]  w^j, w a primitive L-th root; Wc companions
  uint32_t* Wc;
  uint32_t* Wi;       // [K][L/2]  w^-j; Wic companions
  uint32_t* Wic;
  uint32_t* Hf;       // [K][L]    DIF-NTT of q^C(m,2) (m < 2N-1); Hfc companions
  uint32_t* Hfc;
  uint32_t* Mf;       // [K][L]    DIF-NTT of M~_{u+1} (u < N); Mfc companions
  uint32_t* Mfc;
  uint32_t* Linv;     // [K]       1/L mod p
  uint32_t* zr;       // [K][S][N] (1/S) y_t^-r z_t (polyphase plans), companions zrc
  uint32_t* zrc;
  uint8_t* Ab;        // polyphase plans: inverse-Vandermonde bytes for the tensor-core interpolation, or nullptr
};
// build every table of the plan: base tables (ckb_plan.cu), then twiddles and
// the transforms of the two constant convolution operands (ckb_interp.cu)
void launch_plan_base(const Prime* primes, const uint32_t* gens, const InterpPlan& plan, cudaStream_t st);
void launch_plan_ntt(const Prime* primes, const uint32_t* gens, const InterpPlan& plan, cudaStream_t st);
// per call: choose c per prime so that no leading coefficient vanishes at
// x_t = c q^t (t < N).  lc polynomials of f and g (residues) are read from the
// reduced buffer: lcf = red + lcf_off (deg lcf_deg), lcg likewise, row stride C.
void launch_choose_c(const Prime* primes, const InterpPlan& plan, const uint32_t* red, int C, int lcf_off,
                     int lcf_deg, int lcg_off, int lcg_deg, uint32_t* cval, uint32_t* status, cudaStream_t st);

// ---- K2+K3: fused evaluation + univariate resultant (modpoly.py:382-390) ----
struct ImageArgs {
  const uint32_t* red;     // [K][C]
  const uint32_t* tab;     // [K][images_tab_words] residues in the kernel's shared-memory layout
  const int16_t* degs;     // [(m+1) + (n+1)] x-degree of each y-coefficient (-1 = zero)
  const uint32_t* yq;      // [K][M] g^u (plan)
  const uint32_t* om;      // [K][4 S] roots of unity (plan)
  const uint32_t* cval;    // [K] point scale c: image (u, j) at x = w^j c g^u
  const Prime* primes;
  int C, m, n, dfx, dgx, N, K;  // N = S * M images per prime, stored at u * S + j
  int M;
  uint32_t* values;        // [K][N]
  uint32_t* status;        // bit 1: an image hit a vanishing leading coefficient
  uint32_t* fail_list;     // [K*N] flat indices of non-generic images
  uint32_t* fail_count;    // zeroed before the launch
  int span;                // set by launch_images: max primes one CTA's images touch
};
int images_maxd(int m, int n);  // template bucket or -1
// whether the register kernel handles this shape (bucket exists, tables fit in shared memory)
bool images_fast_ok(int m, int n, int dfx, int dgx, int NI, int K);
// every image through the general warp kernel (any degree)
void launch_images_general(const ImageArgs& a, cudaStream_t st);
// K1 for the pipeline: residues straight into the images kernel's transposed,
// top-aligned, zero-padded table layout (and the plain [K][C] layout)
size_t images_tab_words(int m, int n, int dfx, int dgx);
// with plan != nullptr the same launch also chooses every prime's point scale
// (k_choose_c's work, one extra CTA per prime) when reduce_tab_chooses(...)
bool reduce_tab_chooses(int lcf_deg, int lcg_deg);
void launch_reduce_tab(const uint32_t* limbs, int C, int L, const Prime* primes, int K, int m, int n, int dfx,
                       int dgx, uint32_t* red, uint32_t* tab, cudaStream_t st, const InterpPlan* plan = nullptr,
                       int lcf_off = 0, int lcf_deg = 0, int lcg_off = 0, int lcg_deg = 0, uint32_t* cval = nullptr,
                       uint32_t* status = nullptr, uint32_t* zero_word = nullptr);  // zero_word: set to 0 by K1
// fast generic kernel followed by the general warp kernel on its fail list
void launch_images(const ImageArgs& a, cudaStream_t st, bool structured = false);
void launch_images_fallback(const ImageArgs& a, cudaStream_t st);

// batch of independent univariate resultants (modpoly.py:156-161)
// fa/gb: [B][W] padded low-first coefficients; degrees da/db; per-pair prime index
void launch_uni_resultant(const uint32_t* fa, const int32_t* da, const uint32_t* gb, const int32_t* db, int W,
                          const Prime* primes, const int32_t* pidx, int B, uint32_t* out, uint32_t* gs,
                          cudaStream_t st);  // gs: null = operands in shared memory, else 3 W words per pair

struct PeerOut;  // below (multi-device res_y)

// ---- K4: interpolation at the planned points (modpoly.py:164-185) -----------
// values at the planned points -> coeffs [K][Nfull] (canonical residues); with
// crt_c (polyphase plans only) each prime's row is pre-multiplied by crt_c[i]
// for the explicit CRT (then launch_crt must be told the input is already y)
// with plan.Ab set (polyphase plans whose inverse Vandermonde fits) the
// interpolation runs as a tensor-core product (ckb_crt_mma.cu) instead of NTTs
// (po: the peer stores of PeerOut; requires crt_c)
void launch_interp(const InterpPlan& plan, const Prime* primes, const uint32_t* values, const uint32_t* cval,
                   uint32_t* coeffs, cudaStream_t st, const uint32_t* crt_c = nullptr,
                   const uint32_t* crt_cc = nullptr, const PeerOut* po = nullptr);
// tensor-core interpolation (ckb_crt_mma.cu): plan bytes (KCH K-chunks, MT M-tiles), plan build, per-call launch
size_t interp_mma_bytes(int K, int M, int* KCH, int* MT);
void launch_interp_lagrange(const Prime* primes, const InterpPlan& plan, uint8_t* Ab, cudaStream_t st);
void launch_interp_mma(const InterpPlan& plan, const Prime* primes, const uint32_t* values, const uint32_t* cval,
                       uint32_t* coeffs, cudaStream_t st, const uint32_t* crt_c, const PeerOut* po);

// ---- K5: explicit CRT + symmetric lift to two's-complement limbs -----------
struct CrtTables {
  int K, LW;
  const uint32_t* p;      // [K] primes
  const uint32_t* c;      // [K] (M/p_i)^-1 mod p_i
  const uint32_t* cc;     // [K] Shoup companions of c
  const double* pinvd;    // [K] 1/p_i
  const uint32_t* Mi;     // [K][LW] limbs of M/p_i
  const uint32_t* Ml;     // [LW] limbs of M
  const uint32_t* Mh;     // [LW] limbs of floor(M/2)
  const uint8_t* Bt;      // pre-tiled byte table of the M/p_i for the tensor-core product (ckb_crt_mma.cu)
};
// The CRT input y (residues premultiplied by (M/p_i)^-1) is stored directly in
// the tensor-core A-operand layout: tiles of 128 coefficients x 32 primes
// (16 KB), each in the canonical no-swizzle K-major arrangement of 8x16-byte
// core matrices, so the GEMM streams it with bulk copies.  Word index of y_i(n):
__host__ __device__ __forceinline__ size_t crt_a_word(int i, int n, int KC) {
  const size_t tile = (size_t)(n >> 7) * KC + (i >> 5);
  return tile * 4096 + ((n & 127) >> 3) * 256 + ((i & 31) >> 2) * 32 + (n & 7) * 4 + (i & 3);
}
inline size_t crt_a_words(int K, int N) { return (size_t)((N + 127) / 128) * ((K + 31) / 32) * 4096; }
// ---- multi-device res_y: the all-to-all folded into the interpolation -------
// Context d interpolates its block of primes; coefficient idx belongs to context
// s = idx / nc, whose CRT needs it from every prime.  With PeerOut set, the
// interpolation's epilogue stores each y value (already premultiplied for the
// explicit CRT) straight into context s's CRT input -- in that context's HBM, over
// NVLink (peer access) when s lives on another GPU -- at its A-layout position
// (global prime k0 + pi, local coefficient idx - s nc): the exchange step disappears
// and the transfer overlaps the interpolation tile by tile.
constexpr int kMaxPeers = 8;
struct PeerOut {
  uint32_t* dst[kMaxPeers];  // per destination context: its CRT input, A layout over all K primes
  int G;                     // destination contexts (0: plain store into coeffs)
  int nc;                    // coefficients per destination block
  int KC;                    // (K_total + 31) / 32 of the destination layout
  int k0;                    // global index of this context's first prime
};
__device__ __forceinline__ void store_y(uint32_t* coeffs, const PeerOut& po, int pi, int idx, int KC, uint32_t v) {
  if (po.G) {
    const int s = idx / po.nc;
    po.dst[s][crt_a_word(po.k0 + pi, idx - s * po.nc, po.KC)] = v;
  } else {
    coeffs[crt_a_word(pi, idx, KC)] = v;
  }
}
// ---- Descartes sign-variation test (ckb_descartes.cu) -----------------------
struct DescPlan {
  int K, n, L, logL;       // primes, degree, NTT length >= 2n+1
  int direct;              // degree beyond the NTT primes (2n+1 > 2^14): direct O(n^2) correlations
  uint32_t *fact, *ifact;  // [K][n+1] i! and 1/i! mod p
  uint32_t *W, *Wc, *Wi, *Wic;  // [K][L/2] twiddles and companions (NTT mode)
  uint32_t *Vf, *Vfc;      // [K][L] DIF of (1/0!, ..., 1/n!, 0, ...) and companions (NTT mode);
                           // direct mode: Vf = [K][n+1] scan scratch of the plan kernel
  uint32_t* Linv;          // [K] 1/L
};
constexpr int DESC_NTT_LOG2_MAX = 14;  // PRIMES30: p = 1 mod 2^14
void launch_desc_plan(const Prime* primes, const uint32_t* gens, const DescPlan& pl, cudaStream_t st);
// B intervals at once: aw [B][2][AL], ld [B] (device) -> out [K][B N]; signs: B results.
// Direct mode needs scratch of desc_direct_scratch_words(K, n, B) words.
void launch_desc_shift(const Prime* primes, const DescPlan& pl, const uint32_t* res, const uint32_t* aw, int AL,
                       const int32_t* ld, int B, uint32_t* out, uint32_t* scratch, cudaStream_t st);
inline size_t desc_direct_scratch_words(int K, int n, int B) { return (size_t)K * B * 3 * (n + 1); }
void launch_desc_signs(const uint32_t* limbs, int N, int LW, int B, int32_t* result, cudaStream_t st);

// tensor-core CRT product (ckb_crt_mma.cu): byte table size / builder, and the
// GEMM y (A layout) -> S [N][32 ceil(LW/32)] u64 limb sums
size_t crt_btable_bytes(int K, int LW);
void launch_crt_btable(int K, int LW, const uint32_t* Mi, uint32_t* Bt, cudaStream_t st);
void launch_crt_mma(const CrtTables& t, const uint32_t* y, int N, unsigned long long* S, cudaStream_t st);
// coeffs [K][N] residues (or, input_is_y, y in the A layout) -> out [N][LW] (device or mapped
// page-locked host memory); scratch >= crt_scratch_words; status_src -> status_dst when given
// returns the number of kernels launched (GEMM + carry, plus the premultiplication unless input_is_y)
int launch_crt(const CrtTables& t, const uint32_t* coeffs, int N, uint32_t* out, uint32_t* scratch,
               cudaStream_t st, bool input_is_y = false, const uint32_t* status_src = nullptr,
               uint32_t* status_dst = nullptr);
size_t crt_scratch_words(int K, int N, int LW);  // scratch size for launch_crt
// M/p_i limbs [K][LW] and c_i = (M/p_i)^-1 mod p_i (+ Shoup companions) from M's limbs; bad |= 1 on repeated primes
void launch_crt_tables(const uint32_t* primes, int K, const uint32_t* M, int LW, uint32_t* Mi, uint32_t* c,
                       uint32_t* cc, uint32_t* bad, cudaStream_t st);

// ---- K6: batched gcd mod p (modpoly.py:115-122), interpolation at arbitrary points
void launch_gcd_mod(const uint32_t* fa, const int32_t* da, int Wf, const uint32_t* gb, const int32_t* db, int Wg,
                    const Prime* primes, const int32_t* pidx, int B, uint32_t* out, int Wo, int32_t* odeg,
                    uint32_t* gs, cudaStream_t st);  // gs: null or 2 max(Wf, Wg) words per pair
void launch_interp_points(const uint32_t* xs, const uint32_t* vs, const int32_t* ns, int W, const Prime* primes,
                          const int32_t* pidx, int B, uint32_t* out, uint32_t* gs, cudaStream_t st,
                          int xstride = -1);  // gs: null or 4 W + 2 words per problem; xstride -1 = W

// ---- images of the dense modular bivariate gcd (bivpoly.py:266-295)
// res [K][C] residues of A's grid, B's grid, Gamma; out [K*NP][Wo] Gamma(x_t) * monic
// gcd(A(x_t, y), B(x_t, y)) at x_t = t + 1; odeg its degree or -2 (lc vanishes at x_t)
void launch_biv_gcd_images(const uint32_t* res, int C, const int16_t* degs, int m, int n, int dax, int dbx, int dgam,
                           const Prime* primes, int K, int NP, uint32_t* out, int Wo, int32_t* odeg, cudaStream_t st);

// ---- the modular subresultant profile (ckb_psc.cu, modpoly.py:428-526) --------
// points: the first `need` t with lc_f(t) lc_g(t) != 0 -> sel, *count = all such t < ncand
void launch_psc_points(const uint32_t* lcf, int dlf, const uint32_t* lcg, int dlg, const Prime& P, int ncand,
                       int need, uint32_t* sel, int* count, cudaStream_t st);
// psc_i(t) for i = 1..n at pts[0..npts) (pts null: t = index) -> out [n][npts]; valid optional
void launch_psc(const uint32_t* fres, const int16_t* fdeg, int m, int dfx, const uint32_t* gres,
                const int16_t* gdeg, int n, int dgx, const Prime& P, const uint32_t* pts, int npts, uint32_t* out,
                uint8_t* valid, cudaStream_t st);
bool psc_fits(int m, int n);
// S_0 = rstar mod p, S_i = gcd(S_{i-1}, sr_i): chain [n+1] degrees; *status = 2: S_0 lost degree
void launch_gcd_chain(const uint32_t* rmod, int rlen, int rlen_int, const uint32_t* sr, const int* cnt, int W, int n,
                      const Prime& P, int* chain, uint32_t* status, cudaStream_t st);
bool gcd_chain_fits(int rlen, int W);

}  // namespace ckb

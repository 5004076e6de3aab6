// K2+K3: fused evaluation homomorphism + univariate resultant, one thread per
// (prime, point) image.  Restates the reference's inner loop
// (pkg/src/curvekit/modpoly.py:382-390: _zp_eval of every y-coefficient at t,
// then _zp_resultant of the two univariate images) with:
//   * the prime's residue coefficients staged once per CTA in shared memory
//     (all threads of a CTA share the prime; reads are warp broadcasts),
//   * lazy Shoup-Horner evaluation straight into top-aligned registers,
//   * the fused division-free elimination of ckb_resultant.cuh (no inverse in
//     the loop; one Fermat inverse per image),
//   * images whose remainder sequence is not generic appended to a list that
//     the general warp kernel (ckb_general.cu) recomputes exactly.
#include <algorithm>

#include "ckb_kernels.cuh"
#include "ckb_choose.cuh"
#include "ckb_resultant.cuh"
#include "ckb_ntt.cuh"
#include "ckb_images.cuh"

namespace ckb {

static int fallback_warp();

#ifndef CKB_IMG_MINB
#define CKB_IMG_MINB 1
#endif
#ifndef CKB_IMG_MINB_BIG
#define CKB_IMG_MINB_BIG CKB_IMG_MINB
#endif
// CTAs per SM the register allocation must allow (MAXD >= 56: the big buckets)
constexpr int img_minb(int maxd) { return maxd >= 56 ? CKB_IMG_MINB_BIG : CKB_IMG_MINB; }
#ifndef CKB_IMG_THREADS
#define CKB_IMG_THREADS 128
#endif
constexpr int IMG_THREADS = CKB_IMG_THREADS;

// NT = threads (images) per CTA; ALIGNED: grid (ceil(N/NT), K), a CTA never
// straddles primes (one staged table: the register-heavy buckets fit more CTAs)
// EX: 0 any degrees; 1 da = db = MAXD; 2 da = MAXD, db = MAXD - 1 (the dense
// res(f, g) and res(f, f_y) shapes: the elimination chain is unrolled exactly);
// 3 structured inputs: any degree pattern of the remainder sequences, single
// eliminations (no fallback list)
// The unrolled chain lets ptxas keep more values live (cfg4: 178 registers
// uncapped, 8 warps/SM): capped at 128 (16 warps/SM) for MAXD <= 40 and 170
// for 48 it measured fastest (cfg4 images 270 -> 241 us; uncapped 337 us)
#ifndef CKB_IMG_MINB_EX
#define CKB_IMG_MINB_EX 0
#endif
constexpr int exact_minb(int maxd) {
  return CKB_IMG_MINB_EX ? CKB_IMG_MINB_EX : maxd <= 24 ? 4 : maxd <= 32 ? 3 : maxd <= 40 ? 4 : maxd <= 48 ? 3 : img_minb(maxd);
}
template <int MAXD, int NT = IMG_THREADS, bool ALIGNED = false, int EX = 0>
#ifndef CKB_ALIGN_MINB_EX
#define CKB_ALIGN_MINB_EX 1
#endif
__global__ void __launch_bounds__(NT, ALIGNED ? ((EX == 1 || EX == 2) ? CKB_ALIGN_MINB_EX : 1)
                                              : (EX ? exact_minb(MAXD) : img_minb(MAXD))) k_images(ImageArgs a) {
  using LY = ImgLayout<MAXD>;
  constexpr int NCH = LY::NCH, SW = LY::SW;
  extern __shared__ __align__(16) uint32_t sm[];
  CKB_SMEM_POISON(sm);
  const bool sw = a.m < a.n;  // reference swaps so that deg a >= deg b
  const int da = sw ? a.n : a.m, db = sw ? a.m : a.n;
  const int16_t* Adeg = a.degs + (sw ? a.m + 1 : 0);
  const int16_t* Bdeg = a.degs + (sw ? 0 : a.m + 1);
  const int dmax = max(a.dfx, a.dgx);
  const int emax = dmax / POLY;               // Horner steps in z = y^8
  const int rows = POLY * (emax + 1);         // x-power rows, zero-padded
  const int TW = 2 * rows * SW;               // one prime's tables
  // The images of all primes form one flat range (prime-major, N per prime,
  // N a multiple of 8 so a coset never straddles primes); a CTA takes 128
  // consecutive images, so the grid has no per-prime padding and ends in an
  // (almost) full wave.  The tables of every prime the CTA spans are staged
  // (two at most once N >= 128; the launch sizes shared memory for the worst case).
  const int g0 = ALIGNED ? blockIdx.y * a.N + blockIdx.x * NT : blockIdx.x * NT;
  const int total = a.K * a.N;
  const int pi0 = ALIGNED ? blockIdx.y : g0 / a.N;
  const int pi1 = ALIGNED ? blockIdx.y : min(a.K - 1, (g0 + NT - 1) / a.N);
  // per-thread point data first: its global-load latency overlaps the table copy
  const int t = g0 + threadIdx.x;
  // inactive lanes still join the shuffles
  const bool active = ALIGNED ? (int)(blockIdx.x * NT + threadIdx.x) < a.N : t < total;
  const int pi = ALIGNED ? pi0 : (active ? t / a.N : pi1);
  const int tin = ALIGNED ? (active ? t - pi * a.N : 0) : (active ? t - pi * a.N : 0);  // image index within the prime
  const int u = tin >> 3, l = t & (POLY - 1);
  const int tslot = pi - pi0;  // which staged table
  // pdl_launch();  (implicit at exit: measured better)
  const Prime P = a.primes[pi];
  uint32_t y = a.yq[(size_t)pi * a.M + u];  // plan (constant): before the wait
  // TA[e][i] = coefficient of x^e in the y-coefficient of degree da - i (top-aligned),
  // zero beyond each row; maskA[e] = chunks of registers with a term at x^e
  uint32_t* TA = sm + tslot * TW;
  uint32_t* TB = TA + rows * SW;
  const int nspan = pi1 - pi0 + 1;
  uint32_t* maskA = sm + a.span * TW;
  uint32_t* maskB = maskA + rows;
  uint32_t* som = maskB + rows + tslot * 2 * POLY;  // w^k and companions
  // K1 wrote the tables in exactly this layout: ONE bulk copy (TMA engine,
  // cp.async.bulk) lands them in shared memory while the threads build the
  // chunk masks and their points; an mbarrier signals completion
  __shared__ __align__(8) uint64_t tab_bar;
  const uint32_t bar = img_smem_u32(&tab_bar);
  if (threadIdx.x == 0) {
    img_mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  pdl_wait();  // K1's tables and k_choose_c's point scales from here on
  if (threadIdx.x == 0) {
    const uint32_t bytes = (uint32_t)(nspan * TW) * 4u;  // TW * 4 is a multiple of 32
    img_mbar_expect_tx(bar, bytes);
    img_bulk_g2s(img_smem_u32(sm), a.tab + (size_t)pi0 * TW, bytes, bar);
  }
  for (int e = threadIdx.x; e < rows; e += NT) {
    uint32_t ma = 0, mb = 0;
    for (int i = 0; i <= MAXD; ++i) {
      if (i <= da && Adeg[da - i] >= e) ma |= 1u << (i >> 2);
      if (i <= db && Bdeg[db - i] >= e) mb |= 1u << (i >> 2);
    }
    maskA[e] = ma;
    maskB[e] = mb;
  }
  for (int q = threadIdx.x; q < nspan * 2 * POLY; q += NT)
    maskB[rows + q] = a.om[(size_t)(pi0 + q / (2 * POLY)) * 4 * POLY + q % (2 * POLY)];

  // image (u, j): x = w^j c y_u.  Lane l of an 8-lane group evaluates the
  // polyphase component G_l = y^l F_l(y^8) of every y-coefficient; a 3-stage
  // DFT across the group then gives f(w^j y) for all j (j = bitrev(l)).
  const uint32_t c = a.cval[pi];
  const uint32_t p = P.p;
  if (c != 1u) y = shoup(y, c, shoup_comp(c, P), p);  // y_u = c g^u
  const uint32_t y2 = mul_mod(y, y, P), y4 = mul_mod(y2, y2, P);
  const uint32_t z = mul_mod(y4, y4, P);  // Horner variable y^8
  __syncthreads();     // masks, roots (and the barrier's initialisation) visible
  img_mbar_wait(bar, 0);  // tables landed
  uint32_t yl = (l & 1) ? y : 1u;          // y^l, l < 8
  if (l & 2) yl = mul_mod(yl, y2, P);
  if (l & 4) yl = mul_mod(yl, y4, P);
  const uint32_t zc = comp_from_mont(to_mont(z, P), P);

  // Horner in z of all y-coefficients in lock-step: one dynamic loop, every
  // register an independent chain (ILP = m + n + 2); each chunk of 4
  // coefficients is one 16-byte load.  A chain that has not started yet
  // multiplies 0, so the masks only skip work.
  uint32_t A[MAXD + 1], B[MAXD + 1];
#pragma unroll
  for (int i = 0; i <= MAXD; ++i) A[i] = B[i] = 0u;
  uint32_t negp = 0u - p;
  uint32_t zcp = zc;
  // opaque to the optimiser: keeps both in registers instead of letting
  // ptxas rematerialise the companion (7 instructions) in every chunk
  asm volatile("" : "+r"(negp), "+r"(zcp));
  {
    // the top row starts every chain: a plain load (z * 0 + c would cost a product per register)
    const int e = l + POLY * emax;
    const uint4* ta = reinterpret_cast<const uint4*>(TA + e * SW);
    const uint4* tb = reinterpret_cast<const uint4*>(TB + e * SW);
    const uint32_t mA = __reduce_or_sync(0xffffffffu, maskA[e]);
    const uint32_t mB = __reduce_or_sync(0xffffffffu, maskB[e]);
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      if (mA & (1u << c)) {
        const uint4 v = ta[c];
        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (4 * c + k <= MAXD) A[4 * c + k] = vv[k];
      }
      if (mB & (1u << c)) {
        const uint4 v = tb[c];
        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (4 * c + k <= MAXD) B[4 * c + k] = vv[k];
      }
    }
  }
  for (int e2 = emax - 1; e2 >= 0; --e2) {
    const int e = l + POLY * e2;
    const uint4* ta = reinterpret_cast<const uint4*>(TA + e * SW);
    const uint4* tb = reinterpret_cast<const uint4*>(TB + e * SW);
    // union over the warp's rows: a chunk is skipped only where no lane's
    // chains have started (a started chain never sees a cleared bit), so the
    // union is as valid as the lane's own mask and makes the guards uniform
    const uint32_t mA = __reduce_or_sync(0xffffffffu, maskA[e]);
    const uint32_t mB = __reduce_or_sync(0xffffffffu, maskB[e]);
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      if (mA & (1u << c)) {
        const uint4 v = ta[c];
        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (4 * c + k <= MAXD) A[4 * c + k] = shoup_lazy_add(A[4 * c + k], z, zcp, negp, vv[k]);
      }
      if (mB & (1u << c)) {
        const uint4 v = tb[c];
        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (4 * c + k <= MAXD) B[4 * c + k] = shoup_lazy_add(B[4 * c + k], z, zcp, negp, vv[k]);
      }
    }
  }
  // G_l = y^l F_l, then the radix-2 DIF network across the group
  {
    const uint32_t ylc = comp_from_mont(to_mont(yl, P), P);
#pragma unroll
    for (int i = 0; i <= MAXD; ++i) {
      A[i] = shoup_lazy(A[i], yl, ylc, p);
      B[i] = shoup_lazy(B[i], yl, ylc, p);
    }
  }
  const uint32_t p2 = 2u * p;
  const unsigned FULL = 0xffffffffu;
#pragma unroll
  for (int h = POLY / 2; h >= 1; h >>= 1) {
    const bool upper = (l & h) != 0;
    const int widx = (l & (h - 1)) * (POLY / (2 * h));
#ifndef CKB_NO_BF_SPLIT
    if (h > 1) {
      // split butterflies: the lower lane of a pair does the whole butterfly of
      // A[i], the upper lane that of B[i] (one product per butterfly instead of
      // one per lane), then they trade the halves that belong to the other lane
      const uint32_t wp = som[widx], wpc = som[POLY + widx];
#pragma unroll
      for (int i = 0; i <= MAXD; ++i) {
        const uint32_t recv = __shfl_xor_sync(FULL, upper ? A[i] : B[i], h);
        const uint32_t lo = upper ? recv : A[i], hi = upper ? B[i] : recv;  // the pair's lower / upper values
        const uint32_t sum = red2p(lo + hi, p2);
        const uint32_t dif = shoup_lazy(lo - hi + p2, wp, wpc, p);
        const uint32_t recv2 = __shfl_xor_sync(FULL, upper ? sum : dif, h);
        A[i] = upper ? recv2 : sum;
        B[i] = upper ? dif : recv2;
      }
      continue;
    }
#endif
    const uint32_t w = upper ? som[widx] : 1u;
    const uint32_t wc = upper ? som[POLY + widx] : (uint32_t)(0x100000000ull / p);  // companion of 1
#pragma unroll
    for (int i = 0; i <= MAXD; ++i) {
      // upper lane: (lower - own) w in [0, 2p) via min(d, d + 2p); the last
      // stage's twiddle is 1 and the elimination accepts [0, 4p), so it skips
      // the product
      const uint32_t oa = __shfl_xor_sync(FULL, A[i], h), ob = __shfl_xor_sync(FULL, B[i], h);
      const uint32_t da_ = oa - A[i], db_ = ob - B[i];
      const uint32_t xa = upper ? min(da_, da_ + p2) : A[i] + oa;
      const uint32_t xb = upper ? min(db_, db_ + p2) : B[i] + ob;
      A[i] = (h == 1) ? xa : shoup_lazy(xa, w, wc, p);
      B[i] = (h == 1) ? xb : shoup_lazy(xb, w, wc, p);
    }
  }
  const int j = ((l & 1) << 2) | (l & 2) | ((l >> 2) & 1);  // bitrev3(l)
  const int idx = u * POLY + j;  // = tin - l + j
  if (!active) return;  // no shuffles below this point
  uint32_t v;
  if (red4(A[0], p) == 0u || red4(B[0], p) == 0u) {
    atomicOr(a.status, 2u);  // the plan guarantees this never happens
    v = 0u;
  } else {
    const bool neg = sw && ((a.m * a.n) & 1);
    if constexpr (EX == 3)
      v = resultant_anydeg<MAXD>(A, da, B, db, neg, P);  // structured inputs: never CKB_FAIL
    else if constexpr (EX == 1)
      v = resultant_generic<MAXD, MAXD>(A, da, B, db, neg, P);
    else if constexpr (EX == 2)
      v = resultant_generic<MAXD, MAXD - 1>(A, da, B, db, neg, P);
    else
      v = resultant_generic<MAXD>(A, da, B, db, neg, P);
    if (v == CKB_FAIL) {
      const uint32_t slot = atomicAdd(a.fail_count, 1u);
      a.fail_list[slot] = (uint32_t)((size_t)pi * a.N + idx);
      v = 0u;
    }
  }
  a.values[(size_t)pi * a.N + idx] = v;
}

// The images the register kernel could not finish (a remainder sequence that is
// not generic), one THREAD per image: evaluation of every y-coefficient at the
// image's point straight from the residues (Horner, the warp's threads mostly
// share a prime, so the coefficient loads are broadcasts) and the any-degree
// elimination in registers (resultant_anydeg).  A grid of resident CTAs strides
// over the list; an empty list (the usual case) costs one short launch.
template <int MAXD>
__global__ void __launch_bounds__(128) k_images_fallback_reg(ImageArgs a) {
  pdl_wait();
  const uint32_t count = *a.fail_count;
  const bool sw = a.m < a.n;
  const int da = sw ? a.n : a.m, db = sw ? a.m : a.n;
  constexpr int SW = ImgLayout<MAXD>::SW;
  const int dmax = max(a.dfx, a.dgx);
  const int rows = POLY * (dmax / POLY + 1);
  const int TW = 2 * rows * SW;
  for (uint32_t idx = blockIdx.x * blockDim.x + threadIdx.x; idx < count; idx += gridDim.x * blockDim.x) {
    const uint32_t flat = a.fail_list[idx];
    const int pi = (int)(flat / (uint32_t)a.N);
    const Prime P = a.primes[pi];
    const uint32_t p = P.p;
    const uint32_t c = a.cval[pi];
    const int loc = (int)(flat - (uint32_t)pi * (uint32_t)a.N), S = a.N / a.M;
    const uint32_t* om = a.om + (size_t)pi * 4 * S;
    uint32_t x = shoup(a.yq[(size_t)pi * a.M + loc / S], om[loc % S], om[S + loc % S], p);  // w^j g^u
    if (c != 1u) x = shoup(x, c, shoup_comp(c, P), p);
    const uint32_t xc = shoup_comp(x, P);
    // the residues from K1's tables: TA[e][i] = coefficient of x^e in A's y-coefficient of degree da - i
    const uint32_t* TA = a.tab + (size_t)pi * TW;
    const uint32_t* TB = TA + (size_t)rows * SW;
    uint32_t A[MAXD + 1], B[MAXD + 1];
#pragma unroll
    for (int i = 0; i <= MAXD; ++i) {
      // top-aligned: A[i] = (y-coefficient of degree da - i)(x); f is A unless swapped
      uint32_t va = 0u, vb = 0u;
      if (i <= da) {
        const int dg = a.degs[sw ? a.m + 1 + da - i : da - i];
        for (int e = dg; e >= 0; --e) va = add_mod(shoup(va, x, xc, p), TA[e * SW + i], p);
      }
      if (i <= db) {
        const int dg = a.degs[sw ? db - i : a.m + 1 + db - i];
        for (int e = dg; e >= 0; --e) vb = add_mod(shoup(vb, x, xc, p), TB[e * SW + i], p);
      }
      A[i] = va;
      B[i] = vb;
    }
    const bool neg = sw && ((a.m * a.n) & 1);
    a.values[flat] = resultant_anydeg<MAXD>(A, da, B, db, neg, P);
  }
}

#define CKB_MAXD_LIST(X) X(4) X(8) X(12) X(16) X(20) X(24) X(32) X(40) X(48) X(56) X(64)

static int images_sw(int maxd) {
#define SWOF(D) \
  if (maxd == D) return ImgLayout<D>::SW;
  CKB_MAXD_LIST(SWOF)
#undef SWOF
  return 0;
}

size_t images_tab_words(int m, int n, int dfx, int dgx) {
  const int maxd = images_maxd(m, n);
  const int dmax = dfx > dgx ? dfx : dgx;
  const int rows = POLY * (dmax / POLY + 1);
  return (size_t)2 * rows * images_sw(maxd);
}

// K1 for the pipeline, table-major: each CTA owns RT_ROWS rows (x-powers e) of
// one side's table TA[e][i] / TB[e][i] (= coefficient of x^e in the
// y-coefficient of degree d - i of A / B, A the higher y-degree input) for a
// block of RT_PRIMES primes (per-prime constants staged in shared memory).  A
// thread takes one entry (e, i): it gathers that coefficient's limbs (or writes
// the zero padding) and reduces them modulo every prime of the block, so the
// table stores are consecutive words across the warp -- no memset, no
// scattered 4-byte stores (the coefficient-major K1 it replaces issued one L2
// sector write per residue: 1.04 M sector writes at cfg4, now 0.15 M).
// red[pi][c] (coefficient order) is written only when k_choose_c or the warp
// fallback kernel will read it (write_red); the register fallback reads the tables.
constexpr int RT_PRIMES = 8;
constexpr int RT_ROWS = 4;
constexpr int RT_LC_MAX = 256;  // leading-coefficient x-degrees the merged choose role stages
// Roles by CTA index: the first nred CTAs reduce (row block x side x prime
// block); the K CTAs after them each choose one prime's point scale
// (choose_c_prime), reducing the two leading coefficients straight from the
// limbs — so the separate k_choose_c launch disappears from the pipeline.
template <int LMAX>
__global__ void __launch_bounds__(128) k_reduce_tab(const uint32_t* __restrict__ limbs, int C, int L,
                                                    const Prime* __restrict__ primes, int K, int m, int n, int dfx,
                                                    int dgx, int rows, int SW, int nrb, int nred, int write_red,
                                                    uint32_t* __restrict__ red, uint32_t* __restrict__ tab,
                                                    InterpPlan plan, int lcf_off, int lcf_deg, int lcg_off,
                                                    int lcg_deg, uint32_t* __restrict__ cval, uint32_t* status,
                                                    uint32_t* zero_word) {
  __shared__ Prime ps[RT_PRIMES];
  __shared__ LimbModFast kc[RT_PRIMES];
  pdl_wait();
  // the images kernel's fail counter (it runs after this grid completes): no memset node
  if (zero_word && blockIdx.x == 0 && threadIdx.x == 0) *zero_word = 0u;
  if ((int)blockIdx.x >= nred) {  // choose role
    __shared__ uint32_t lc[2 * RT_LC_MAX];
    const int pi = blockIdx.x - nred;
    const Prime P = primes[pi];
    for (int i = threadIdx.x; i <= lcf_deg + 1 + lcg_deg; i += blockDim.x) {
      const int c = i <= lcf_deg ? lcf_off + i : lcg_off + (i - lcf_deg - 1);
      lc[i] = limbs_mod(limbs + (size_t)c * L, L, P);
    }
    __syncthreads();
    choose_c_prime(P, pi, plan, lc, lcf_deg < 0 ? 0 : lcf_deg, lc + lcf_deg + 1, lcg_deg < 0 ? 0 : lcg_deg, cval,
                   status);
    return;
  }
  const int rb = blockIdx.x % nrb, side = (blockIdx.x / nrb) & 1, pg = blockIdx.x / (2 * nrb);
  const int p0 = pg * RT_PRIMES, np = min(RT_PRIMES, K - p0);
  const int TW = 2 * rows * SW;
  if (threadIdx.x < np) {
    const Prime P = primes[p0 + threadIdx.x];
    ps[threadIdx.x] = P;
    kc[threadIdx.x] = limbs_mod_fast_const(L, P);
  }
  // side 0 = A: f unless the reference swaps (deg_y g > deg_y f)
  const bool isf = (side == 0) != (m < n);
  const int deg = isf ? m : n, dx = isf ? dfx : dgx;
  const int cbase = isf ? 0 : (m + 1) * (dfx + 1);
  __syncthreads();
  const int e0 = rb * RT_ROWS;
  uint32_t* tbase = tab + (size_t)side * rows * SW + (size_t)e0 * SW;
  for (int t = threadIdx.x; t < RT_ROWS * SW; t += blockDim.x) {
    const int e = e0 + t / SW, i = t - (t / SW) * SW;
    const bool live = i <= deg && e <= dx;
    const int c = live ? cbase + (deg - i) * (dx + 1) + e : 0;
    uint32_t w[LMAX > 0 ? LMAX : 1];
    bool neg = false;
    if (LMAX > 0 && live) {
#pragma unroll
      for (int l = 0; l < LMAX; ++l) {
        w[l] = (l < L) ? limbs[(size_t)c * L + l] : 0u;
        if (l == L - 1) neg = w[l] >> 31;
      }
    }
    for (int q = 0; q < np; ++q) {
      uint32_t r = 0;
      if (live) {
        const uint32_t p = ps[q].p;
        if (LMAX > 0) {
          const LimbModFast k = kc[q];
          constexpr int NB = (LMAX + 2) / 3;  // blocks of three limbs, top block first
#pragma unroll
          for (int b = NB - 1; b >= 0; --b) {
            if (3 * b < L) {
              const uint32_t v = mod3_fast(w[3 * b], 3 * b + 1 < LMAX ? w[3 * b + 1] : 0u,
                                           3 * b + 2 < LMAX ? w[3 * b + 2] : 0u, k, p);
              r = (3 * b + 3 < L) ? add_mod(shoup(r, k.c96, k.c96c, p), v, p) : v;
            }
          }
          if (neg) r = sub_mod(r, k.big, p);
        } else {  // very wide coefficients: limbs straight from global memory
          r = limbs_mod(limbs + (size_t)c * L, L, ps[q]);
        }
        if (write_red) red[(size_t)(p0 + q) * C + c] = r;
      }
      tbase[(size_t)(p0 + q) * TW + t] = r;
    }
  }
}

bool reduce_tab_chooses(int lcf_deg, int lcg_deg) { return lcf_deg + lcg_deg + 2 <= 2 * RT_LC_MAX; }

void launch_reduce_tab(const uint32_t* limbs, int C, int L, const Prime* primes, int K, int m, int n, int dfx,
                       int dgx, uint32_t* red, uint32_t* tab, cudaStream_t st, const InterpPlan* plan, int lcf_off,
                       int lcf_deg, int lcg_off, int lcg_deg, uint32_t* cval, uint32_t* status,
                       uint32_t* zero_word) {
  const int maxd = images_maxd(m, n);
  const int dmax = dfx > dgx ? dfx : dgx;
  const int rows = POLY * (dmax / POLY + 1);  // a multiple of RT_ROWS
  const int SW = images_sw(maxd);
  const int nrb = rows / RT_ROWS;
  const int nred = ((K + RT_PRIMES - 1) / RT_PRIMES) * 2 * nrb;
  const int nch = plan ? K : 0;  // + one choose CTA per prime
  // red: for k_choose_c (no choose role) and the warp fallback kernel (CKB_FALLBACK_WARP=1)
  const int write_red = (!plan || fallback_warp()) ? 1 : 0;
  InterpPlan pl = plan ? *plan : InterpPlan{};
  const dim3 grid(nred + nch);
#define RT_LAUNCH(LM)                                                                                          \
  launch_pdl(k_reduce_tab<LM>, grid, dim3(128), 0, st, limbs, C, L, primes, K, m, n, dfx, dgx, rows, SW, nrb, \
             nred, write_red, red, tab, pl, lcf_off, lcf_deg, lcg_off, lcg_deg, cval, status, zero_word)
  if (L <= 4)
    RT_LAUNCH(4);
  else if (L <= 8)
    RT_LAUNCH(8);
  else if (L <= 16)
    RT_LAUNCH(16);
  else
    RT_LAUNCH(0);
#undef RT_LAUNCH
}

int images_maxd(int m, int n) {
  const int d = m > n ? m : n;
#define PICK(D) \
  if (d <= D) return D;
  CKB_MAXD_LIST(PICK)
#undef PICK
  return -1;
}

static size_t images_smem_bytes(int maxd, int dfx, int dgx, int NI, int K) {
  const int dmax = dfx > dgx ? dfx : dgx;
  const int rows = POLY * (dmax / POLY + 1);
  int span = (IMG_THREADS - 1 + NI - 1) / NI + 1;
  if (span > K) span = K;
  return (size_t)(span * (2 * rows * images_sw(maxd) + 2 * POLY) + 2 * rows) * 4;
}

bool images_fast_ok(int m, int n, int dfx, int dgx, int NI, int K) {
  const int maxd = images_maxd(m, n);
  return maxd > 0 && images_smem_bytes(maxd, dfx, dgx, NI, K) <= 200 * 1024;
}

// the register-heavy buckets (MAXD >= 56: ~200 registers) in prime-aligned CTAs
// of 64 images: one staged table per CTA, so registers AND shared memory allow 5
// CTAs (10 warps) per SM instead of 2 x 128 threads (8 warps).  CKB_IMG_ALIGN=0 disables.
static bool images_aligned(int maxd) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("CKB_IMG_ALIGN");
    on = e ? atoi(e) : 1;
  }
  // smaller buckets measured slower aligned (cfg4 images 270 -> 289 us: per-prime padding, no occupancy gain)
  return on && maxd >= 56;
}

// the kernel for a bucket: the exactly unrolled chains only up to MAXD 48 (at
// 56 / 64 they exceed the register file and spill; the run-time exit sweep
// measured faster there: cfg5 images 10.42 -> 9.97 ms)
#ifndef CKB_EXACT_MAXD
#define CKB_EXACT_MAXD 48
#endif
constexpr int EXACT_MAXD = CKB_EXACT_MAXD;
template <int D, int NT, bool AL>
static void (*images_kernel(int ex))(ImageArgs) {
  if (ex == 3) return k_images<D, NT, AL, 3>;
  if constexpr (D > EXACT_MAXD) {
    return k_images<D, NT, AL, 0>;
  } else {
    return ex == 1 ? k_images<D, NT, AL, 1> : ex == 2 ? k_images<D, NT, AL, 2> : k_images<D, NT, AL, 0>;
  }
}

// the exactly unrolled elimination for the dense shapes (CKB_IMG_EXACT=0 disables)
static int images_exact(int maxd, int m, int n) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("CKB_IMG_EXACT");
    on = e ? atoi(e) : 1;
  }
  if (!on) return 0;
  const int da = m > n ? m : n, db = m > n ? n : m;
  if (da != maxd || maxd > EXACT_MAXD) return 0;
  return db == maxd ? 1 : db == maxd - 1 ? 2 : 0;
}

// the failed images of the register kernel: thread per image (CKB_FALLBACK_WARP=1: the warp kernel)
static int fallback_warp() {
  static int warp = -1;
  if (warp < 0) {
    const char* e = getenv("CKB_FALLBACK_WARP");
    warp = e ? atoi(e) : 0;
  }
  return warp;
}
static void launch_fallback_reg(int maxd, const ImageArgs& a, cudaStream_t st) {
  if (fallback_warp()) return launch_images_fallback(a, st);
#define FB(D) \
  if (maxd == D) launch_pdl(k_images_fallback_reg<D>, dim3(2 * 148), dim3(128), 0, st, a);
  CKB_MAXD_LIST(FB)
#undef FB
}

void launch_images(const ImageArgs& a, cudaStream_t st, bool structured) {
  const int maxd = images_maxd(a.m, a.n);
  int ex = structured ? 3 : images_exact(maxd, a.m, a.n);
  // below ~2.5 warps of images per scheduler (one prime shard of cfg4 at 8 GPUs) the
  // unrolled chains stall on instruction fetch (ncu: 4.4 no-instruction stalls per
  // issue at 8 warps/SM); the compact exit sweeps measured faster there (68 -> 62 us)
  if (ex == 1 || ex == 2) {
    const double warps = (double)a.K * a.N / 32.0;
    // (buckets <= 24 keep it: their chains are short enough for the instruction
    // cache -- cfg2, bucket 20 at one warp per scheduler: images 23.0 -> 21.2 us)
    if (warps < 2.5 * 148 * 4 && maxd > 24) ex = 0;
  }
  if (images_aligned(maxd)) {
    constexpr int NTA = 64;
    ImageArgs b = a;
    b.span = 1;
    const dim3 grid((unsigned)((a.N + NTA - 1) / NTA), (unsigned)a.K);
    const int dmax = a.dfx > a.dgx ? a.dfx : a.dgx;
    const int rows = POLY * (dmax / POLY + 1);
#define LAUNCH_AL(D)                                                                                     \
  if (maxd == D) {                                                                                       \
    const size_t smem = (size_t)((2 * rows * ImgLayout<D>::SW + 2 * POLY) + 2 * rows) * 4;              \
    auto kern = images_kernel<D, NTA, true>(ex);                                                         \
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    launch_pdl(kern, grid, dim3(NTA), smem, st, b);                                                      \
  }
    LAUNCH_AL(56) LAUNCH_AL(64)
#undef LAUNCH_AL
    launch_fallback_reg(maxd, a, st);
    return;
  }
  dim3 grid((unsigned)(((size_t)a.K * a.N + IMG_THREADS - 1) / IMG_THREADS));
  ImageArgs b = a;
  b.span = (IMG_THREADS - 1 + a.N - 1) / a.N + 1;  // primes a window of IMG_THREADS images can touch
  if (b.span > a.K) b.span = a.K;
  const int dmax = a.dfx > a.dgx ? a.dfx : a.dgx;
  const int rows = POLY * (dmax / POLY + 1);
#define LAUNCH(D)                                                                                    \
  if (maxd == D) {                                                                                   \
    const size_t smem = (size_t)(b.span * (2 * rows * ImgLayout<D>::SW + 2 * POLY) + 2 * rows) * 4; \
    auto kern = images_kernel<D, IMG_THREADS, false>(ex);                                            \
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    launch_pdl(kern, grid, dim3(IMG_THREADS), smem, st, b);                                          \
  }
  CKB_MAXD_LIST(LAUNCH)
#undef LAUNCH
  launch_fallback_reg(maxd, a, st);
}

}  // namespace ckb

// K2+K3 with TWO lanes per image ("paired lanes"), for launches too small to
// fill the machine: below ~3 warps of images per scheduler (cfg2, cfg3, the
// per-rank share of cfg4 at 4-8 GPUs) a warp's elimination chain is latency
// bound -- at 8 ranks cfg4's 38,600 images leave ~2 warps per scheduler and take
// 68 us for 1/8 of the work one GPU does in 242 us.  Splitting every image over
// two lanes doubles the warps and halves each warp's chain.
//
// Same algorithm and outputs as k_images (ckb_images.cu: polyphase Horner +
// 8-point DFT per coset, the fused division-free remainder sequence of
// ckb_resultant.cuh, exact trip counts).  Lane layout in a warp: bit 4 = parity
// `par`, bit 3 = coset group, bits 0-2 = polyphase lane l; a warp holds 16
// images (2 cosets).  Lane `par` keeps the top-aligned coefficients of even
// (par 0) or odd (par 1) index: local t <-> global i = 2t + par.  In the fused
// update D''[i] = w1 D[i+2] + w2 V[i+2] + w3 V[i+1] the first two operands have
// i's parity (own registers) and V[i+1] the other one: one shuffle with the
// partner lane (lane ^ 16) per output.  The leading coefficients (i = 0, 1) are
// exchanged the same way; the bookkeeping runs redundantly in both lanes.
#include "ckb_kernels.cuh"
#include "ckb_resultant.cuh"
#include "ckb_ntt.cuh"
#include "ckb_images.cuh"

namespace ckb {

namespace {
constexpr unsigned FULLM = 0xffffffffu;

// the value of x held by the pair's par-0 / par-1 lane (every lane executes the shuffle)
__device__ __forceinline__ uint32_t from_par(uint32_t x, int par, int want) {
  const uint32_t o = __shfl_xor_sync(FULLM, x, 16);
  return par == want ? x : o;
}

// single step D <- lb D - lc(D) V (global D[i] = lb D[i+1] - la V[i+1]); both
// operands of output i have the other parity: two shuffles per output
template <int H>
__device__ __forceinline__ void step1_pair(uint32_t (&D)[H], const uint32_t (&V)[H], int nom, uint32_t lb,
                                           uint32_t lbc, const Prime& P, int par) {
  const uint32_t p = P.p;
  const uint32_t la = red4(from_par(D[0], par, 0), p);
  const uint32_t nla = la ? p - la : 0u;
  const uint32_t nlac = comp_from_mont(to_mont(nla, P), P);
#pragma unroll
  for (int t = 0; t < H - 1; ++t) {
    if (2 * t <= nom + 1) {
      // partner's D / V at global i + 1 = 2t + par + 1: its local t + par; it sends its local t + 1 - par
      const uint32_t dp = __shfl_xor_sync(FULLM, par ? D[t] : D[t + 1], 16);
      const uint32_t vp = __shfl_xor_sync(FULLM, par ? V[t] : V[t + 1], 16);
      D[t] = shoup_lazy(dp, lb, lbc, p) + shoup_lazy(vp, nla, nlac, p);
    }
  }
  D[H - 1] = 0u;  // global MAXD (par 0) and MAXD + 1 (par 1)
}

// the fused generic remainder (ckb_resultant.cuh step2) on paired lanes; returns lc(V)
template <int H>
__device__ __forceinline__ void pair_multipliers(const uint32_t (&D)[H], const uint32_t (&V)[H], const Prime& P,
                                                 int par, uint32_t& lb, uint32_t& w1m, uint32_t& w2m,
                                                 uint32_t& w3m) {
  const uint32_t p = P.p;
  lb = red4(from_par(V[0], par, 0), p);
  const uint32_t la = red4(from_par(D[0], par, 0), p);
  const uint32_t d1 = red4(from_par(D[0], par, 1), p), v1 = red4(from_par(V[0], par, 1), p);
  const uint32_t nla = la ? p - la : 0u;
  w1m = redc((uint64_t)lb * lb, P);
  w2m = redc((uint64_t)lb * nla, P);
  const uint32_t l3 = redc((uint64_t)lb * d1 + (uint64_t)nla * v1, P);
  w3m = l3 ? p - l3 : 0u;
}

// compile-time divisor degree K: outputs i < K, then global entries K and K + 1 zeroed
template <int H, int K>
__device__ __forceinline__ uint32_t step2_pair_exact(uint32_t (&D)[H], const uint32_t (&V)[H], const Prime& P,
                                                     int par) {
  uint32_t lb, w1m, w2m, w3m;
  pair_multipliers<H>(D, V, P, par, lb, w1m, w2m, w3m);
  const uint32_t pinv = P.pinv, p = P.p;
#pragma unroll
  for (int t = 0; t < (K + 1) / 2; ++t) {
    if (t + 1 < H) {
      const uint32_t vp = __shfl_xor_sync(FULLM, par ? V[t] : V[t + 1], 16);  // global V[i + 1]
      if (2 * t + 1 < K || par == 0) D[t] = mont3(D[t + 1], w1m, V[t + 1], w2m, vp, w3m, pinv, p);
    }
  }
  // global K and K + 1: local K/2 in the lane of K's parity, (K+1)/2 in the other
  if ((K >> 1) < H && par == (K & 1)) D[K >> 1] = 0u;
  if (((K + 1) >> 1) < H && par == ((K + 1) & 1)) D[(K + 1) >> 1] = 0u;
  return lb;
}

// run-time divisor degree k: outputs while 2T + par < k, then global D[k] zeroed
template <int H, int T>
__device__ __forceinline__ void sweep_pair(uint32_t (&D)[H], const uint32_t (&V)[H], int k, uint32_t w1m,
                                           uint32_t w2m, uint32_t w3m, const Prime& P, int par) {
  if constexpr (T < H) {
    if (2 * T >= k) {  // uniform: k depends on the launch's degrees only
      if (k & 1) {
        if (par) D[T - 1] = 0u;  // global k = 2T - 1
      } else if (!par) {
        D[T] = 0u;               // global k = 2T
      }
    } else {
      if constexpr (T + 1 < H) {
        const uint32_t vp = __shfl_xor_sync(FULLM, par ? V[T] : V[T + 1], 16);
        if (2 * T + par < k) D[T] = mont3(D[T + 1], w1m, V[T + 1], w2m, vp, w3m, P.pinv, P.p);
      }
      sweep_pair<H, T + 1>(D, V, k, w1m, w2m, w3m, P, par);
    }
  }
}

template <int H>
__device__ __forceinline__ uint32_t step2_pair_run(uint32_t (&D)[H], const uint32_t (&V)[H], int k, const Prime& P,
                                                   int par) {
  uint32_t lb, w1m, w2m, w3m;
  pair_multipliers<H>(D, V, P, par, lb, w1m, w2m, w3m);
  sweep_pair<H, 0>(D, V, k, w1m, w2m, w3m, P, par);
  return lb;
}

template <int H, int K, bool BA>
__device__ __forceinline__ void chain_pair(uint32_t (&A)[H], uint32_t (&B)[H], uint32_t& T, uint32_t& Q,
                                           uint32_t& num, bool& bad, const Prime& P, int par) {
  if constexpr (K >= 1) {
    const uint32_t lm = BA ? step2_pair_exact<H, K>(B, A, P, par) : step2_pair_exact<H, K>(A, B, P, par);
    T = mmul(T, lm, P);
    Q = mmul(Q, T, P);
    const uint32_t d0 = red4(from_par(BA ? B[0] : A[0], par, 0), P.p);
    bad |= (d0 == 0u);
    if constexpr (K == 1) {
      num = mmul(num, to_mont(d0, P), P);
    } else {
      chain_pair<H, K - 1, !BA>(A, B, T, Q, num, bad, P, par);
    }
  }
}

// resultant_generic (ckb_resultant.cuh) on paired lanes; DB > 0: db == DB unrolled
template <int MAXD, int DB>
__device__ __forceinline__ uint32_t resultant_pair(uint32_t (&A)[MAXD / 2 + 1], int da, uint32_t (&B)[MAXD / 2 + 1],
                                                   int db, bool neg, const Prime& P, int par) {
  constexpr int H = MAXD / 2 + 1;
  const uint32_t p = P.p;
  const uint32_t one = redc(P.r2, P);
  const uint32_t lb = red4(from_par(B[0], par, 0), p);
  const uint32_t lbm = to_mont(lb, P);
  const uint32_t lbc = comp_from_mont(lbm, P);
  bool bad = false;
  const int e0 = da - db + 1;
  for (int s = 0; s < e0; ++s) step1_pair<H>(A, B, da - s, lb, lbc, P, par);
  uint32_t a0 = red4(from_par(A[0], par, 0), p);
  bad |= (a0 == 0u);
  neg ^= (bool)(da & db & 1);
  const uint32_t l1e = mpow(lbm, e0, one, P);
  uint32_t num = l1e, den = mpow(l1e, db, one, P);
  uint32_t T = one, Q = one;
  int k = db - 1;
  if (k == 0) {
    num = mmul(num, to_mont(a0, P), P);
  } else if constexpr (DB > 1) {
    chain_pair<H, DB - 1, true>(A, B, T, Q, num, bad, P, par);
    num = mmul(num, mmul(T, T, P), P);
    den = mmul(den, mmul(Q, Q, P), P);
  } else {
    for (;;) {
      uint32_t lm = step2_pair_run<H>(B, A, k, P, par);
      T = mmul(T, lm, P);
      Q = mmul(Q, T, P);
      --k;
      const uint32_t b0 = red4(from_par(B[0], par, 0), p);
      bad |= (b0 == 0u);
      if (k == 0) {
        num = mmul(num, to_mont(b0, P), P);
        break;
      }
      lm = step2_pair_run<H>(A, B, k, P, par);
      T = mmul(T, lm, P);
      Q = mmul(Q, T, P);
      --k;
      a0 = red4(from_par(A[0], par, 0), p);
      bad |= (a0 == 0u);
      if (k == 0) {
        num = mmul(num, to_mont(a0, P), P);
        break;
      }
    }
    num = mmul(num, mmul(T, T, P), P);
    den = mmul(den, mmul(Q, Q, P), P);
  }
  if (bad) return CKB_FAIL;
  const uint32_t corr = mpow(P.r2, 2 * (db - 1), one, P);
  uint32_t inv = one, b = den;
  uint32_t ex = p - 2;
  while (ex) {
    if (ex & 1) inv = mmul(inv, b, P);
    ex >>= 1;
    if (ex) b = mmul(b, b, P);
  }
  const uint32_t r = redc((uint64_t)mmul(mmul(num, inv, P), corr, P), P);
  return neg ? neg_mod(r, p) : r;
}
}  // namespace

#ifndef CKB_PAIR_MINB
#define CKB_PAIR_MINB 4
#endif
constexpr int PAIR_NT = 128;       // threads per CTA
constexpr int PAIR_IMG = PAIR_NT / 2;  // images per CTA

// EX: 0 run-time exit sweeps (any degrees); 1 da = db = MAXD; 2 da = MAXD, db = MAXD - 1 (unrolled chains)
template <int MAXD, int EX>
__global__ void __launch_bounds__(PAIR_NT, CKB_PAIR_MINB) k_images_pair(ImageArgs a) {
  constexpr int H = MAXD / 2 + 1;
  using LY = ImgLayout<MAXD>;
  constexpr int NCH = LY::NCH, SW = LY::SW;
  extern __shared__ __align__(16) uint32_t sm[];
  const bool sw = a.m < a.n;
  const int da = sw ? a.n : a.m, db = sw ? a.m : a.n;
  const int16_t* Adeg = a.degs + (sw ? a.m + 1 : 0);
  const int16_t* Bdeg = a.degs + (sw ? 0 : a.m + 1);
  const int dmax = max(a.dfx, a.dgx);
  const int emax = dmax / POLY;
  const int rows = POLY * (emax + 1);
  const int TW = 2 * rows * SW;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int par = lane >> 4, grp = (lane >> 3) & 1, l = lane & 7;
  const int g0 = blockIdx.x * PAIR_IMG;
  const int total = a.K * a.N;
  const int pi0 = g0 / a.N;
  const int pi1 = min(a.K - 1, (g0 + PAIR_IMG - 1) / a.N);
  const int t = g0 + warp * 16 + grp * 8 + l;  // this lane's image slot (before the DFT permutation)
  const bool active = t < total;
  const int pi = active ? t / a.N : pi1;
  const int tin = active ? t - pi * a.N : 0;
  const int u = tin >> 3;
  const int tslot = pi - pi0;
  const Prime P = a.primes[pi];
  uint32_t y = a.yq[(size_t)pi * a.M + u];
  uint32_t* TA = sm + tslot * TW;
  uint32_t* TB = TA + rows * SW;
  const int nspan = pi1 - pi0 + 1;
  uint32_t* maskA = sm + a.span * TW;
  uint32_t* maskB = maskA + rows;
  uint32_t* som = maskB + rows + tslot * 2 * POLY;
  __shared__ __align__(8) uint64_t tab_bar;
  const uint32_t bar = img_smem_u32(&tab_bar);
  if (threadIdx.x == 0) {
    img_mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  pdl_wait();
  if (threadIdx.x == 0) {
    const uint32_t bytes = (uint32_t)(nspan * TW) * 4u;
    img_mbar_expect_tx(bar, bytes);
    img_bulk_g2s(img_smem_u32(sm), a.tab + (size_t)pi0 * TW, bytes, bar);
  }
  for (int e = threadIdx.x; e < rows; e += PAIR_NT) {
    uint32_t ma = 0, mb = 0;
    for (int i = 0; i <= MAXD; ++i) {
      if (i <= da && Adeg[da - i] >= e) ma |= 1u << (i >> 2);
      if (i <= db && Bdeg[db - i] >= e) mb |= 1u << (i >> 2);
    }
    maskA[e] = ma;
    maskB[e] = mb;
  }
  for (int q = threadIdx.x; q < nspan * 2 * POLY; q += PAIR_NT)
    maskB[rows + q] = a.om[(size_t)(pi0 + q / (2 * POLY)) * 4 * POLY + q % (2 * POLY)];

  const uint32_t c = a.cval[pi];
  const uint32_t p = P.p;
  if (c != 1u) y = shoup(y, c, shoup_comp(c, P), p);
  const uint32_t y2 = mul_mod(y, y, P), y4 = mul_mod(y2, y2, P);
  const uint32_t z = mul_mod(y4, y4, P);
  __syncthreads();
  img_mbar_wait(bar, 0);
  uint32_t yl = (l & 1) ? y : 1u;
  if (l & 2) yl = mul_mod(yl, y2, P);
  if (l & 4) yl = mul_mod(yl, y4, P);
  const uint32_t zc = comp_from_mont(to_mont(z, P), P);

  // Horner in z: this lane's parity of every chunk of 4 top-aligned entries
  // (entries 4c + par and 4c + par + 2 -> local 2c and 2c + 1)
  uint32_t A[H], B[H];
#pragma unroll
  for (int i = 0; i < H; ++i) A[i] = B[i] = 0u;
  uint32_t negp = 0u - p;
  uint32_t zcp = zc;
  asm volatile("" : "+r"(negp), "+r"(zcp));
  {
    const int e = l + POLY * emax;
    const uint4* ta = reinterpret_cast<const uint4*>(TA + e * SW);
    const uint4* tb = reinterpret_cast<const uint4*>(TB + e * SW);
    const uint32_t mA = __reduce_or_sync(FULLM, maskA[e]);
    const uint32_t mB = __reduce_or_sync(FULLM, maskB[e]);
#pragma unroll
    for (int cc = 0; cc < NCH; ++cc) {
      if (mA & (1u << cc)) {
        const uint4 v = ta[cc];
        if (2 * cc < H) A[2 * cc] = par ? v.y : v.x;
        if (2 * cc + 1 < H) A[2 * cc + 1] = par ? v.w : v.z;
      }
      if (mB & (1u << cc)) {
        const uint4 v = tb[cc];
        if (2 * cc < H) B[2 * cc] = par ? v.y : v.x;
        if (2 * cc + 1 < H) B[2 * cc + 1] = par ? v.w : v.z;
      }
    }
  }
  for (int e2 = emax - 1; e2 >= 0; --e2) {
    const int e = l + POLY * e2;
    const uint4* ta = reinterpret_cast<const uint4*>(TA + e * SW);
    const uint4* tb = reinterpret_cast<const uint4*>(TB + e * SW);
    const uint32_t mA = __reduce_or_sync(FULLM, maskA[e]);
    const uint32_t mB = __reduce_or_sync(FULLM, maskB[e]);
#pragma unroll
    for (int cc = 0; cc < NCH; ++cc) {
      if (mA & (1u << cc)) {
        const uint4 v = ta[cc];
        if (2 * cc < H) A[2 * cc] = shoup_lazy_add(A[2 * cc], z, zcp, negp, par ? v.y : v.x);
        if (2 * cc + 1 < H) A[2 * cc + 1] = shoup_lazy_add(A[2 * cc + 1], z, zcp, negp, par ? v.w : v.z);
      }
      if (mB & (1u << cc)) {
        const uint4 v = tb[cc];
        if (2 * cc < H) B[2 * cc] = shoup_lazy_add(B[2 * cc], z, zcp, negp, par ? v.y : v.x);
        if (2 * cc + 1 < H) B[2 * cc + 1] = shoup_lazy_add(B[2 * cc + 1], z, zcp, negp, par ? v.w : v.z);
      }
    }
  }
  {
    const uint32_t ylc = comp_from_mont(to_mont(yl, P), P);
#pragma unroll
    for (int i = 0; i < H; ++i) {
      A[i] = shoup_lazy(A[i], yl, ylc, p);
      B[i] = shoup_lazy(B[i], yl, ylc, p);
    }
  }
  const uint32_t p2 = 2u * p;
#pragma unroll
  for (int h = POLY / 2; h >= 1; h >>= 1) {
    const bool upper = (l & h) != 0;
    const int widx = (l & (h - 1)) * (POLY / (2 * h));
    if (h > 1) {
      const uint32_t wp = som[widx], wpc = som[POLY + widx];
#pragma unroll
      for (int i = 0; i < H; ++i) {
        const uint32_t recv = __shfl_xor_sync(FULLM, upper ? A[i] : B[i], h);
        const uint32_t lo = upper ? recv : A[i], hi = upper ? B[i] : recv;
        const uint32_t sum = red2p(lo + hi, p2);
        const uint32_t dif = shoup_lazy(lo - hi + p2, wp, wpc, p);
        const uint32_t recv2 = __shfl_xor_sync(FULLM, upper ? sum : dif, h);
        A[i] = upper ? recv2 : sum;
        B[i] = upper ? dif : recv2;
      }
      continue;
    }
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const uint32_t oa = __shfl_xor_sync(FULLM, A[i], h), ob = __shfl_xor_sync(FULLM, B[i], h);
      const uint32_t da_ = oa - A[i], db_ = ob - B[i];
      A[i] = upper ? min(da_, da_ + p2) : A[i] + oa;
      B[i] = upper ? min(db_, db_ + p2) : B[i] + ob;
    }
  }
  // the global entry MAXD + 1 (par 1's last local) is outside the arrays: zero
  if (par) {
    A[H - 1] = 0u;
    B[H - 1] = 0u;
  }
  const int j = ((l & 1) << 2) | (l & 2) | ((l >> 2) & 1);
  const int idx = u * POLY + j;
  // every lane of the warp takes part in the elimination's shuffles (inactive
  // slots compute on zeros and write nothing)
  // (no branch around the elimination: its shuffles need every lane of the warp, and
  // an inactive slot or a vanishing leading coefficient just computes on and is dropped)
  const uint32_t a0 = red4(from_par(A[0], par, 0), p), b0 = red4(from_par(B[0], par, 0), p);
  const bool neg = sw && ((a.m * a.n) & 1);
  uint32_t v;
  if constexpr (EX == 1)
    v = resultant_pair<MAXD, MAXD>(A, da, B, db, neg, P, par);
  else if constexpr (EX == 2)
    v = resultant_pair<MAXD, MAXD - 1>(A, da, B, db, neg, P, par);
  else
    v = resultant_pair<MAXD, 0>(A, da, B, db, neg, P, par);
  if (!active || par) return;
  if (a0 == 0u || b0 == 0u) {
    atomicOr(a.status, 2u);  // the plan guarantees this never happens
    v = 0u;
  } else if (v == CKB_FAIL) {
    const uint32_t slot = atomicAdd(a.fail_count, 1u);
    a.fail_list[slot] = (uint32_t)((size_t)pi * a.N + idx);
    v = 0u;
  }
  a.values[(size_t)pi * a.N + idx] = v;
}

size_t images_pair_smem(int maxd_sw, int rows, int span) {
  return (size_t)(span * (2 * rows * maxd_sw + 2 * POLY) + 2 * rows) * 4;
}

// the paired-lane launch for the bucket maxd (EX as in k_images; the caller
// checked images_fast_ok and launches the fallback afterwards)
bool launch_images_pair(int maxd, int ex, const ImageArgs& a0, cudaStream_t st) {
  ImageArgs a = a0;
  a.span = (PAIR_IMG - 1 + a.N - 1) / a.N + 1;
  if (a.span > a.K) a.span = a.K;
  const int dmax = a.dfx > a.dgx ? a.dfx : a.dgx;
  const int rows = POLY * (dmax / POLY + 1);
  const dim3 grid((unsigned)(((size_t)a.K * a.N + PAIR_IMG - 1) / PAIR_IMG));
#define PAIR_LAUNCH(D)                                                                                   \
  if (maxd == D) {                                                                                       \
    const size_t smem = images_pair_smem(ImgLayout<D>::SW, rows, a.span);                                \
    auto kern = ex == 1 ? k_images_pair<D, 1> : ex == 2 ? k_images_pair<D, 2> : k_images_pair<D, 0>;    \
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    launch_pdl(kern, grid, dim3(PAIR_NT), smem, st, a);                                                  \
    return true;                                                                                          \
  }
  PAIR_LAUNCH(8) PAIR_LAUNCH(12) PAIR_LAUNCH(16) PAIR_LAUNCH(24) PAIR_LAUNCH(32) PAIR_LAUNCH(40) PAIR_LAUNCH(48)
#undef PAIR_LAUNCH
  return false;
}

}  // namespace ckb

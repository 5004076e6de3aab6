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
#include "ckb_kernels.cuh"
#include "ckb_resultant.cuh"

namespace ckb {

constexpr int IMG_THREADS = 128;

// shared-memory row width of the transposed, top-aligned residue tables
template <int MAXD>
struct ImgLayout {
  static constexpr int NCH = (MAXD + 4) / 4;  // chunks of 4 registers
  static constexpr int SW = NCH * 4;          // words per x-power row
};

template <int MAXD>
__global__ void __launch_bounds__(IMG_THREADS) k_images(ImageArgs a) {
  using LY = ImgLayout<MAXD>;
  constexpr int NCH = LY::NCH, SW = LY::SW;
  extern __shared__ __align__(16) uint32_t sm[];
  const int pi = blockIdx.y;
  const bool sw = a.m < a.n;  // reference swaps so that deg a >= deg b
  const int da = sw ? a.n : a.m, db = sw ? a.m : a.n;
  const int offF = 0, offG = (a.m + 1) * (a.dfx + 1);
  const int offA = sw ? offG : offF, offB = sw ? offF : offG;
  const int Astr = sw ? a.dgx + 1 : a.dfx + 1, Bstr = sw ? a.dfx + 1 : a.dgx + 1;
  const int16_t* Adeg = a.degs + (sw ? a.m + 1 : 0);
  const int16_t* Bdeg = a.degs + (sw ? 0 : a.m + 1);
  const int dmax = max(a.dfx, a.dgx);
  // TA[e][i] = coefficient of x^e in the y-coefficient of degree da - i (top-aligned),
  // zero beyond each row; maskA[e] = chunks of registers with a term at x^e
  uint32_t* TA = sm;
  uint32_t* TB = sm + (dmax + 1) * SW;
  uint32_t* maskA = sm + 2 * (dmax + 1) * SW;
  uint32_t* maskB = maskA + (dmax + 1);
  const uint32_t* gres = a.red + (size_t)pi * a.C;
  for (int idx = threadIdx.x; idx < (dmax + 1) * SW; idx += IMG_THREADS) {
    const int e = idx / SW, i = idx % SW;
    TA[idx] = (i <= da && e < Astr) ? gres[offA + (da - i) * Astr + e] : 0u;
    TB[idx] = (i <= db && e < Bstr) ? gres[offB + (db - i) * Bstr + e] : 0u;
  }
  for (int e = threadIdx.x; e <= dmax; e += IMG_THREADS) {
    uint32_t ma = 0, mb = 0;
    for (int i = 0; i <= MAXD; ++i) {
      if (i <= da && Adeg[da - i] >= e) ma |= 1u << (i >> 2);
      if (i <= db && Bdeg[db - i] >= e) mb |= 1u << (i >> 2);
    }
    maskA[e] = ma;
    maskB[e] = mb;
  }
  __syncthreads();

  const int t = blockIdx.x * IMG_THREADS + threadIdx.x;
  if (t >= a.N) return;
  const Prime P = a.primes[pi];
  const uint32_t p = P.p;
  const uint32_t c = a.cval[pi];
  uint32_t x = a.xq[(size_t)pi * a.N + t];
  if (c != 1u) x = shoup(x, c, shoup_comp(c, P), p);  // x_t = c q^t
  const uint32_t xc = comp_from_mont(to_mont(x, P), P);

  // Horner of all y-coefficients in lock-step: one dynamic loop over the x
  // power, every register an independent chain (ILP = m + n + 2); each chunk
  // of 4 coefficients is one 16-byte broadcast load.  A chain that has not
  // started yet multiplies 0, so the masks only skip work.
  uint32_t A[MAXD + 1], B[MAXD + 1];
#pragma unroll
  for (int i = 0; i <= MAXD; ++i) A[i] = B[i] = 0u;
  uint32_t negp = 0u - p;
  uint32_t xcp = xc;
  // opaque to the optimiser: keeps both in registers instead of letting
  // ptxas rematerialise the companion (7 instructions) in every chunk
  asm volatile("" : "+r"(negp), "+r"(xcp));
  for (int e = dmax; e >= 0; --e) {
    const uint4* ta = reinterpret_cast<const uint4*>(TA + e * SW);
    const uint4* tb = reinterpret_cast<const uint4*>(TB + e * SW);
    const uint32_t mA = maskA[e], mB = maskB[e];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      if (mA & (1u << c)) {
        const uint4 v = ta[c];
        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (4 * c + k <= MAXD) A[4 * c + k] = shoup_lazy_add(A[4 * c + k], x, xcp, negp, vv[k]);
      }
      if (mB & (1u << c)) {
        const uint4 v = tb[c];
        const uint32_t vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (4 * c + k <= MAXD) B[4 * c + k] = shoup_lazy_add(B[4 * c + k], x, xcp, negp, vv[k]);
      }
    }
  }
  uint32_t v;
  if (red4(A[0], p) == 0u || red4(B[0], p) == 0u) {
    atomicOr(a.status, 2u);  // the plan guarantees this never happens
    v = 0u;
  } else {
    const bool neg = sw && ((a.m * a.n) & 1);
    v = resultant_generic<MAXD>(A, da, B, db, neg, P);
    if (v == CKB_FAIL) {
      const uint32_t slot = atomicAdd(a.fail_count, 1u);
      a.fail_list[slot] = (uint32_t)((size_t)pi * a.N + t);
      v = 0u;
    }
  }
  a.values[(size_t)pi * a.N + t] = v;
}

#define CKB_MAXD_LIST(X) X(4) X(8) X(12) X(16) X(24) X(32) X(40) X(48) X(56) X(64)

int images_maxd(int m, int n) {
  const int d = m > n ? m : n;
#define PICK(D) \
  if (d <= D) return D;
  CKB_MAXD_LIST(PICK)
#undef PICK
  return -1;
}

void launch_images(const ImageArgs& a, cudaStream_t st) {
  const int maxd = images_maxd(a.m, a.n);
  dim3 grid((a.N + IMG_THREADS - 1) / IMG_THREADS, a.K);
  const int dmax = a.dfx > a.dgx ? a.dfx : a.dgx;
#define LAUNCH(D)                                                                                    \
  if (maxd == D) {                                                                                   \
    const size_t smem = (size_t)(2 * (dmax + 1) * ImgLayout<D>::SW + 2 * (dmax + 1)) * 4;          \
    if (smem > 48 * 1024)                                                                            \
      cudaFuncSetAttribute(k_images<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
    k_images<D><<<grid, IMG_THREADS, smem, st>>>(a);                                                 \
  }
  CKB_MAXD_LIST(LAUNCH)
#undef LAUNCH
  launch_images_fallback(a, st);
}

}  // namespace ckb

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

template <int MAXD>
__global__ void __launch_bounds__(IMG_THREADS) k_images(ImageArgs a) {
  extern __shared__ uint32_t sm[];
  const int pi = blockIdx.y;
  uint32_t* sres = sm;                                  // C residues
  int* sdeg = reinterpret_cast<int*>(sm + a.C);          // (m+1)+(n+1) degrees
  const uint32_t* gres = a.red + (size_t)pi * a.C;
  for (int i = threadIdx.x; i < a.C; i += IMG_THREADS) sres[i] = gres[i];
  const int nd = a.m + a.n + 2;
  for (int i = threadIdx.x; i < nd; i += IMG_THREADS) sdeg[i] = a.degs[i];
  __syncthreads();

  const int t = blockIdx.x * IMG_THREADS + threadIdx.x;
  if (t >= a.N) return;
  const Prime P = a.primes[pi];
  const uint32_t p = P.p;
  const uint32_t x = a.xpts[(size_t)pi * a.N + t];
  const uint32_t xc = comp_from_mont(to_mont(x, P), P);

  const bool sw = a.m < a.n;  // reference swaps so that deg a >= deg b
  const int da = sw ? a.n : a.m, db = sw ? a.m : a.n;
  const int offF = 0, offG = (a.m + 1) * (a.dfx + 1);
  const uint32_t* Ares = sres + (sw ? offG : offF);
  const uint32_t* Bres = sres + (sw ? offF : offG);
  const int Astr = sw ? a.dgx + 1 : a.dfx + 1, Bstr = sw ? a.dfx + 1 : a.dgx + 1;
  const int* Adeg = sdeg + (sw ? a.m + 1 : 0);
  const int* Bdeg = sdeg + (sw ? 0 : a.m + 1);

  // Horner of all y-coefficients in lock-step: one dynamic loop over the x
  // power, every register an independent chain (ILP = m + n + 2).  Rows are
  // zero-padded to their common length, so a chain that has not started yet
  // stays 0; the per-chunk max-degree guards only skip work.
  constexpr int NCH = (MAXD + 4) / 4;
  int cmA[NCH], cmB[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    int ma = -1, mb = -1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = 4 * c + k;
      if (i <= da) ma = max(ma, Adeg[da - i]);
      if (i <= db) mb = max(mb, Bdeg[db - i]);
    }
    cmA[c] = ma;
    cmB[c] = mb;
  }
  uint32_t A[MAXD + 1], B[MAXD + 1];
#pragma unroll
  for (int i = 0; i <= MAXD; ++i) A[i] = B[i] = 0u;
  const int dmax = max(sw ? a.dgx : a.dfx, sw ? a.dfx : a.dgx);
  for (int e = dmax; e >= 0; --e) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      if (cmA[c] >= e) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int i = 4 * c + k;
          if (i <= MAXD && i <= da) A[i] = shoup_lazy(A[i], x, xc, p) + Ares[(da - i) * Astr + e];
        }
      }
      if (cmB[c] >= e) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int i = 4 * c + k;
          if (i <= MAXD && i <= db) B[i] = shoup_lazy(B[i], x, xc, p) + Bres[(db - i) * Bstr + e];
        }
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
  const size_t smem = (size_t)(a.C + a.m + a.n + 2) * 4;
#define LAUNCH(D)                                                                                    \
  if (maxd == D) {                                                                                   \
    if (smem > 48 * 1024)                                                                            \
      cudaFuncSetAttribute(k_images<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);     \
    k_images<D><<<grid, IMG_THREADS, smem, st>>>(a);                                                 \
  }
  CKB_MAXD_LIST(LAUNCH)
#undef LAUNCH
  launch_images_fallback(a, st);
}

}  // namespace ckb

// K2+K3: fused evaluation homomorphism + univariate resultant, one thread per
// (prime, point) image.  Restates the reference's inner loop
// (pkg/src/curvekit/modpoly.py:382-390: _zp_eval of every y-coefficient at t,
// then _zp_resultant of the two univariate images) with:
//   * the prime's residue coefficients staged once per CTA in shared memory
//     (all threads of a CTA share the prime; reads are warp broadcasts),
//   * Shoup-Horner evaluation straight into top-aligned registers,
//   * the division-free elimination of ckb_resultant.cuh (no inverse in the
//     loop; one Fermat inverse per image).
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
  const uint32_t xc = shoup_comp(x, P);

  const bool sw = a.m < a.n;  // reference swaps so that deg a >= deg b
  const int da = sw ? a.n : a.m, db = sw ? a.m : a.n;
  const int offF = 0, offG = (a.m + 1) * (a.dfx + 1);
  const uint32_t* Ares = sres + (sw ? offG : offF);
  const uint32_t* Bres = sres + (sw ? offF : offG);
  const int Astr = sw ? a.dgx + 1 : a.dfx + 1, Bstr = sw ? a.dfx + 1 : a.dgx + 1;
  const int* Adeg = sdeg + (sw ? a.m + 1 : 0);
  const int* Bdeg = sdeg + (sw ? 0 : a.m + 1);

  uint32_t A[MAXD + 1], B[MAXD + 1];
#pragma unroll
  for (int i = 0; i <= MAXD; ++i) {
    A[i] = (i <= da) ? horner(Ares + (da - i) * Astr, Adeg[da - i], x, xc, p) : 0u;
    B[i] = (i <= db) ? horner(Bres + (db - i) * Bstr, Bdeg[db - i], x, xc, p) : 0u;
  }
  uint32_t v;
  if (A[0] == 0u || B[0] == 0u) {
    atomicOr(a.status, 2u);  // the plan guarantees this never happens
    v = 0u;
  } else {
    const bool neg = sw && ((a.m * a.n) & 1);
    v = resultant_topaligned<MAXD>(A, da, B, db, neg, P);
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
#define LAUNCH(D)                                                                          \
  if (maxd == D) {                                                                         \
    if (smem > 48 * 1024)                                                                  \
      cudaFuncSetAttribute(k_images<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
    k_images<D><<<grid, IMG_THREADS, smem, st>>>(a);                                       \
    return;                                                                                \
  }
  CKB_MAXD_LIST(LAUNCH)
#undef LAUNCH
}

// ---------------------------------------------------------------------------
// batch of independent univariate resultants (zp_resultant_uni, modpoly.py:156)
// ---------------------------------------------------------------------------
template <int MAXD>
__global__ void __launch_bounds__(IMG_THREADS) k_uni_resultant(const uint32_t* __restrict__ fa,
                                                              const int32_t* __restrict__ da_,
                                                              const uint32_t* __restrict__ gb,
                                                              const int32_t* __restrict__ db_, int W,
                                                              const Prime* __restrict__ primes,
                                                              const int32_t* __restrict__ pidx, int Bn,
                                                              uint32_t* __restrict__ out) {
  const int b = blockIdx.x * IMG_THREADS + threadIdx.x;
  if (b >= Bn) return;
  const Prime P = primes[pidx[b]];
  int da = da_[b], db = db_[b];
  if (da < 0 || db < 0) {  // a zero polynomial (modpoly.py:135-136)
    out[b] = 0u;
    return;
  }
  const uint32_t* fp = fa + (size_t)b * W;
  const uint32_t* gp = gb + (size_t)b * W;
  bool neg = false;
  if (da < db) {  // modpoly.py:138-141
    neg = (da * db) & 1;
    const uint32_t* tp = fp; fp = gp; gp = tp;
    int td = da; da = db; db = td;
  }
  uint32_t A[MAXD + 1], B[MAXD + 1];
#pragma unroll
  for (int i = 0; i <= MAXD; ++i) {
    A[i] = (i <= da) ? fp[da - i] : 0u;
    B[i] = (i <= db) ? gp[db - i] : 0u;
  }
  uint32_t v;
  if (db == 0) {  // modpoly.py:145-146: res * b0^da
    const uint32_t one = redc(P.r2, P);
    v = redc(mpow(to_mont(B[0], P), da, one, P), P);
    if (neg) v = neg_mod(v, P.p);
  } else {
    v = resultant_topaligned<MAXD>(A, da, B, db, neg, P);
  }
  out[b] = v;
}

void launch_uni_resultant(const uint32_t* fa, const int32_t* da, const uint32_t* gb, const int32_t* db, int W,
                          const Prime* primes, const int32_t* pidx, int B, uint32_t* out, cudaStream_t st) {
  const int maxd = W - 1;
  const int bucket = images_maxd(maxd, 0);
  const int grid = (B + IMG_THREADS - 1) / IMG_THREADS;
#define LAUNCH(D)                                                                                 \
  if (bucket == D) {                                                                              \
    k_uni_resultant<D><<<grid, IMG_THREADS, 0, st>>>(fa, da, gb, db, W, primes, pidx, B, out);    \
    return;                                                                                       \
  }
  CKB_MAXD_LIST(LAUNCH)
#undef LAUNCH
}

}  // namespace ckb

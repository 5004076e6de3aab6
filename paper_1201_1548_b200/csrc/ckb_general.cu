// General (any degree, any degree-drop pattern) univariate resultant mod p,
// one warp per problem, operands low-degree-first in shared memory.
//
// A line-by-line restatement of curvekit.modpoly._zp_resultant and _zp_rem
// (pkg/src/curvekit/modpoly.py:102-112, :132-153) with the coefficient
// updates spread over the lanes.  Used for
//   * the images whose remainder sequence is not generic (the fast kernel's
//     fail list; rare for random inputs, systematic for sparse ones), and
//   * the batched zp_resultant_uni API (modpoly.py:156-161), valid for every
//     odd prime below 2^31 and every degree.
#include "ckb_kernels.cuh"

namespace ckb {

__device__ __forceinline__ int warp_trim(const uint32_t* c, int len) {
  while (len > 0 && c[len - 1] == 0u) --len;
  return len;
}

// res(a, b) mod p; a, b, r are shared buffers of capacity >= max(la, lb)
__device__ uint32_t warp_resultant(uint32_t* a, int la, uint32_t* b, int lb, uint32_t* r, const Prime& P) {
  const int lane = threadIdx.x & 31;
  const uint32_t p = P.p;
  la = warp_trim(a, la);
  lb = warp_trim(b, lb);
  if (!la || !lb) return 0u;
  uint32_t res = 1u % p;
  if (la < lb) {  // modpoly.py:138-141
    if (((la - 1) * (lb - 1)) & 1) res = p - 1;
    uint32_t* t = a; a = b; b = t;
    int tl = la; la = lb; lb = tl;
  }
  for (;;) {
    const int da = la - 1, db = lb - 1;
    if (db == 0) return mul_mod(res, pow_mod(b[0], (uint64_t)da, P), P);
    // r = _zp_rem(a, b)
    for (int i = lane; i < la; i += 32) r[i] = a[i];
    __syncwarp();
    const uint32_t inv = inv_mod(b[lb - 1], P);
    int lr = la;
    while (lr >= lb) {
      const uint32_t c = mul_mod(r[lr - 1], inv, P);
      __syncwarp();  // every lane has read r[lr - 1] before its owner updates it
      if (c) {
        const int k = lr - lb;
        const uint32_t nc = p - c;
        const uint32_t ncc = shoup_comp(nc, P);
        for (int j = lane; j < lb; j += 32) r[k + j] = add_mod(r[k + j], shoup(b[j], nc, ncc, p), p);
      }
      __syncwarp();
      --lr;  // r.pop()
    }
    lr = warp_trim(r, lr);
    if (!lr) return 0u;
    const int dr = lr - 1;
    if ((da * db) & 1) res = res ? p - res : 0u;
    res = mul_mod(res, pow_mod(b[lb - 1], (uint64_t)(da - dr), P), P);
    uint32_t* t = a;  // a, b = b, r
    a = b;
    b = r;
    r = t;
    la = lb;
    lb = lr;
    __syncwarp();
  }
}

// recompute the fast kernel's failed images
__global__ void k_images_fallback(ImageArgs a, int W) {
  extern __shared__ uint32_t sm[];
  CKB_SMEM_POISON(sm);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t* fa = sm + (size_t)warp * 3 * W;  // one warp per failed image
  uint32_t* gb = fa + W;
  uint32_t* rr = fa + 2 * W;
  // pdl_launch();  (implicit at exit: measured better)
  pdl_wait();
  const uint32_t count = *a.fail_count;
  for (uint32_t idx = blockIdx.x * nw + warp; idx < count; idx += gridDim.x * nw) {
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
    const uint32_t* res = a.red + (size_t)pi * a.C;
    const int offG = (a.m + 1) * (a.dfx + 1);
    for (int j = lane; j <= a.m + a.n + 1; j += 32) {
      const bool isf = j <= a.m;
      const int jj = isf ? j : j - a.m - 1;
      const uint32_t* c = res + (isf ? j * (a.dfx + 1) : offG + jj * (a.dgx + 1));
      const int deg = a.degs[j];
      uint32_t acc = 0u;
      for (int i = deg; i >= 0; --i) acc = add_mod(shoup(acc, x, xc, p), c[i], p);
      (isf ? fa : gb)[jj] = acc;
    }
    __syncwarp();
    const uint32_t v = warp_resultant(fa, a.m + 1, gb, a.n + 1, rr, P);
    if (lane == 0) a.values[flat] = v;
    __syncwarp();
  }
}

void launch_images_fallback(const ImageArgs& a, cudaStream_t st) {
  // one CTA of 4 warps per SM (the same 592 warps as 592 one-warp CTAs, a quarter of the CTA launches:
  // the list is usually empty and the launch is pure overhead)
  const int W = (a.m > a.n ? a.m : a.n) + 2;
  launch_pdl(k_images_fallback, dim3(148), dim3(128), (size_t)4 * 3 * W * 4, st, a, W);
}

__global__ void k_iota(uint32_t* list, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) list[i] = i;
  if (i == 0) list[n] = n;  // the count slot follows the list
}

// shapes beyond the register kernel: the general kernel over every image
void launch_images_general(const ImageArgs& a, cudaStream_t st) {
  const uint32_t n = (uint32_t)a.K * (uint32_t)a.N;
  k_iota<<<(n + 255) / 256, 256, 0, st>>>(a.fail_list, n);
  const int W = (a.m > a.n ? a.m : a.n) + 2;
  const size_t smem = (size_t)4 * 3 * W * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_images_fallback, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_images_fallback<<<8 * 148, 128, smem, st>>>(a, W);
}

// batched zp_resultant_uni: one warp per pair
__global__ void k_uni_resultant(const uint32_t* __restrict__ fa, const int32_t* __restrict__ da,
                                const uint32_t* __restrict__ gb, const int32_t* __restrict__ db, int W,
                                const Prime* __restrict__ primes, const int32_t* __restrict__ pidx,
                                uint32_t* __restrict__ out, uint32_t* __restrict__ gs) {
  extern __shared__ uint32_t sm[];
  CKB_SMEM_POISON(sm);
  const int b = blockIdx.x, lane = threadIdx.x;
  // operands in shared memory, or (degrees beyond it) in a global scratch slice per pair
  uint32_t* x = gs ? gs + (size_t)b * 3 * W : sm;
  uint32_t* y = x + W;
  uint32_t* r = x + 2 * W;
  const int la = da[b] + 1, lb = db[b] + 1;
  for (int i = lane; i < W; i += 32) {
    x[i] = i < la ? fa[(size_t)b * W + i] : 0u;
    y[i] = i < lb ? gb[(size_t)b * W + i] : 0u;
  }
  __syncwarp();
  const uint32_t v = warp_resultant(x, la, y, lb, r, primes[pidx[b]]);
  if (lane == 0) out[b] = v;
}

void launch_uni_resultant(const uint32_t* fa, const int32_t* da, const uint32_t* gb, const int32_t* db, int W,
                          const Prime* primes, const int32_t* pidx, int B, uint32_t* out, uint32_t* gs,
                          cudaStream_t st) {
  const size_t smem = gs ? 0 : (size_t)3 * W * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_uni_resultant, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_uni_resultant<<<B, 32, smem, st>>>(fa, da, gb, db, W, primes, pidx, out, gs);
}

}  // namespace ckb

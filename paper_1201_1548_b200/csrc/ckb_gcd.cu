// K6: batched univariate gcd mod p (one CTA per pair) and interpolation at
// arbitrary points (one CTA per problem).
//
// gcd: restates curvekit.modpoly._zp_gcd (pkg/src/curvekit/modpoly.py:115-122)
// -- Euclid, then monic -- but division-free: A <- lc(B) A - lc(A) x^s B keeps
// every remainder a nonzero scalar multiple of the reference's, so the monic
// normalisation at the end (one Fermat inverse) yields the identical result.
// Operands live low-degree-first in shared memory; a degree drop is just a
// decrement of the degree, no data moves.
//
// interpolation at arbitrary points: restates _zp_interp (modpoly.py:164-185)
// step for step (Newton divided differences, then Newton -> monomial), each
// O(n) sweep parallel across the CTA.
#include "ckb_kernels.cuh"

namespace ckb {

constexpr int GCD_THREADS = 256;

__global__ void __launch_bounds__(GCD_THREADS) k_gcd_mod(const uint32_t* __restrict__ fa,
                                                         const int32_t* __restrict__ da_, int Wf,
                                                         const uint32_t* __restrict__ gb,
                                                         const int32_t* __restrict__ db_, int Wg,
                                                         const Prime* __restrict__ primes,
                                                         const int32_t* __restrict__ pidx, uint32_t* __restrict__ out,
                                                         int Wo, int32_t* __restrict__ odeg, uint32_t* __restrict__ gs) {
  extern __shared__ uint32_t sm_[];
  __shared__ int s_da, s_db, s_swap;
  __shared__ uint32_t s_la, s_lb;
  const int b = blockIdx.x, tid = threadIdx.x, T = blockDim.x;
  const Prime P = primes[pidx[b]];
  const uint32_t p = P.p;
  const int W = max(Wf, Wg);
  // two operand buffers of W words: shared memory, or a global scratch slice beyond it
  uint32_t* sm = gs ? gs + (size_t)b * 2 * W : sm_;
  uint32_t* X = sm;
  uint32_t* Y = sm + W;
  int da = da_[b], db = db_[b];
  for (int i = tid; i < W; i += T) {
    X[i] = (i <= da && i < Wf) ? fa[(size_t)b * Wf + i] : 0u;
    Y[i] = (i <= db && i < Wg) ? gb[(size_t)b * Wg + i] : 0u;
  }
  __syncthreads();
  // a, b = trim(a), trim(b);  while b: a, b = b, a rem b
  uint32_t* A = X;
  uint32_t* B = Y;
  while (db >= 0) {
    // A <- A rem B (division-free): repeat while deg A >= deg B
    while (da >= db) {
      const uint32_t la = A[da], lb = B[db];
      const int s = da - db;
      const uint32_t lbc = shoup_comp(lb, P);
      const uint32_t nla = neg_mod(la, p), nlac = shoup_comp(nla, P);
      for (int j = tid; j < da; j += T) {
        uint32_t v = shoup(A[j], lb, lbc, p);
        if (j >= s) v = add_mod(v, shoup(B[j - s], nla, nlac, p), p);
        A[j] = v;
      }
      __syncthreads();
      if (tid == 0) {
        int d = da - 1;
        while (d >= 0 && A[d] == 0u) --d;
        s_da = d;
      }
      __syncthreads();
      da = s_da;
      if (da < 0) break;
    }
    // swap roles
    uint32_t* tp = A;
    A = B;
    B = tp;
    const int td = da;
    da = db;
    db = td;
    __syncthreads();
  }
  // A holds the gcd (deg da), make it monic
  const uint32_t inv = (da >= 0) ? inv_mod(A[da], P) : 0u;
  const uint32_t invc = shoup_comp(inv, P);
  for (int i = tid; i < Wo; i += T) out[(size_t)b * Wo + i] = (i <= da) ? shoup(A[i], inv, invc, p) : 0u;
  if (tid == 0) odeg[b] = da;
  (void)s_db;
  (void)s_swap;
  (void)s_la;
  (void)s_lb;
}

void launch_gcd_mod(const uint32_t* fa, const int32_t* da, int Wf, const uint32_t* gb, const int32_t* db, int Wg,
                    const Prime* primes, const int32_t* pidx, int B, uint32_t* out, int Wo, int32_t* odeg,
                    uint32_t* gs, cudaStream_t st) {
  const size_t smem = gs ? 0 : (size_t)2 * (Wf > Wg ? Wf : Wg) * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_gcd_mod, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_gcd_mod<<<B, GCD_THREADS, smem, st>>>(fa, da, Wf, gb, db, Wg, primes, pidx, out, Wo, odeg, gs);
}

// ---------------------------------------------------------------------------
// interpolation at arbitrary distinct points (one problem per CTA)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(GCD_THREADS) k_interp_points(const uint32_t* __restrict__ xs,
                                                               const uint32_t* __restrict__ vs, const int32_t* __restrict__ ns,
                                                               int W, const Prime* __restrict__ primes,
                                                               const int32_t* __restrict__ pidx,
                                                               uint32_t* __restrict__ out, uint32_t* __restrict__ gs) {
  extern __shared__ uint32_t sm_[];
  const int b = blockIdx.x, tid = threadIdx.x, T = blockDim.x;
  const int n = ns[b];
  uint32_t* sm = gs ? gs + (size_t)b * (4 * W + 2) : sm_;  // global scratch beyond shared memory
  const Prime P = primes[pidx[b]];
  const uint32_t p = P.p;
  uint32_t* x = sm;            // points
  uint32_t* c = sm + W;        // divided differences
  uint32_t* o = sm + 2 * W;    // output (n + 1 words)
  uint32_t* o2 = sm + 3 * W + 1;
  for (int i = tid; i < n; i += T) {
    x[i] = xs[(size_t)b * W + i];
    c[i] = vs[(size_t)b * W + i];
  }
  __syncthreads();
  // for j in 1..n-1: for i = n-1 .. j: c[i] = (c[i] - c[i-1]) / (x[i] - x[i-j]).
  // The reference takes one Fermat inverse per entry (modpoly.py:172-178); here
  // each thread inverts the denominators of its strided entries of a row at
  // once (Montgomery's trick: running products in o2, one inverse, a backward
  // pass), so a row costs T inverses instead of n - j.
  for (int j = 1; j < n; ++j) {
    int last = -1;
    uint32_t run = 1u;
    for (int i = j + tid; i < n; i += T) {
      run = mul_mod(run, sub_mod(x[i], x[i - j], p), P);
      o2[i] = run;  // prefix product of this thread's denominators
      last = i;
    }
    if (last >= 0) {
      uint32_t inv = inv_mod(run, P);
      for (int i = last; i >= j; i -= T) {
        const uint32_t d = sub_mod(x[i], x[i - j], p);
        const uint32_t invd = (i - T >= j) ? mul_mod(inv, o2[i - T], P) : inv;  // 1/d_i
        inv = mul_mod(inv, d, P);
        o2[i] = mul_mod(sub_mod(c[i], c[i - 1], p), invd, P);
      }
    }
    __syncthreads();
    for (int i = j + tid; i < n; i += T) c[i] = o2[i];
    __syncthreads();
  }
  // out = 0; for i = n-1 .. 0: out = out * (x - x_i) + c_i
  for (int k = tid; k <= n; k += T) o[k] = 0u;
  __syncthreads();
  for (int i = n - 1; i >= 0; --i) {
    const uint32_t xi = x[i];
    const uint32_t nxi = neg_mod(xi, p), nxic = shoup_comp(nxi, P);
    for (int k = tid; k <= n; k += T) {
      uint32_t v = shoup(o[k], nxi, nxic, p);  // -x_i * out[k]
      if (k > 0) v = add_mod(v, o[k - 1], p);
      if (k == 0) v = add_mod(v, c[i], p);
      o2[k] = v;
    }
    __syncthreads();
    for (int k = tid; k <= n; k += T) o[k] = o2[k];
    __syncthreads();
  }
  for (int k = tid; k < n; k += T) out[(size_t)b * W + k] = o[k];
}

void launch_interp_points(const uint32_t* xs, const uint32_t* vs, const int32_t* ns, int W, const Prime* primes,
                          const int32_t* pidx, int B, uint32_t* out, uint32_t* gs, cudaStream_t st) {
  const size_t smem = gs ? 0 : (size_t)(4 * W + 2) * 4;
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_interp_points, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_interp_points<<<B, GCD_THREADS, smem, st>>>(xs, vs, ns, W, primes, pidx, out, gs);
}

}  // namespace ckb

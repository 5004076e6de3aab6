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
  CKB_SMEM_POISON(sm_);
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

// inclusive multiplicative scan of buf[0..n) by one CTA; rev: suffix products
constexpr int INTERP_THREADS = 1024;
// scratch shared by the device functions below (one static allocation per kernel)
struct InterpShared {
  uint32_t sh[INTERP_THREADS];      // scan partials
  uint32_t bnd[2][INTERP_THREADS];  // row boundaries (two slots)
};
static __device__ void interp_scan_mul(uint32_t* buf, int n, bool rev, const Prime& P, uint32_t* sh) {
  const int T = blockDim.x, tid = threadIdx.x;
  const int seg = (n + T - 1) / T;
  const int s0 = min(n, tid * seg), s1 = min(n, s0 + seg);
  auto at = [&](int i) -> uint32_t& { return buf[rev ? n - 1 - i : i]; };
  uint32_t acc = 1u % P.p;
  for (int i = s0; i < s1; ++i) {
    acc = mul_mod(acc, at(i), P);
    at(i) = acc;
  }
  sh[tid] = acc;
  __syncthreads();
  for (int off = 1; off < T; off <<= 1) {
    const uint32_t v = (tid >= off) ? sh[tid - off] : 1u % P.p;
    __syncthreads();
    if (tid >= off) sh[tid] = mul_mod(sh[tid], v, P);
    __syncthreads();
  }
  const uint32_t pre = tid ? sh[tid - 1] : 1u % P.p;
  __syncthreads();
  if (tid)
    for (int i = s0; i < s1; ++i) at(i) = mul_mod(at(i), pre, P);
  __syncthreads();
}

// register-resident variant: thread t owns entries [t SEG, (t+1) SEG) of the
// difference table and of the output in registers; per row only the boundary
// value crosses threads (two-slot array, one barrier).  Needs n + 1 <= SEG T.
template <int SEG>
__device__ __forceinline__ void interp_consecutive_reg(uint32_t* x, uint32_t* c, uint32_t* o, uint32_t* o2, int n, const Prime& P,
                                       uint32_t* __restrict__ out, InterpShared& S) {
  auto& bnd = S.bnd;
  const int T = blockDim.x, tid = threadIdx.x;
  const uint32_t p = P.p;
  const uint32_t x0 = x[0];
  __syncthreads();
  for (int i = tid; i < n; i += T) o2[i] = i ? (uint32_t)i % p : 1u % p;
  __syncthreads();
  interp_scan_mul(o2, n, false, P, S.sh);
  const uint32_t inv_last = inv_mod(o2[n - 1], P);
  for (int i = tid; i < n; i += T) o[i] = (i == n - 1) ? inv_last : (uint32_t)(i + 1) % p;
  __syncthreads();
  interp_scan_mul(o, n, true, P, S.sh);
  for (int j = tid; j < n; j += T) x[j] = j ? mul_mod(o[j], o2[j - 1], P) : 0u;  // 1/j
  __syncthreads();
  for (int j = tid; j < n; j += T) o[j] = shoup_comp(x[j], P);  // and its Shoup companion
  const int s0 = tid * SEG;
  uint32_t v[SEG];
#pragma unroll
  for (int e = 0; e < SEG; ++e) v[e] = s0 + e < n ? c[s0 + e] : 0u;
  __syncthreads();
  for (int j = 1; j < n; ++j) {
    const int slot = j & 1;
    const uint32_t w = x[j], wc = o[j];  // independent of this row's barrier
    bnd[slot][tid] = v[SEG - 1];
    __syncthreads();
    const uint32_t prev = tid ? bnd[slot][tid - 1] : 0u;
#pragma unroll
    for (int e = SEG - 1; e >= 0; --e) {
      const uint32_t lo = e ? v[e - 1] : prev;
      if (s0 + e >= j) v[e] = shoup(sub_mod(v[e], lo, p), w, wc, p);
    }
  }
#pragma unroll
  for (int e = 0; e < SEG; ++e)
    if (s0 + e < n) c[s0 + e] = v[e];
  __syncthreads();
  // Newton -> monomial over entries 0..n (o = 0 initially)
#pragma unroll
  for (int e = 0; e < SEG; ++e) v[e] = 0u;
  for (int i = n - 1; i >= 0; --i) {
    const int slot = i & 1;
    const uint32_t xi = (uint32_t)(((uint64_t)x0 + (uint64_t)i) % p);
    const uint32_t nxi = neg_mod(xi, p), nxic = shoup_comp(nxi, P);
    const uint32_t ci = c[i];
    bnd[slot][tid] = v[SEG - 1];
    __syncthreads();
    const uint32_t prev = tid ? bnd[slot][tid - 1] : 0u;
#pragma unroll
    for (int e = SEG - 1; e >= 0; --e) {
      uint32_t t = add_mod(shoup(v[e], nxi, nxic, p), e ? v[e - 1] : prev, p);
      if (s0 + e == 0) t = add_mod(t, ci, p);
      v[e] = t;
    }
  }
#pragma unroll
  for (int e = 0; e < SEG; ++e)
    if (s0 + e < n) out[s0 + e] = v[e];
}

// Newton interpolation at x_i = x_0 + i: c (values, n >= 2) -> o (coefficients).
// x is reused for the table 1/j; every row / Horner step is one pass over
// contiguous per-thread segments with the left neighbour's old boundary value
// passed through a two-slot array (one barrier per row).
__device__ __forceinline__ void interp_consecutive(uint32_t* x, uint32_t* c, uint32_t* o, uint32_t* o2, int n, const Prime& P,
                                   InterpShared& S) {
  auto& bnd = S.bnd;
  const int T = blockDim.x, tid = threadIdx.x;
  const uint32_t p = P.p;
  const uint32_t x0 = x[0];
  __syncthreads();  // every thread has read x[0]
  // 1/j = (j-1)! / j!:  o2[i] = i!, o[i] = 1/i! (suffix products from 1/(n-1)!)
  for (int i = tid; i < n; i += T) o2[i] = i ? (uint32_t)i % p : 1u % p;
  __syncthreads();
  interp_scan_mul(o2, n, false, P, S.sh);
  const uint32_t inv_last = inv_mod(o2[n - 1], P);
  for (int i = tid; i < n; i += T) o[i] = (i == n - 1) ? inv_last : (uint32_t)(i + 1) % p;
  __syncthreads();
  interp_scan_mul(o, n, true, P, S.sh);  // o[i] = inv_last * (i+1) ... (n-1) = 1/i!
  for (int j = tid; j < n; j += T) x[j] = j ? mul_mod(o[j], o2[j - 1], P) : 0u;  // 1/j
  __syncthreads();
  const int seg = (n + T - 1) / T;
  const int s0 = min(n, tid * seg), s1 = min(n, s0 + seg);
  // forward differences: row j, i >= j: c[i] = (c[i] - c[i-1]) / j
  for (int j = 1; j < n; ++j) {
    const int slot = j & 1;
    if (s1 > s0) bnd[slot][tid] = c[s1 - 1];  // this thread's old last entry
    __syncthreads();
    const uint32_t prev = (tid > 0 && s0 > 0) ? bnd[slot][tid - 1] : 0u;
    const uint32_t w = x[j], wc = shoup_comp(w, P);
    for (int i = s1 - 1; i >= max(s0, j); --i) {
      const uint32_t lo = i > s0 ? c[i - 1] : prev;
      c[i] = shoup(sub_mod(c[i], lo, p), w, wc, p);
    }
  }
  __syncthreads();
  // Newton -> monomial: o = 0; for i = n-1 .. 0: o = o (x - x_i) + c_i  (x_i = x0 + i)
  for (int k = tid; k <= n; k += T) o[k] = 0u;
  __syncthreads();
  const int seg2 = (n + 1 + T - 1) / T;
  const int u0 = min(n + 1, tid * seg2), u1 = min(n + 1, u0 + seg2);
  for (int i = n - 1; i >= 0; --i) {
    const int slot = i & 1;
    if (u1 > u0) bnd[slot][tid] = o[u1 - 1];
    __syncthreads();
    const uint32_t prev = (tid > 0 && u0 > 0) ? bnd[slot][tid - 1] : 0u;
    const uint32_t xi = (uint32_t)(((uint64_t)x0 + (uint64_t)i) % p);
    const uint32_t nxi = neg_mod(xi, p), nxic = shoup_comp(nxi, P);
    const uint32_t ci = c[i];
    for (int k = u1 - 1; k >= u0; --k) {
      uint32_t v = shoup(o[k], nxi, nxic, p);  // -x_i o[k]
      v = add_mod(v, k > u0 ? o[k - 1] : prev, p);
      if (k == 0) v = add_mod(v, ci, p);
      o[k] = v;
    }
  }
  __syncthreads();
  (void)o2;
}
__global__ void __launch_bounds__(INTERP_THREADS) k_interp_points(const uint32_t* __restrict__ xs,
                                                               const uint32_t* __restrict__ vs, const int32_t* __restrict__ ns,
                                                               int W, const Prime* __restrict__ primes,
                                                               const int32_t* __restrict__ pidx,
                                                               uint32_t* __restrict__ out, uint32_t* __restrict__ gs,
                                                               int xstride) {
  extern __shared__ uint32_t sm_[];
  CKB_SMEM_POISON(sm_);
  __shared__ InterpShared S;
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
    x[i] = xs[(size_t)b * xstride + i];  // xstride 0: one point list shared by every problem
    c[i] = vs[(size_t)b * W + i];
  }
  __syncthreads();
  // consecutive points x_i = x_0 + i (the reference's t = 0, 1, 2, ... when no t
  // is skipped): the divided differences are forward differences and row j
  // divides by j alone
  int cons = 1;
  for (int i = tid; i < n; i += T)
    if (x[i] != (uint32_t)(((uint64_t)x[0] + (uint64_t)i) % p)) cons = 0;
  if (__syncthreads_and(cons) && n >= 2) {
    uint32_t* ob = out + (size_t)b * W;
    if (n + 1 <= T) return interp_consecutive_reg<1>(x, c, o, o2, n, P, ob, S);
    if (n + 1 <= 2 * T) return interp_consecutive_reg<2>(x, c, o, o2, n, P, ob, S);
    if (n + 1 <= 4 * T) return interp_consecutive_reg<4>(x, c, o, o2, n, P, ob, S);
    if (n + 1 <= 8 * T) return interp_consecutive_reg<8>(x, c, o, o2, n, P, ob, S);
    interp_consecutive(x, c, o, o2, n, P, S);
    for (int k = tid; k < n; k += T) ob[k] = o[k];
    return;
  }
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
                          const int32_t* pidx, int B, uint32_t* out, uint32_t* gs, cudaStream_t st, int xstride) {
  const size_t smem = gs ? 0 : (size_t)(4 * W + 2) * 4;
  // the static InterpShared (12 KB) counts against the 48 KB default too
  if (smem + sizeof(InterpShared) > 48 * 1024)
    cudaFuncSetAttribute(k_interp_points, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_interp_points<<<B, INTERP_THREADS, smem, st>>>(xs, vs, ns, W, primes, pidx, out, gs, xstride < 0 ? W : xstride);
}

}  // namespace ckb

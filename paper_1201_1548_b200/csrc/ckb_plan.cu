// K1 coefficient reduction and the per-prime evaluation/interpolation plan.
//
// Reduction restates modpoly.py:376-377 (`[[c % p for c in cf] for cf in fc]`)
// for two's-complement multi-word integers.  The plan replaces the
// reference's point walk t = 0, 1, 2, ... with lc_f(t) lc_g(t) != 0 skips
// (modpoly.py:380-390) by a geometric progression x_t = c q^t (q a primitive
// root, c = 1, 2, ... chosen per prime so that no point annihilates a leading
// coefficient).  For geometric points the interpolation matrix has closed
// form (q-binomial theorem), so every table below is a prefix product.
#include "ckb_kernels.cuh"
#include "ckb_choose.cuh"

namespace ckb {

// ---------------------------------------------------------------------------
// K1 reduce
// ---------------------------------------------------------------------------
__global__ void k_reduce(const uint32_t* __restrict__ limbs, int C, int L, const Prime* __restrict__ primes,
                         uint32_t* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int pi = blockIdx.y;
  if (c >= C) return;
  out[(size_t)pi * C + c] = limbs_mod(limbs + (size_t)c * L, L, primes[pi]);
}

void launch_reduce(const uint32_t* limbs, int C, int L, const Prime* primes, int K, uint32_t* out,
                   cudaStream_t st) {
  dim3 grid((C + 127) / 128, K);
  k_reduce<<<grid, 128, 0, st>>>(limbs, C, L, primes, out);
}

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
constexpr int PLAN_THREADS = 256;

// inclusive multiplicative scan of buf[0..n) in global memory by one CTA:
// sequential segments + Hillis-Steele over the segment totals (reverse = suffix)
__device__ void block_scan_mul(uint32_t* buf, int n, bool reverse, const Prime& P, uint32_t* sh) {
  const int T = blockDim.x, tid = threadIdx.x;
  const int seg = (n + T - 1) / T;
  const int s0 = min(n, tid * seg), s1 = min(n, s0 + seg);
  auto at = [&](int i) -> uint32_t& { return reverse ? buf[n - 1 - i] : buf[i]; };
  uint32_t acc = 1u;
  for (int i = s0; i < s1; ++i) {
    acc = mul_mod(acc, at(i), P);
    at(i) = acc;
  }
  sh[tid] = acc;
  __syncthreads();
  for (int off = 1; off < T; off <<= 1) {
    uint32_t v = (tid >= off) ? sh[tid - off] : 1u;
    __syncthreads();
    if (tid >= off) sh[tid] = mul_mod(sh[tid], v, P);
    __syncthreads();
  }
  const uint32_t pre = tid ? sh[tid - 1] : 1u;
  __syncthreads();
  if (tid && pre != 1u)
    for (int i = s0; i < s1; ++i) at(i) = mul_mod(at(i), pre, P);
  __syncthreads();
}

__device__ __forceinline__ uint64_t binom2(uint64_t m) { return m * (m - 1) / 2; }

// base tables of the plan for c = 1 (one CTA per prime)
__global__ void __launch_bounds__(PLAN_THREADS) k_plan(const Prime* __restrict__ primes,
                                                       const uint32_t* __restrict__ gens, int N, InterpPlan plan) {
  __shared__ uint32_t sh[PLAN_THREADS];
  const int pi = blockIdx.x, tid = threadIdx.x, T = blockDim.x;
  const Prime P = primes[pi];
  const uint32_t p = P.p;
  const uint64_t pm1 = p - 1;
  const uint32_t q = pow_mod(gens[pi] % p, (uint64_t)plan.S, P);  // ratio of the interpolation points
  const uint32_t qinv = inv_mod(q, P);
  const uint32_t qc = shoup_comp(q, P), qinvc = shoup_comp(qinv, P);
  const size_t oN = (size_t)pi * N, o2N = (size_t)pi * 2 * N, oN1 = (size_t)pi * (N + 1);

  // q^C(m,2) for m in [0, 2N): segment start by pow, then h(m+1) = h(m) q^m
  {
    const int n = 2 * N, seg = (n + T - 1) / T;
    const int s0 = min(n, tid * seg), s1 = min(n, s0 + seg);
    if (s0 < s1) {
      uint32_t h = pow_mod(q, binom2(s0) % pm1, P), qm = pow_mod(q, s0, P);
      for (int m = s0; m < s1; ++m) {
        plan.hC[o2N + m] = h;
        h = mul_mod(h, qm, P);
        qm = shoup(qm, q, qc, p);
      }
    }
  }
  // q^-C(m,2) for m in [0, N)
  {
    const int n = N, seg = (n + T - 1) / T;
    const int s0 = min(n, tid * seg), s1 = min(n, s0 + seg);
    if (s0 < s1) {
      uint32_t h = pow_mod(qinv, binom2(s0) % pm1, P), qm = pow_mod(qinv, s0, P);
      for (int m = s0; m < s1; ++m) {
        plan.hCinv[oN + m] = h;
        h = mul_mod(h, qm, P);
        qm = shoup(qm, qinv, qinvc, p);
      }
    }
  }
  // phi_j = prod_{i=1..j} (q^i - 1), j = 0..N  (phi_0 = 1)
  uint32_t* phi = plan.phi + oN1;
  uint32_t* iphi = plan.iphi + oN1;
  {
    const int n = N + 1, seg = (n + T - 1) / T;
    const int s0 = min(n, tid * seg), s1 = min(n, s0 + seg);
    if (s0 < s1) {
      uint32_t qi = pow_mod(q, s0, P);
      for (int j = s0; j < s1; ++j) {
        phi[j] = j ? sub_mod(qi, 1u, p) : 1u;
        qi = shoup(qi, q, qc, p);
      }
    }
  }
  __syncthreads();
  block_scan_mul(phi, N + 1, false, P, sh);
  // iphi_j = phi_N^-1 * prod_{i=j+1..N} (q^i - 1): suffix product of the
  // factors shifted by one, times the single inverse of phi_N
  __shared__ uint32_t s_inv;
  if (tid == 0) s_inv = inv_mod(phi[N], P);
  __syncthreads();
  // factors g_j = q^(j+1) - 1 (j < N), g_N = phi_N^-1; suffix products give 1/phi_j
  {
    const int n = N + 1, seg = (n + T - 1) / T;
    const int s0 = min(n, tid * seg), s1 = min(n, s0 + seg);
    if (s0 < s1) {
      uint32_t qi = pow_mod(q, s0 + 1, P);
      for (int j = s0; j < s1; ++j) {
        iphi[j] = (j == N) ? s_inv : sub_mod(qi, 1u, p);
        qi = shoup(qi, q, qc, p);
      }
    }
  }
  __syncthreads();
  block_scan_mul(iphi, N + 1, true, P, sh);

  const uint32_t r = pow_mod(qinv, (uint64_t)(N >= 2 ? N - 2 : 0) % pm1, P);  // q^-(N-2)
  const uint32_t rc = shoup_comp(r, P);
  const uint32_t phiN = phi[N];
  __syncthreads();
  // per-point tables: x_t = q^t and z_t = (-1)^(N-1-t) q^-t(N-2) iphi_t iphi_{N-1-t}
  {
    const int n = N, seg = (n + T - 1) / T;
    const int s0 = min(n, tid * seg), s1 = min(n, s0 + seg);
    if (s0 < s1) {
      uint32_t qt = pow_mod(q, s0, P);
      uint32_t rt = (N >= 2) ? pow_mod(r, s0, P) : 1u;
      for (int t = s0; t < s1; ++t) {
        plan.xq[oN + t] = qt;
        uint32_t z = mul_mod(mul_mod(rt, iphi[t], P), iphi[N - 1 - t], P);
        if ((N - 1 - t) & 1) z = neg_mod(z, p);
        plan.z[oN + t] = z;
        qt = shoup(qt, q, qc, p);
        rt = shoup(rt, r, rc, p);
      }
    }
  }
  // M~_{N-k} = (-1)^k q^C(k,2) phi_N iphi_k iphi_{N-k}, k = 0..N
  for (int k = tid; k <= N; k += T) {
    uint32_t v = mul_mod(mul_mod(plan.hC[o2N + k], phiN, P), mul_mod(iphi[k], iphi[N - k], P), P);
    if (k & 1) v = neg_mod(v, p);
    plan.Mt[oN1 + (N - k)] = v;
  }
}

// per call: the point scale c of every prime (choose_c_prime, ckb_choose.cuh);
// the pipeline's fast path runs the same function inside the merged K1 kernel
__global__ void __launch_bounds__(PLAN_THREADS) k_choose_c(const Prime* __restrict__ primes, InterpPlan plan,
                                                           const uint32_t* __restrict__ red, int C, int lcf_off,
                                                           int lcf_deg, int lcg_off, int lcg_deg,
                                                           uint32_t* __restrict__ cval, uint32_t* status) {
  const int pi = blockIdx.x;
  // pdl_launch();  (implicit at exit: measured better)
  pdl_wait();
  const Prime P = primes[pi];
  choose_c_prime(P, pi, plan, red + (size_t)pi * C + lcf_off, lcf_deg, red + (size_t)pi * C + lcg_off, lcg_deg, cval,
                 status);
}

void launch_choose_c(const Prime* primes, const InterpPlan& plan, const uint32_t* red, int C, int lcf_off,
                     int lcf_deg, int lcg_off, int lcg_deg, uint32_t* cval, uint32_t* status, cudaStream_t st) {
  launch_pdl(k_choose_c, dim3(plan.K), dim3(PLAN_THREADS), 0, st, primes, plan, red, C, lcf_off, lcf_deg, lcg_off,
             lcg_deg, cval,
                                               status);
}

// polyphase point tables: y_u = g^u, g^-u (u < M) and the S-th roots of unity
__global__ void __launch_bounds__(PLAN_THREADS) k_plan_poly(const Prime* __restrict__ primes,
                                                            const uint32_t* __restrict__ gens, InterpPlan plan) {
  const int pi = blockIdx.x, tid = threadIdx.x, T = blockDim.x, M = plan.N, S = plan.S;
  const Prime P = primes[pi];
  const uint32_t p = P.p;
  const uint32_t g = gens[pi] % p, gi = inv_mod(g, P);
  const uint32_t gc = shoup_comp(g, P), gic = shoup_comp(gi, P);
  const size_t oM = (size_t)pi * M;
  const int seg = (M + T - 1) / T;
  const int s0 = min(M, tid * seg), s1 = min(M, s0 + seg);
  if (s0 < s1) {
    uint32_t a = pow_mod(g, s0, P), b = pow_mod(gi, s0, P);
    for (int u = s0; u < s1; ++u) {
      plan.yq[oM + u] = a;
      plan.yqi[oM + u] = b;
      a = shoup(a, g, gc, p);
      b = shoup(b, gi, gic, p);
    }
  }
  if (tid < S) {  // om[pi]: w^k, companions, w^-k, companions (w a primitive S-th root)
    const uint32_t w = pow_mod(g, (uint64_t)(p - 1) / S, P);
    const uint32_t wk = pow_mod(w, tid, P), wik = inv_mod(wk, P);
    uint32_t* om = plan.om + (size_t)pi * 4 * S;
    om[tid] = wk;
    om[S + tid] = shoup_comp(wk, P);
    om[2 * S + tid] = wik;
    om[3 * S + tid] = shoup_comp(wik, P);
  }
}

void launch_plan_base(const Prime* primes, const uint32_t* gens, const InterpPlan& plan, cudaStream_t st) {
  k_plan<<<plan.K, PLAN_THREADS, 0, st>>>(primes, gens, plan.N, plan);
  k_plan_poly<<<plan.K, PLAN_THREADS, 0, st>>>(primes, gens, plan);
}

}  // namespace ckb

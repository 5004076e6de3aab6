// Kernel declarations shared by the stage files and the C-ABI layer.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "ckb_modarith.cuh"

namespace ckb {

// ---- K1: coefficient reduction (modpoly.py:376-377) ------------------------
// limbs: [C][L] two's-complement little-endian u32 words; out: [K][C] in [0,p)
void launch_reduce(const uint32_t* limbs, int C, int L, const Prime* primes, int K, uint32_t* out,
                   cudaStream_t st);

// ---- plan: evaluation points + interpolation tables per prime ---------------
struct InterpPlan {
  int N;              // points per prime
  int K;              // primes
  uint32_t* xpts;     // [K][N]    x_t = c * q^t
  uint32_t* hC;       // [K][2N]   q^C(m,2)
  uint32_t* z;        // [K][N]    w_t * q^-C(t,2), w_t = 1/M'(q^t)
  uint32_t* hCinv;    // [K][N]    q^-C(e,2)
  uint32_t* Mt;       // [K][N+1]  coefficients of prod_t (y - q^t)
  uint32_t* Mtc;      // [K][N+1]  Shoup companions of Mt
  uint32_t* cinv;     // [K][N]    c^-k
  uint32_t* phi;      // [K][N+1]  scratch: prod_{i<=j} (q^i - 1)
  uint32_t* iphi;     // [K][N+1]  scratch: inverses of phi
  uint32_t* cval;     // [K]       chosen scale c
};
// lc polynomials of f and g (residues) are read from the reduced buffer:
// lcf = red + lcf_off (deg lcf_deg), lcg = red + lcg_off (deg lcg_deg), row stride C.
void launch_plan(const Prime* primes, const uint32_t* gens, int K, int N, const uint32_t* red, int C,
                 int lcf_off, int lcf_deg, int lcg_off, int lcg_deg, const InterpPlan& plan,
                 uint32_t* status, cudaStream_t st);

// ---- K2+K3: fused evaluation + univariate resultant (modpoly.py:382-390) ----
struct ImageArgs {
  const uint32_t* red;     // [K][C]
  const int16_t* degs;     // [(m+1) + (n+1)] x-degree of each y-coefficient (-1 = zero)
  const uint32_t* xpts;    // [K][N]
  const Prime* primes;
  int C, m, n, dfx, dgx, N, K;
  uint32_t* values;        // [K][N]
  uint32_t* status;        // bit 1: an image hit a vanishing leading coefficient
  uint32_t* fail_list;     // [K*N] flat indices of non-generic images
  uint32_t* fail_count;    // zeroed before the launch
};
int images_maxd(int m, int n);  // template bucket or -1
// fast generic kernel followed by the general warp kernel on its fail list
void launch_images(const ImageArgs& a, cudaStream_t st);
void launch_images_fallback(const ImageArgs& a, cudaStream_t st);

// batch of independent univariate resultants (modpoly.py:156-161)
// fa/gb: [B][W] padded low-first coefficients; degrees da/db; per-pair prime index
void launch_uni_resultant(const uint32_t* fa, const int32_t* da, const uint32_t* gb, const int32_t* db, int W,
                          const Prime* primes, const int32_t* pidx, int B, uint32_t* out, cudaStream_t st);

// ---- K4: interpolation at the planned points (modpoly.py:164-185) -----------
// values [K][N] -> coeffs [K][N] (canonical residues), scratch a/ac/S [K][N]
void launch_interp(const InterpPlan& plan, const Prime* primes, const uint32_t* values, uint32_t* coeffs,
                   uint32_t* a, uint32_t* ac, uint32_t* S, cudaStream_t st);

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
};
// coeffs [K][N] -> out [N][LW]; scratch >= 3 N LW words
void launch_crt(const CrtTables& t, const uint32_t* coeffs, int N, uint32_t* out, uint32_t* scratch,
                cudaStream_t st);

// ---- K6: batched gcd mod p (modpoly.py:115-122), interpolation at arbitrary points
void launch_gcd_mod(const uint32_t* fa, const int32_t* da, int Wf, const uint32_t* gb, const int32_t* db, int Wg,
                    const Prime* primes, const int32_t* pidx, int B, uint32_t* out, int Wo, int32_t* odeg,
                    cudaStream_t st);
void launch_interp_points(const uint32_t* xs, const uint32_t* vs, const int32_t* ns, int W, const Prime* primes,
                          const int32_t* pidx, int B, uint32_t* out, cudaStream_t st);

}  // namespace ckb

/* C-ABI of the B200 multi-modular resultant engine (libcurvekit_b200.so).
 *
 * The reference (arXiv 1201.1548 artifact, package `curvekit`) is pure
 * Python; its hot path is pkg/src/curvekit/modpoly.py.  Each entry point below
 * replaces one reference function or loop; the Python drop-in
 * (paper_1201_1548_b200/modpoly.py) binds them with ctypes, keeping the
 * reference's names, argument meaning and exceptions.
 *
 * Conventions: plain pointers and sizes; all host buffers are caller-owned and
 * never retained after return; device memory belongs to one process-global
 * context (ckb_init); calls are serialised by a mutex (ctypes releases the
 * GIL).  Integers cross the boundary as little-endian two's-complement 32-bit
 * limbs.  Primes must be odd with 3 <= p < 2^31 and pairwise distinct.
 * Return: 0 ok, > 0 recoverable (CKB_STATUS_*), < 0 failure (ckb_last_error()).
 */
#ifndef CURVEKIT_B200_H
#define CURVEKIT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CKB_ABI_VERSION 6
#define CKB_STATUS_REPLAN 1 /* a prime had no admissible evaluation points: re-plan without it */

int ckb_abi_version(void);
const char* ckb_last_error(void);
int ckb_init(int device);
int ckb_shutdown(void);
unsigned long long ckb_launch_count(void);

/* res_y(f, g) in Z[x] — replaces curvekit.modpoly.biv_resultant
 * (pkg/src/curvekit/modpoly.py:348-394) after its degenerate branches.
 *   limbs  [C][L]  f's dense grid f[j][i] (coefficient of x^i y^j, j <= m,
 *                  i <= dfx) followed by g's grid (j <= n, i <= dgx);
 *                  C = (m+1)(dfx+1) + (n+1)(dgx+1)
 *   degs   [m+n+2] trimmed x-degree of each y-coefficient (-1 = zero)
 *   primes/gens [K] primes and a generator of large order for each
 *   N      evaluation points per prime (N > deg_x res)
 *   any degrees: y-degrees up to 64 run the register kernel, larger ones (or
 *          tables beyond its shared memory) the general warp kernel
 *   out    [N][LW] coefficients of res (low degree first), two's complement;
 *          requires prod(primes) > 2 * (coefficient bound) and 2^(32 LW) > prod
 *   status bit 0: some prime had no admissible point set (CKB_STATUS_REPLAN)
 *   device_ms (optional) CUDA-event time of the device work incl. copies */
int ckb_biv_resultant(const uint32_t* limbs, int C, int L, const int16_t* degs, int m, int n, int dfx, int dgx,
                      const uint32_t* primes, const uint32_t* gens, int K, int N, int LW, uint32_t* out,
                      uint32_t* status, float* device_ms);

/* Several devices in one process: contexts 0..n-1 on
 * devices[0..n-1] (each with its own stream, buffers and cached tables); with
 * distinct devices the residue exchange uses NCCL (ncclCommInitAll, loaded at
 * run time) over NVLink, else peer copies.  A device may repeat (contexts that
 * share one GPU: a correctness configuration).  ckb_init(device) is the n = 1
 * case.  ckb_devices reports the context count and whether NCCL is in use. */
int ckb_init_devices(int n, const int* devices);

/* Images of the last res_y pipeline call that left the register kernel for the
 * general warp kernel (non-generic remainder sequences), and all its images. */
int ckb_last_fallback(unsigned long long* fallback, unsigned long long* images);

/* Diagnostics of the last ckb_biv_resultant call: host microseconds from entry
 * until the work was enqueued, and waiting for it to finish (us[0], us[1]). */
int ckb_host_times(float* us, int max);
int ckb_devices(int* n_contexts, int* nccl);

/* How the last ckb_biv_resultant_multi call exchanged residues: 0 one context,
 * 1 peer stores from the interpolation epilogue, 2 NCCL send/recv, 3 peer copies. */
int ckb_last_exchange(void);

/* ckb_biv_resultant over the first G contexts (primes sharded, SURVEY §8e
 * option B): context d runs the modular stages for its contiguous block of
 * K/G primes; one exchange gives every context all K residues of its block of
 * ceil(N/G) coefficients; each lifts its block by CRT and writes its rows of
 * `out`.  When every context can reach every other's memory (peer access over
 * NVLink, or contexts sharing a device) the exchange is folded into the
 * interpolation: its epilogue stores each residue straight into the owning
 * context's CRT input (CKB_EXCHANGE=nccl / copy: the separate step).  Same
 * arguments, result and status as ckb_biv_resultant; device_ms is the maximum
 * over the contexts. */
int ckb_biv_resultant_multi(const uint32_t* limbs, int C, int L, const int16_t* degs, int m, int n, int dfx, int dgx,
                            const uint32_t* primes, const uint32_t* gens, int K, int N, int LW, int G, uint32_t* out,
                            uint32_t* status, float* device_ms);

/* A batch of 1-4 independent res_y problems in one call (SURVEY.md §8(f) #1:
 * bisolve.biproject's res_y and res_x, bisolve.py:107-108): every argument of
 * ckb_biv_resultant becomes an array indexed by problem (pointer arrays for the
 * buffers); each problem's pipeline runs on its own stream so their kernels
 * overlap, and the call returns once all are done.  status [P]. */
int ckb_biv_resultant_batch(int P, const uint32_t* const* limbs, const int* C, const int* L,
                            const int16_t* const* degs, const int* m, const int* n, const int* dfx, const int* dgx,
                            const uint32_t* const* primes, const uint32_t* const* gens, const int* K, const int* N,
                            const int* LW, uint32_t* const* out, uint32_t* status);

/* K1: residues of every coefficient mod every prime — replaces
 * `[[c % p for c in cf] for cf in fc]` (modpoly.py:376-377).
 *   limbs [C][L] -> out [K][C] */
int ckb_reduce(const uint32_t* limbs, int C, int L, const uint32_t* primes, int K, uint32_t* out);

/* Batch of univariate resultants mod p — replaces _zp_resultant / zp_resultant_uni
 * (modpoly.py:132-161).  fa, gb [B][W] low-first residues (< p), da/db their
 * trimmed degrees (-1 = zero polynomial -> result 0), pidx [B] index into
 * primes [P].  W <= 4096 (one warp per pair, operands in shared memory). */
int ckb_uni_resultant_batch(const uint32_t* fa, const int32_t* da, const uint32_t* gb, const int32_t* db, int W,
                            const uint32_t* primes, int P, const int32_t* pidx, int B, uint32_t* out);

/* The planned evaluation points x_t = q^t (t < N) for each prime. */
int ckb_interp_plan_points(const uint32_t* primes, const uint32_t* gens, int K, int N, uint32_t* xpts);

/* Interpolation at the planned points — replaces _zp_interp (modpoly.py:164-185)
 * on the pipeline's point set.  values [K][N] at x_t = q^t -> coeffs [K][N]. */
int ckb_interp_geometric(const uint32_t* values, const uint32_t* primes, const uint32_t* gens, int K, int N,
                         uint32_t* coeffs);

/* Mixed-radix CRT + symmetric lift — replaces _CrtAccumulator.add/symmetric and
 * crt_reconstruct (modpoly.py:264-300).  residues [K][N] -> out [N][LW]. */
int ckb_crt_lift(const uint32_t* residues, int K, int N, const uint32_t* primes, int LW, uint32_t* out);

/* Batch of monic gcds mod p — replaces _zp_gcd (modpoly.py:115-122), the
 * per-prime step of int_gcd_uni (:307-341).  fa [B][Wf], gb [B][Wg] low-first
 * residues with trimmed degrees da/db (-1 = zero); out [B][Wo] monic gcd,
 * odeg [B] its degree (-1 if both inputs are zero). */
int ckb_gcd_mod_batch(const uint32_t* fa, const int32_t* da, int Wf, const uint32_t* gb, const int32_t* db, int Wg,
                      const uint32_t* primes, int P, const int32_t* pidx, int B, uint32_t* out, int Wo,
                      int32_t* odeg);

/* Interpolation at arbitrary distinct points — replaces _zp_interp /
 * zp_interpolate (modpoly.py:164-189).  xs, vs [B][W] (points reduced mod p),
 * ns [B] point counts (<= W <= 12288) -> out [B][W] coefficients (low first). */
int ckb_interp_points(const uint32_t* xs, const uint32_t* vs, const int32_t* ns, int W, const uint32_t* primes, int P,
                      const int32_t* pidx, int B, uint32_t* out);

/* Principal subresultant coefficients psc_i(t) mod p, i = 1..n, at the points
 * t = 0..ncand-1 — the values _psc_det (modpoly.py:477-501) gives at each point
 * of modular_subres_profile, read off one remainder sequence per point (one warp
 * each).  fres [(m+1)][(dfx+1)], gres [(n+1)][(dgx+1)]:
 * residues of the y-coefficients (m >= n, as the reference swaps), fdeg/gdeg
 * their x-degrees.  out [n][ncand]; valid [ncand] = 1 where neither leading
 * coefficient vanishes at t (the reference skips those t; their values are 0). */
int ckb_psc_values(const uint32_t* fres, const int16_t* fdeg, int m, int dfx, const uint32_t* gres,
                   const int16_t* gdeg, int n, int dgx, uint32_t p, int ncand, uint32_t* out, uint8_t* valid);

#define CKB_STATUS_UNLUCKY 2 /* UnluckyPrime(p) (modpoly.py:439, :451, :463) */

/* The whole modular subresultant degree profile on the device — replaces the
 * body of curvekit.modpoly.modular_subres_profile (modpoly.py:428-474) after its
 * reduction and swap: the reference's points, every psc_i at every point
 * (remainder sequences), every psc_i interpolated, and the gcd chain
 * S_0 = rstar mod p, S_i = gcd(S_{i-1}, psc_i).  rmod [rlen]: rstar mod p
 * (low first); rlen_int = rstar's length over Z (S_0 must keep it); dmax =
 * max(deg_x f, deg_x g).  chain [n+1] = deg S_i.  Returns CKB_STATUS_UNLUCKY
 * where the reference raises UnluckyPrime(p). */
int ckb_subres_profile(const uint32_t* fres, const int16_t* fdeg, int m, int dfx, const uint32_t* gres,
                       const int16_t* gdeg, int n, int dgx, const uint32_t* rmod, int rlen, int rlen_int, int dmax,
                       uint32_t p, int32_t* chain);

/* Images of the dense modular bivariate gcd — the modular core that replaces
 * the primitive PRS of curvekit.bivpoly.gcd_biv (pkg/src/curvekit/bivpoly.py:266-295;
 * used by is_squarefree_biv / square_part :307-320 and bisolve.py:110).
 *   limbs [C][L]: A's dense grid A[j][i] (x^i y^j, j <= m, i <= dax), B's grid
 *          (j <= n, i <= dbx), then Gamma = gcd(lc_y A, lc_y B) (dgam + 1 coefficients);
 *          C = (m+1)(dax+1) + (n+1)(dbx+1) + dgam + 1, m >= n >= 0
 *   degs  [m+n+2] trimmed x-degree of each y-coefficient of A then B (-1 = zero)
 *   out   [K][NP][Wo] (Wo > m): Gamma(x_t) * monic gcd(A(x_t, y), B(x_t, y)) mod p_k at
 *          x_t = t + 1, low degree first; odeg [K][NP] its degree, -2 where lc_y A or
 *          lc_y B vanishes at x_t (the point is unusable). */
int ckb_biv_gcd_images(const uint32_t* limbs, int C, int L, const int16_t* degs, int m, int n, int dax, int dbx,
                       int dgam, const uint32_t* primes, int K, int NP, uint32_t* out, int Wo, int32_t* odeg);

/* Descartes test of real-root isolation — replaces upoly._variations_on
 * (pkg/src/curvekit/upoly.py:338-346; compose_linear :202-212, taylor_shift
 * :193-199, sign_variations :215-224), the inner loop of descartes_isolate
 * (:358-408).  prepare: the polynomial's limbs [n+1][L] (low degree first) and
 * K primes (< 2^30, 1 mod the NTT length 2^ceil(log2(2n+1)), e.g. PRIMES30) with
 * generators; returns a handle >= 0.  variations: aw = [a limbs][w limbs] (AL
 * words each, unsigned) of the numerators a = a_num, w = b_num - a_num, ld = the
 * common log2 denominator; uses the first K primes of the handle (their product
 * must exceed 4x the coefficient bound of the shifted polynomial) and writes the
 * exact sign-variation count of taylor_shift(reversed(compose_linear(p, a, w, ld)), 1). */
int ckb_descartes_prepare(const uint32_t* limbs, int n, int L, const uint32_t* primes, const uint32_t* gens, int K);
int ckb_descartes_variations(int handle, const uint32_t* aw, int AL, int ld, int K, int LW, int32_t* variations);
int ckb_descartes_release(int handle);
/* B intervals of one handle in one call (a breadth-first isolation tests a whole
 * subdivision level at once): aw [B][2][AL], ld [B], variations [B]; K and LW
 * must cover the largest bound of the batch (1 <= B <= 4096). */
int ckb_descartes_variations_batch(int handle, const uint32_t* aw, int AL, const int32_t* ld, int B, int K, int LW,
                                   int32_t* variations);

/* Device-pointer stages for the multi-GPU driver (one process per GPU); primes
 * and gens are HOST arrays (they key the cached interpolation plan).
 * stream: a cudaStream_t or NULL for the context stream.
 * modular_images: limbs/degs on device (h_degs: host copy) -> d_coeffs [K][N]
 * residues of res's coefficients for this rank's primes. */
int ckb_dev_modular_images(const uint32_t* d_limbs, int C, int L, const int16_t* d_degs, const int16_t* h_degs, int m,
                           int n, int dfx, int dgx, const uint32_t* primes, const uint32_t* gens, int K, int N,
                           uint32_t* d_coeffs, uint32_t* d_status, void* stream);
int ckb_dev_crt(const uint32_t* d_coeffs, int K, int N, const uint32_t* primes, int LW, uint32_t* d_out,
                void* stream);

/* Whole pipeline on device buffers (inputs already resident in HBM):
 * same arguments as ckb_biv_resultant with d_ pointers; d_out [N][LW]. */
int ckb_dev_biv_resultant(const uint32_t* d_limbs, int C, int L, const int16_t* d_degs, const int16_t* h_degs, int m,
                          int n, int dfx, int dgx, const uint32_t* primes, const uint32_t* gens, int K, int N, int LW,
                          uint32_t* d_out, uint32_t* d_status, void* stream);

/* Page-locked host memory.  ckb_biv_resultant copies straight from / into
 * page-locked limbs / out buffers (no staging memcpy); these allocate and free
 * such buffers (NULL on failure). */
void* ckb_host_alloc(unsigned long long bytes);
int ckb_host_free(void* p);

/* Instrumentation: record CUDA events between the stages of the next pipeline
 * calls; ckb_stage_times returns the durations (ms) of reduce, plan, images,
 * interpolation, CRT for the last call (count returned). */
int ckb_set_timing(int on);
/* Internal graph replay on (1, default) or off (0): off while a caller captures
 * the library's launches into its own CUDA graph (e.g. a whole multi-GPU step
 * with its NCCL collective), so they are recorded as plain kernel nodes. */
int ckb_set_graphs(int on);
int ckb_stage_times(float* ms, int max);

/* Roofline denominators measured on the current device (csrc/ckb_peak.cu):
 * out[0..n) = IMAD, IMAD.HI, IMAD.WIDE rates in T ops/s, then Shoup-pair and
 * three-product-Montgomery modular products in T products/s (n <= 5 used). */
int ckb_measure_peak(float* out, int n);

#ifdef __cplusplus
}
#endif
#endif

// Univariate resultant mod p, one thread per image, operands in registers.
//
// Behavioural reference: curvekit.modpoly._zp_resultant (pkg/src/curvekit/
// modpoly.py:132-153), the Euclidean remainder sequence
//     res(P_{i-1}, P_i) = (-1)^(d_{i-1} d_i) lc(P_i)^(d_{i-1} - d_{i+1}) res(P_i, r_i).
// This header computes the same value division-free on TOP-ALIGNED registers
// (X[i] = coefficient of degree deg X - i), so every elimination is a
// static-index register update.  (One elimination is one step of the Schur
// algorithm on the rank-2 displacement generators of the Sylvester matrix,
// PAPER.md:1384-1443, with generators that shrink as the degrees fall.)
//
// Division-free remainders P_{i+1} = prem(P_{i-1}, P_i) = L_i^{e_i} r_i, with
// L_i = lc(P_i) and e_i = d_{i-1} - d_i + 1, turn the reference's product into
//     res = sgn * prod_i L_i^{(d_{i-1} - d_{i+1}) - e_i d_i} * lc(P_K)^{d_{K-1}}
// (res(B, c R) = c^deg B res(B, R)); no scale factors need tracking.  On the
// GENERIC sequence (every remainder drops the degree by exactly one) the
// exponents are 2 - 2 d_i, so with running products T = prod L_i and
// Q = prod_j T_j (which equals prod L_i^{d_i}) the whole bookkeeping is two
// Montgomery products per remainder and one inverse per image.  The two
// elimination steps of a generic remainder are fused into one sweep:
//     D''[i] = L^2 D[i+2] - L lc(D) V[i+2] - lc(D') V[i+1]      (3 products)
// Arithmetic is lazy: for p < 2^30 every register holds a value in [0, 4p)
// (entries beyond a degree are only congruent to 0), a Shoup product accepts
// any 32-bit input, and the fused remainder sums its three products in 64 bits
// before one Montgomery reduction, so no reduction is needed per output.
// A non-generic image (a leading coefficient vanishing mid-way) returns
// CKB_FAIL and is recomputed by the general warp kernel.
#pragma once
#include "ckb_modarith.cuh"

namespace ckb {

constexpr uint32_t CKB_FAIL = 0xffffffffu;

__device__ __forceinline__ uint32_t red4(uint32_t x, uint32_t p) {  // [0, 4p) -> [0, p)
  return red1(red1(x, 2u * p), p);
}
__device__ __forceinline__ uint32_t to_mont(uint32_t a, const Prime& P) { return redc((uint64_t)a * P.r2, P); }
__device__ __forceinline__ uint32_t mmul(uint32_t a, uint32_t b, const Prime& P) { return redc((uint64_t)a * b, P); }
__device__ __forceinline__ uint32_t mpow(uint32_t a, int e, uint32_t one, const Prime& P) {
  uint32_t r = one;
  while (e > 0) {
    if (e & 1) r = mmul(r, a, P);
    e >>= 1;
    if (e) a = mmul(a, a, P);
  }
  return r;
}
// Shoup companion from a Montgomery form wm = w R mod p
__device__ __forceinline__ uint32_t comp_from_mont(uint32_t wm, const Prime& P) { return (0u - wm) * P.pinv; }

// (a x + b y + c z) R^-1 mod p, lazily in (0, 4p): three products summed in
// 64 bits (IMAD.WIDE chain), one signed Montgomery reduction (+p keeps it positive)
__device__ __forceinline__ uint32_t mont3(uint32_t x, uint32_t a, uint32_t y, uint32_t b, uint32_t z, uint32_t c,
                                          uint32_t pinv, uint32_t p) {
  const uint64_t t = (uint64_t)x * a + (uint64_t)y * b + (uint64_t)z * c;
  return (uint32_t)(t >> 32) - __umulhi((uint32_t)t * pinv, p) + p;
}

// step2 with an exact trip count at run time: outputs i = 0 .. k-1 in
// ascending order (each reads D[i+2] before it is overwritten), the loop
// leaving through a uniform branch right after output k-1 and zeroing D[k]
// (the one entry past the new degree the next step reads).  Code size is one
// copy of the sweep per role (the compile-time chain unrolls every k: ~100 KB
// of SASS, instruction-cache misses).
// outputs I, I+1, ... while below k, each followed by the uniform exit test;
// the exit zeroes D[k] (also at k = MAXD - 1, past the last computable output)
template <int MAXD, int I>
__device__ __forceinline__ void sweep_exit(uint32_t (&D)[MAXD + 1], const uint32_t (&V)[MAXD + 1], int k, uint32_t w1m,
                                           uint32_t w2m, uint32_t w3m, uint32_t pinv, uint32_t p) {
  if constexpr (I < MAXD) {
    if (I >= k) {
      D[I] = 0u;
    } else if constexpr (I < MAXD - 1) {
      D[I] = mont3(D[I + 2], w1m, V[I + 2], w2m, V[I + 1], w3m, pinv, p);
      sweep_exit<MAXD, I + 1>(D, V, k, w1m, w2m, w3m, pinv, p);
    }
  }
}
template <int MAXD>
__device__ __forceinline__ uint32_t step2_exit(uint32_t (&D)[MAXD + 1], const uint32_t (&V)[MAXD + 1], int k,
                                               const Prime& P) {
  const uint32_t p = P.p;
  const uint32_t lb = red4(V[0], p), la = red4(D[0], p);
  const uint32_t nla = la ? p - la : 0u;
  const uint32_t d1 = red4(D[1], p), v1 = red4(V[1], p);
  const uint32_t w1m = redc((uint64_t)lb * lb, P);
  const uint32_t w2m = redc((uint64_t)lb * nla, P);
  const uint32_t l3 = redc((uint64_t)lb * d1 + (uint64_t)nla * v1, P);
  const uint32_t w3m = l3 ? p - l3 : 0u;
  const uint32_t pinv = P.pinv;
  sweep_exit<MAXD, 0>(D, V, k, w1m, w2m, w3m, pinv, p);
  return lb;
}

// single division-free step D <- lb D - lc(D) V (aligned tops); nom = nominal deg D
template <int MAXD>
__device__ __forceinline__ void step1(uint32_t (&D)[MAXD + 1], const uint32_t (&V)[MAXD + 1], int nom, uint32_t lb,
                                      uint32_t lbc, const Prime& P) {
  const uint32_t p = P.p;
  const uint32_t la = red4(D[0], p);
  const uint32_t nla = la ? p - la : 0u;
  const uint32_t nlac = comp_from_mont(to_mont(nla, P), P);
#pragma unroll
  for (int c = 0; c < (MAXD + 3) / 4; ++c) {
    if (4 * c <= nom) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = 4 * c + k;
        if (i < MAXD) D[i] = shoup_lazy(D[i + 1], lb, lbc, p) + shoup_lazy(V[i + 1], nla, nlac, p);
      }
    }
  }
  D[MAXD] = 0u;
}

// fused generic remainder: D (nominal deg k+1) <- R^-2 prem(D, V) (deg k-1), V
// of deg k.  The three multipliers are formed with one REDC each, so they
// carry a factor R^-1 and the single reduction of the update another; the
// caller compensates the R^-2 with R^{2k} (res(V, c X) = c^{deg V} res(V, X)).
// Returns lc(V) (canonical: the running products absorb one R^-1 per step,
// compensated once at the end).
template <int MAXD>
__device__ __forceinline__ uint32_t step2(uint32_t (&D)[MAXD + 1], const uint32_t (&V)[MAXD + 1], int k,
                                          const Prime& P) {
  const uint32_t p = P.p;
  const uint32_t lb = red4(V[0], p), la = red4(D[0], p);
  const uint32_t nla = la ? p - la : 0u;
  // R^-1 (lb^2, -lb la, -la') with la' = lb D[1] - la V[1] the lc of the intermediate remainder
  const uint32_t d1 = red4(D[1], p), v1 = red4(V[1], p);
  const uint32_t w1m = redc((uint64_t)lb * lb, P);
  const uint32_t w2m = redc((uint64_t)lb * nla, P);
  const uint32_t l3 = redc((uint64_t)lb * d1 + (uint64_t)nla * v1, P);
  const uint32_t w3m = l3 ? p - l3 : 0u;
  const uint32_t pinv = P.pinv;
  // outputs i < k are the new coefficients; i = k, k+1 held the old tail and
  // must become 0 (later sweeps read one entry past a degree), so chunks up to
  // index k+1 are written, but only entries below k are computed
#ifndef CKB_SWEEP_CHUNK
#define CKB_SWEEP_CHUNK 4
#endif
  constexpr int CW = CKB_SWEEP_CHUNK;  // entries per uniform guard
#pragma unroll
  for (int c = 0; c < (MAXD + CW - 1) / CW; ++c) {
    if (CW * c <= k + 1) {
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const int i = CW * c + j;
        if (i < MAXD - 1) {
          if (i < k) {
            // inputs < 4p < 2^32, multipliers < p: t < 12 p^2 < 2^64, result in (0, 4p)
            D[i] = mont3(D[i + 2], w1m, V[i + 2], w2m, V[i + 1], w3m, pinv, p);
          } else {
            D[i] = 0u;
          }
        }
      }
    }
  }
  D[MAXD - 1] = 0u;
  D[MAXD] = 0u;
  return lb;
}

// The fused remainders with the divisor degree K a COMPILE-TIME constant, the
// whole chain unrolled (K, K-1, ..., 1, roles alternating): every chunk guard
// and every `i < k` test folds, so a step issues exactly its k outputs (the
// run-time loop issues whole chunks and predicates the tail off: ~3.5 wasted
// outputs per step, 17% of the elimination at r = 80).
template <int MAXD, int K, bool BA>  // BA: dividend B, divisor A
__device__ __forceinline__ void chain_exact(uint32_t (&A)[MAXD + 1], uint32_t (&B)[MAXD + 1], uint32_t& T, uint32_t& Q,
                                            uint32_t& num, bool& bad, const Prime& P) {
  if constexpr (K >= 1) {
    const uint32_t lm = BA ? step2<MAXD>(B, A, K, P) : step2<MAXD>(A, B, K, P);
    T = mmul(T, lm, P);
    Q = mmul(Q, T, P);
    const uint32_t d0 = red4(BA ? B[0] : A[0], P.p);
    bad |= (d0 == 0u);
    if constexpr (K == 1) {
      num = mmul(num, to_mont(d0, P), P);
    } else {
      chain_exact<MAXD, K - 1, !BA>(A, B, T, Q, num, bad, P);
    }
  }
}

// res(A, B) for top-aligned A (deg da) and B (deg db), da >= db >= 1 with
// nonzero leading coefficients; `neg` carries the sign of an initial swap.
// Returns CKB_FAIL on a non-generic remainder sequence.  DB > 0: the caller
// guarantees db == DB (the chain is unrolled for it).
#ifndef CKB_STEP_EXIT
#define CKB_STEP_EXIT 1
#endif
template <int MAXD, int DB = 0>
__device__ __forceinline__ uint32_t resultant_generic(uint32_t (&A)[MAXD + 1], int da, uint32_t (&B)[MAXD + 1], int db,
                                                      bool neg, const Prime& P) {
  const uint32_t p = P.p;
  const uint32_t one = redc(P.r2, P);  // R mod p
  // first remainder: e0 single steps (e0 = 1 for m = n)
  const uint32_t lb = red4(B[0], p);
  const uint32_t lbm = to_mont(lb, P);
  const uint32_t lbc = comp_from_mont(lbm, P);
  // Control flow depends only on (da, db), which are the same for every lane
  // of the launch: a lane whose sequence turns out non-generic keeps running
  // the (now meaningless) generic schedule with `bad` set, so every loop
  // bound and chunk guard stays warp-uniform (no divergence scaffolding).
  bool bad = false;
  const int e0 = da - db + 1;
  for (int s = 0; s < e0; ++s) step1<MAXD>(A, B, da - s, lb, lbc, P);
  uint32_t a0 = red4(A[0], p);
  bad |= (a0 == 0u);
  neg ^= (bool)(da & db & 1);
  const uint32_t l1e = mpow(lbm, e0, one, P);
  uint32_t num = l1e, den = mpow(l1e, db, one, P);
  uint32_t T = one, Q = one;
  int k = db - 1;
  if (k == 0) {
    num = mmul(num, to_mont(a0, P), P);  // lc(P_K)^(d_{K-1}), d_{K-1} = db = 1
  } else if constexpr (DB > 1) {
    chain_exact<MAXD, DB - 1, true>(A, B, T, Q, num, bad, P);
    num = mmul(num, mmul(T, T, P), P);
    den = mmul(den, mmul(Q, Q, P), P);
  } else {
    for (;;) {
      // dividend B (deg k+1), divisor A (deg k)
      uint32_t lm = CKB_STEP_EXIT ? step2_exit<MAXD>(B, A, k, P) : step2<MAXD>(B, A, k, P);
      T = mmul(T, lm, P);
      Q = mmul(Q, T, P);
      --k;
      const uint32_t b0 = red4(B[0], p);
      bad |= (b0 == 0u);
      if (k == 0) {
        num = mmul(num, to_mont(b0, P), P);
        break;
      }
      // dividend A (deg k+1), divisor B (deg k)
      lm = CKB_STEP_EXIT ? step2_exit<MAXD>(A, B, k, P) : step2<MAXD>(A, B, k, P);
      T = mmul(T, lm, P);
      Q = mmul(Q, T, P);
      --k;
      a0 = red4(A[0], p);
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
  // Compensation, one power of R: each fused remainder with divisor degree k
  // was stored as R^-2 prem (factor R^{2 sum k} = R^{db (db - 1)}), and the
  // running products took the canonical L_i (T_j carries R^-j, Q_J carries
  // R^-J(J+1)/2 with J = db - 1 steps), which scales num / den by R^{J(J-1)};
  // together R^{db (db - 1) - (db - 1)(db - 2)} = R^{2 (db - 1)}
  // (in Montgomery form: mpow of R^2 mod p)
  const uint32_t corr = mpow(P.r2, 2 * (db - 1), one, P);
  // num / den (Fermat inverse in the Montgomery domain), leave the domain
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

// shift a top-aligned register array up by one position (the leading entry was 0)
template <int MAXD>
__device__ __forceinline__ void shift_up(uint32_t (&D)[MAXD + 1]) {
#pragma unroll
  for (int i = 0; i < MAXD; ++i) D[i] = D[i + 1];
  D[MAXD] = 0u;
}

// one pseudo-remainder of the dividend D (deg dd) by V (deg dv >= 1), D <- prem(D, V)
// by e = dd - dv + 1 single eliminations, then the leading zeros shifted out;
// returns the remainder's degree (-1: zero remainder).  An elimination whose
// quotient term is zero (lc(D) = 0 in every converged lane: the y -> y^2
// structured inputs have one per remainder) only shifts D instead of scaling it
// by lb: the remainder is then prem / lb^skip, which the caller's power of lb
// absorbs (res(V, c R) = c^deg V res(V, R)); *skip counts those steps.
template <int MAXD>
__device__ __forceinline__ int prem_any(uint32_t (&D)[MAXD + 1], const uint32_t (&V)[MAXD + 1], int dd, int dv,
                                        uint32_t lb, uint32_t lbc, const Prime& P, int* skip) {
  *skip = 0;
  // two-term quotient with a vanishing middle term in every converged lane (degree drop 2 of a
  // y -> y^2 input): both eliminations fused into one pass of three products per output,
  //   D'[i] = lb^2 D[i+3] - lb la V[i+3] - l2 V[i+1],  l2 = lb D[2] - la V[2],
  // the same values as the single steps with the middle one skipped (multipliers in
  // Montgomery form so mont3 returns them exactly, lazily in (0, 4p))
  if (dd - dv == 2 && dv >= 1 && MAXD >= 3) {
    const uint32_t p = P.p;
    const uint32_t la = red4(D[0], p);
    const bool mid0 = mul_mod(lb, red4(D[1], p), P) == mul_mod(la, red4(V[1], p), P);
    if (__all_sync(__activemask(), mid0)) {
      const uint32_t l2 = sub_mod(mul_mod(lb, red4(D[2], p), P), mul_mod(la, red4(V[2], p), P), p);
      const uint32_t w1m = to_mont(mul_mod(lb, lb, P), P);
      const uint32_t w2m = to_mont(neg_mod(mul_mod(lb, la, P), p), P);
      const uint32_t w3m = to_mont(neg_mod(l2, p), P);
#pragma unroll
      for (int c = 0; c < (MAXD + 3) / 4; ++c) {
        if (4 * c <= dd) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int i = 4 * c + k;
            if (i < MAXD - 2) D[i] = mont3(D[i + 3], w1m, V[i + 3], w2m, V[i + 1], w3m, P.pinv, p);
          }
        }
      }
      D[MAXD - 2] = 0u;  // beyond the new nominal degree dd - 3
      D[MAXD - 1] = 0u;
      D[MAXD] = 0u;
      *skip = 1;
      int dr = dv - 1;
      while (dr >= 0 && red4(D[0], p) == 0u) {
        shift_up<MAXD>(D);
        --dr;
      }
      return dr;
    }
  }
  for (int s = 0; s <= dd - dv; ++s) {
    if (__all_sync(__activemask(), red4(D[0], P.p) == 0u)) {
      shift_up<MAXD>(D);
      ++*skip;
    } else {
      step1<MAXD>(D, V, dd - s, lb, lbc, P);
    }
  }
  int dr = dv - 1;
  while (dr >= 0 && red4(D[0], P.p) == 0u) {
    shift_up<MAXD>(D);
    --dr;
  }
  return dr;
}

// res(A, B) for top-aligned A (deg da) and B (deg db), da >= db >= 1, nonzero
// leading coefficients, ANY degree pattern of the remainder sequence (the
// structured inputs whose subresultant coefficients vanish identically: every
// image of F(x, y^2) drops the degree by two).  The reference's recursion
// (modpoly.py:138-152) with division-free remainders: prem(A, B) = lb^e rem(A, B),
// e = da - db + 1, so res(A, B) = (-1)^(da db) lb^(da - dr) res(B, rem)
//                              = (-1)^(da db) lb^(da - dr - e db) res(B, prem).
// Two register arrays swap roles in a loop written twice (static indices only).
template <int MAXD>
__device__ __forceinline__ uint32_t resultant_anydeg(uint32_t (&A)[MAXD + 1], int da, uint32_t (&B)[MAXD + 1], int db,
                                                     bool neg, const Prime& P) {
  const uint32_t p = P.p;
  const uint32_t one = redc(P.r2, P);  // R mod p
  uint32_t num = one, den = one;       // Montgomery form
  for (;;) {
    // dividend A (deg da), divisor B (deg db >= 1)
    {
      const uint32_t lb = red4(B[0], p);
      const uint32_t lbm = to_mont(lb, P), lbc = comp_from_mont(lbm, P);
      int skip;
      const int e = da - db + 1;
      const int dr = prem_any<MAXD>(A, B, da, db, lb, lbc, P, &skip);
      if (dr < 0) return 0u;  // a common factor
      neg ^= (bool)(da & db & 1);
      {  // lb^(da - dr) / lb^((e - skip) db): one power, into num or den by the exponent's sign
        const int x = (da - dr) - (e - skip) * db;
        if (x >= 0)
          num = mmul(num, mpow(lbm, x, one, P), P);
        else
          den = mmul(den, mpow(lbm, -x, one, P), P);
      }
      da = dr;
      if (da == 0) {  // res(B, c) = c^db
        num = mmul(num, mpow(to_mont(red4(A[0], p), P), db, one, P), P);
        break;
      }
    }
    // dividend B (deg db), divisor A (deg da >= 1)
    {
      const uint32_t lb = red4(A[0], p);
      const uint32_t lbm = to_mont(lb, P), lbc = comp_from_mont(lbm, P);
      int skip;
      const int e = db - da + 1;
      const int dr = prem_any<MAXD>(B, A, db, da, lb, lbc, P, &skip);
      if (dr < 0) return 0u;
      neg ^= (bool)(da & db & 1);
      {
        const int x = (db - dr) - (e - skip) * da;
        if (x >= 0)
          num = mmul(num, mpow(lbm, x, one, P), P);
        else
          den = mmul(den, mpow(lbm, -x, one, P), P);
      }
      db = dr;
      if (db == 0) {
        num = mmul(num, mpow(to_mont(red4(B[0], p), P), da, one, P), P);
        break;
      }
    }
  }
  // num / den in the Montgomery domain (Fermat inverse), then leave it
  uint32_t inv = one, b = den;
  uint32_t ex = p - 2;
  while (ex) {
    if (ex & 1) inv = mmul(inv, b, P);
    ex >>= 1;
    if (ex) b = mmul(b, b, P);
  }
  const uint32_t r = redc((uint64_t)mmul(num, inv, P), P);
  return neg ? neg_mod(r, p) : r;
}

// Lazy Shoup-Horner evaluation of a residue polynomial c[0..deg] at x: [0, 3p)
__device__ __forceinline__ uint32_t horner_lazy(const uint32_t* c, int deg, uint32_t x, uint32_t xc, uint32_t p) {
  if (deg < 0) return 0u;
  uint32_t acc = c[deg];
  for (int i = deg - 1; i >= 0; --i) acc = shoup_lazy(acc, x, xc, p) + c[i];
  return acc;
}

}  // namespace ckb

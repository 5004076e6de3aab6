// Univariate resultant mod p, one thread per image, operands in registers.
//
// Behavioural reference: curvekit.modpoly._zp_resultant (pkg/src/curvekit/
// modpoly.py:132-153), the Euclidean remainder sequence
//     res = prod_i (-1)^(d_{i-1} d_i) lc(R_i)^(d_{i-1} - d_{i+1}) * lc(R_K)^(d_{K-1}).
// Here the sequence is computed division-free.  Both operands are kept
// TOP-ALIGNED in registers (X[i] = coefficient of degree deg X - i), so one
// elimination step is the same static-index register update for every
// degree difference:
//     A[i] <- lc(B) * A[i+1] - A[0] * B[i+1]
// (this is one step of the Schur algorithm on the rank-2 displacement
// generators of the Sylvester matrix, with the generators
// shrinking as the degrees fall and the zero-pivot case handled by look-ahead
// = a degree drop larger than one).  With P_i = c_i R_i the pseudo-remainders,
//     P_{i+1} = lc(P_i)^{e_i} c_{i-1} R_{i+1},  e_i = d_{i-1} - d_i + 1,
// so the reference product is rebuilt from lc(P_i) and c_i with a handful of
// Montgomery products per remainder and ONE inverse per image.
#pragma once
#include "ckb_modarith.cuh"

namespace ckb {

// Montgomery-domain helpers for the bookkeeping scalars
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

// one division-free elimination step on top-aligned registers; `nom` is the
// nominal degree of A before the step (entries beyond it are zero)
template <int MAXD>
__device__ __forceinline__ void elim_step(uint32_t (&A)[MAXD + 1], const uint32_t (&B)[MAXD + 1], int nom,
                                          uint32_t L, uint32_t Lc, const Prime& P) {
  const uint32_t p = P.p;
  const uint32_t nla = neg_mod(A[0], p);
  const uint32_t nlac = shoup_comp(nla, P);
#pragma unroll
  for (int c = 0; c < (MAXD + 3) / 4; ++c) {
    if (4 * c <= nom) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int i = 4 * c + k;
        if (i < MAXD) {
          uint32_t u = red1(shoup_lazy(A[i + 1], L, Lc, p), p);
          uint32_t v = red1(shoup_lazy(B[i + 1], nla, nlac, p), p);
          A[i] = red1(u + v, p);
        }
      }
    }
  }
  A[MAXD] = 0u;
}

// shift A up until its top entry is nonzero; returns the true degree (-1: zero)
template <int MAXD>
__device__ __forceinline__ int normalize(uint32_t (&A)[MAXD + 1], int d) {
  while (d >= 0 && A[0] == 0u) {
#pragma unroll
    for (int i = 0; i < MAXD; ++i) A[i] = A[i + 1];
    A[MAXD] = 0u;
    --d;
  }
  return d;
}

// Pseudo-remainder of (A, da) by (B, db) in place in A; bookkeeping of the
// reference product.  Returns the degree of the remainder (-1 if zero).
template <int MAXD>
__device__ __forceinline__ int prem_and_account(uint32_t (&A)[MAXD + 1], int da, uint32_t cA,
                                                const uint32_t (&B)[MAXD + 1], int db, uint32_t cB,
                                                uint32_t& num, uint32_t& den, uint32_t& cR, bool& neg,
                                                uint32_t one, const Prime& P) {
  const uint32_t L = B[0];
  const uint32_t Lc = shoup_comp(L, P);
  const int e = da - db + 1;
  int nom = da;
  for (int s = 0; s < e; ++s) {
    elim_step<MAXD>(A, B, nom, L, Lc, P);
    --nom;
  }
  const int dr = normalize<MAXD>(A, db - 1);
  if (dr < 0) return -1;
  neg ^= (bool)(da & db & 1);
  const int x = da - dr;
  const uint32_t Lm = to_mont(L, P);
  if (x == 2 && e == 2) {  // the generic step
    const uint32_t L2 = mmul(Lm, Lm, P);
    num = mmul(num, L2, P);
    den = mmul(den, mmul(cB, cB, P), P);
    cR = mmul(L2, cA, P);
  } else {
    num = mmul(num, mpow(Lm, x, one, P), P);
    den = mmul(den, mpow(cB, x, one, P), P);
    cR = mmul(mpow(Lm, e, one, P), cA, P);
  }
  return dr;
}

// res(A, B) for top-aligned A (deg da) and B (deg db), da >= db >= 1, both
// leading coefficients nonzero; `neg` carries the sign of an initial swap.
template <int MAXD>
__device__ __forceinline__ uint32_t resultant_topaligned(uint32_t (&A)[MAXD + 1], int da, uint32_t (&B)[MAXD + 1],
                                                         int db, bool neg, const Prime& P) {
  const uint32_t one = redc(P.r2, P);  // R mod p = Montgomery 1
  uint32_t num = one, den = one, cA = one, cB = one, cR = one, resm;
  for (;;) {
    // (A, da, cA) dividend, (B, db, cB) divisor, db >= 1
    int dr = prem_and_account<MAXD>(A, da, cA, B, db, cB, num, den, cR, neg, one, P);
    if (dr < 0) return 0u;
    if (dr == 0) {
      num = mmul(num, mpow(to_mont(A[0], P), db, one, P), P);
      den = mmul(den, mpow(cR, db, one, P), P);
      break;
    }
    // roles swap: (B, db, cB) dividend, (A, dr, cR) divisor
    uint32_t cR2 = one;
    int dr2 = prem_and_account<MAXD>(B, db, cB, A, dr, cR, num, den, cR2, neg, one, P);
    if (dr2 < 0) return 0u;
    if (dr2 == 0) {
      num = mmul(num, mpow(to_mont(B[0], P), dr, one, P), P);
      den = mmul(den, mpow(cR2, dr, one, P), P);
      break;
    }
    da = dr;
    db = dr2;
    cA = cR;
    cB = cR2;
  }
  // num / den, leave the Montgomery domain; Fermat inverse den^(p-2)
  uint32_t inv = one, b = den;
  uint32_t ex = P.p - 2;
  while (ex) {
    if (ex & 1) inv = mmul(inv, b, P);
    ex >>= 1;
    if (ex) b = mmul(b, b, P);
  }
  resm = mmul(num, inv, P);
  uint32_t r = redc((uint64_t)resm, P);
  return neg ? neg_mod(r, P.p) : r;
}

// Shoup-Horner evaluation of a residue polynomial c[0..deg] at x
__device__ __forceinline__ uint32_t horner(const uint32_t* c, int deg, uint32_t x, uint32_t xc, uint32_t p) {
  if (deg < 0) return 0u;
  uint32_t acc = c[deg];
  for (int i = deg - 1; i >= 0; --i) acc = red1(red1(shoup_lazy(acc, x, xc, p), p) + c[i], p);
  return acc;
}

}  // namespace ckb

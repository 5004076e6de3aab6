// Word-size modular arithmetic for odd primes 3 <= p < 2^31 on sm_100a.
//
// Measured on B200 (tools/imad_peak.cu, profiles/r01_imad_peak.json): IMAD runs
// at ~71 lanes/clk/SM but IMAD.WIDE.U32 and IMAD.HI.U32 at only ~23-25.  A
// product therefore costs what its *high-half* multiplies cost, and the kernels
// use Shoup multiplication by a fixed multiplier w (companion w' = floor(w*2^32/p)):
//     q = hi(x*w'), r = x*w - q*p  (mod 2^32)   -> r in [0, 2p)
// one IMAD.HI + two IMAD, valid for every 32-bit x.  General products (both
// operands varying, rare: bookkeeping, plans) use signed Montgomery REDC.
#pragma once
#include <cstdint>

namespace ckb {

struct Prime {
  uint32_t p;     // odd prime < 2^31
  uint32_t pinv;  // p^-1 mod 2^32
  uint32_t r2;    // 2^64 mod p
};

__host__ __device__ __forceinline__ uint32_t inv32(uint32_t p) {
  uint32_t x = p;  // Newton: correct to 3 bits for odd p
  for (int i = 0; i < 5; ++i) x *= 2u - p * x;
  return x;
}

// [0, 2p) -> [0, p) without a branch (unsigned wrap makes r - p huge if r < p)
__device__ __forceinline__ uint32_t red1(uint32_t r, uint32_t p) { return min(r, r - p); }

__device__ __forceinline__ uint32_t add_mod(uint32_t a, uint32_t b, uint32_t p) {
  return red1(a + b, p);  // a, b < p < 2^31
}
__device__ __forceinline__ uint32_t sub_mod(uint32_t a, uint32_t b, uint32_t p) {
  uint32_t d = a - b;
  return min(d, d + p);
}
__device__ __forceinline__ uint32_t neg_mod(uint32_t a, uint32_t p) { return a ? p - a : 0u; }

// signed Montgomery reduction: t < p * 2^32  ->  t * 2^-32 mod p in [0, p)
__device__ __forceinline__ uint32_t redc(uint64_t t, const Prime& P) {
  uint32_t m = (uint32_t)t * P.pinv;
  int32_t u = (int32_t)((uint32_t)(t >> 32) - __umulhi(m, P.p));
  return (uint32_t)(u + ((u >> 31) & (int32_t)P.p));
}

// general product a*b mod p (a, b < p): two REDCs
__device__ __forceinline__ uint32_t mul_mod(uint32_t a, uint32_t b, const Prime& P) {
  uint32_t t = redc((uint64_t)a * b, P);   // a b 2^-32
  return redc((uint64_t)t * P.r2, P);      // a b
}

// Shoup companion of w < p: floor(w * 2^32 / p) = (w*2^32 - (w*2^32 mod p)) / p,
// and exact division by odd p is multiplication by p^-1 mod 2^32.
__device__ __forceinline__ uint32_t shoup_comp(uint32_t w, const Prime& P) {
  uint32_t r = redc((uint64_t)w * P.r2, P);  // w * 2^32 mod p
  return (0u - r) * P.pinv;
}

// x * w mod p, lazily in [0, 2p); any 32-bit x.  Written as x w + q (-p) so
// that it compiles to IMAD.HI + IMAD + IMAD with no negation of q.
__device__ __forceinline__ uint32_t shoup_lazy(uint32_t x, uint32_t w, uint32_t wc, uint32_t p) {
  const uint32_t q = __umulhi(x, wc);
  return x * w + q * (0u - p);
}
// x * w + c mod p, lazily in [0, 2p) + c (the add folds into the first IMAD)
__device__ __forceinline__ uint32_t shoup_lazy_add(uint32_t x, uint32_t w, uint32_t wc, uint32_t negp, uint32_t c) {
  const uint32_t q = __umulhi(x, wc);
  return (x * w + c) + q * negp;
}
__device__ __forceinline__ uint32_t shoup(uint32_t x, uint32_t w, uint32_t wc, uint32_t p) {
  return red1(shoup_lazy(x, w, wc, p), p);
}

__device__ __forceinline__ uint32_t pow_mod(uint32_t a, uint64_t e, const Prime& P) {
  uint32_t r = 1u % P.p, b = a;
  while (e) {
    if (e & 1) r = mul_mod(r, b, P);
    b = mul_mod(b, b, P);
    e >>= 1;
  }
  return r;
}

__device__ __forceinline__ uint32_t inv_mod(uint32_t a, const Prime& P) {
  return pow_mod(a, P.p - 2, P);  // Fermat; a != 0
}

// x mod p for an arbitrary 32-bit x (Shoup with w = 1)
__device__ __forceinline__ uint32_t mod_word(uint32_t x, uint32_t one_comp, uint32_t p) {
  return shoup(x, 1u, one_comp, p);
}

// per-prime constants of limbs_mod: 2^32 mod p and companions, 2^(32 L) mod p
struct LimbModConst {
  uint32_t R1, R1c, onec, big;
};
__device__ __forceinline__ LimbModConst limbs_mod_const(int L, const Prime& P) {
  LimbModConst k;
  const uint32_t p = P.p;
  k.R1 = redc(P.r2, P);
  k.R1c = shoup_comp(k.R1, P);
  k.onec = shoup_comp(1u % p, P);
  uint32_t big = 1u % p;
  for (int l = 0; l < L; ++l) big = shoup(big, k.R1, k.R1c, p);
  k.big = big;
  return k;
}
// residue of an UNSIGNED integer of L little-endian 32-bit limbs
__device__ __forceinline__ uint32_t limbs_mod_k(const uint32_t* w, int L, uint32_t p, const LimbModConst& k) {
  uint32_t r = 0;
  for (int l = L - 1; l >= 0; --l) r = add_mod(shoup(r, k.R1, k.R1c, p), mod_word(w[l], k.onec, p), p);
  return r;
}

// Faster per-prime form for K1 (p < 2^30): three limbs at a time as ONE 64-bit sum
// w0 a0 + w1 a1 + w2 a2 (a_l = 2^(32(l+1)) mod p, i.e. 2^(32 l) in Montgomery form,
// so the sum is < 3 * 2^32 * p) and one Montgomery reduction into (0, 4p) -- about a
// quarter of the Shoup-Horner instructions per limb; blocks of three limbs are
// combined by Horner in 2^96.
struct LimbModFast {
  uint32_t a0, a1, a2, c96, c96c, big, pinv;
};
__device__ __forceinline__ LimbModFast limbs_mod_fast_const(int L, const Prime& P) {
  LimbModFast k;
  const uint32_t p = P.p;
  const uint32_t R1 = redc(P.r2, P), R1c = shoup_comp(R1, P);  // 2^32 mod p
  k.a0 = R1;
  k.a1 = shoup(k.a0, R1, R1c, p);
  k.a2 = shoup(k.a1, R1, R1c, p);
  k.c96 = k.a2;  // 2^96 mod p
  k.c96c = shoup_comp(k.c96, P);
  uint32_t big = 1u % p;
  for (int l = 0; l < L; ++l) big = shoup(big, R1, R1c, p);
  k.big = big;  // 2^(32 L) mod p
  k.pinv = P.pinv;
  return k;
}
__device__ __forceinline__ uint32_t mod3_fast(uint32_t w0, uint32_t w1, uint32_t w2, const LimbModFast& k,
                                              uint32_t p) {
  const uint64_t t = (uint64_t)w0 * k.a0 + (uint64_t)w1 * k.a1 + (uint64_t)w2 * k.a2;
  const uint32_t m = (uint32_t)t * k.pinv;
  uint32_t u = (uint32_t)(t >> 32) + p - __umulhi(m, p);  // in (0, 4p)
  u = u >= 2 * p ? u - 2 * p : u;
  return u >= p ? u - p : u;
}

// residue mod p of a two's-complement integer of L little-endian 32-bit limbs
__device__ __forceinline__ uint32_t limbs_mod(const uint32_t* w, int L, const Prime& P) {
  const uint32_t p = P.p;
  const uint32_t R1 = redc(P.r2, P);            // 2^32 mod p
  const uint32_t R1c = shoup_comp(R1, P);
  const uint32_t onec = shoup_comp(1u % p, P);
  uint32_t r = 0;
  for (int l = L - 1; l >= 0; --l) {
    r = add_mod(shoup(r, R1, R1c, p), mod_word(w[l], onec, p), p);
  }
  if (w[L - 1] >> 31) {  // negative: subtract 2^(32L) mod p
    uint32_t big = 1u % p;
    for (int l = 0; l < L; ++l) big = shoup(big, R1, R1c, p);
    r = sub_mod(r, big, p);
  }
  return r;
}

__device__ __forceinline__ Prime make_prime(uint32_t p) {
  Prime P;
  P.p = p;
  P.pinv = inv32(p);
  // 2^64 mod p via (2^32 mod p)^2
  uint64_t r1 = (uint64_t)(0x100000000ull % p);
  P.r2 = (uint32_t)((r1 * r1) % p);
  return P;
}

}  // namespace ckb

"""Algorithmic work model of the hot path (used for roofline reporting).

Two counts are kept apart:
  * ``images_products`` -- modular products the B200 algorithm performs
    (Shoup-Horner evaluation + division-free elimination), the work the
    images kernel must do; achieved = products / kernel time.  The peak is
    mix-weighted: Shoup-form products (evaluation, first remainder) at the
    measured Shoup-pair rate, fused-remainder products at the measured
    three-product Montgomery rate (csrc/ckb_peak.cu).
  * ``contract_imad`` -- SURVEY.md §8(d)'s fixed per-res_y figure
    W = 3 IMAD x [k N (E + 4 r (r + 1)) + k N^2 + N k (k - 1)/2 + C L k]
    (the Schur-algorithm count of PAPER.md's design), reported unchanged so
    the two can be compared.
"""

from __future__ import annotations


POLY = 8  # images per polyphase coset (csrc/ckb_images.cu)


def eval_products(degs_f, degs_g) -> int:
    """Horner steps of a plain per-point evaluation: sum of the x-degrees."""
    return sum(max(d, 0) for d in degs_f) + sum(max(d, 0) for d in degs_g)


def eval_products_poly(degs_f, degs_g, S: int = POLY) -> int:
    """Products per image of the polyphase evaluation: each lane of an S-lane
    coset runs Horner in y^S over its share of the coefficients (ceil((D+1)/S)
    terms of a degree-D poly: one product fewer than terms, the top term is a
    load), then one product by y^r and log2(S) - 1 DFT stages with products (the
    last stage's twiddle is 1)."""
    stages = S.bit_length() - 2
    tot = 0
    for d in list(degs_f) + list(degs_g):
        if d >= 0:
            tot += -(-(d + 1) // S) - 1 + 1 + stages
    return tot


def elim_products(m: int, n: int) -> int:
    """Vector products of the generic division-free elimination (ckb_resultant.cuh):
    the first remainder is e0 = da - db + 1 single steps (a step with nominal
    degree `nom` forms nom outputs of 2 products); every later remainder with
    divisor degree k is one fused sweep of k outputs of 3 products."""
    da, db = max(m, n), min(m, n)
    if db < 1:
        return 0
    total = sum(2 * (da - s) for s in range(da - db + 1))
    total += sum(3 * k for k in range(1, db))
    return total


def elim_split(m: int, n: int):
    """(Shoup products of the first remainder, Montgomery-fold products of the fused remainders)."""
    da, db = max(m, n), min(m, n)
    if db < 1:
        return 0, 0
    return sum(2 * (da - s) for s in range(da - db + 1)), sum(3 * k for k in range(1, db))


def images_products_split(m, n, degs_f, degs_g, K, N):
    """(Shoup-form, Montgomery-fold) products of one k_images launch: the
    roofline weights each class by its own measured peak."""
    NI = POLY * -(-N // POLY)
    s1, m3 = elim_split(m, n)
    return K * NI * (eval_products_poly(degs_f, degs_g) + s1), K * NI * m3


def images_products(m, n, degs_f, degs_g, K, N) -> int:
    """Modular products of one launch of k_images: K primes x S*ceil(N/S) images."""
    NI = POLY * -(-N // POLY)
    return K * NI * (eval_products_poly(degs_f, degs_g) + elim_products(m, n))


def interp_products(K: int, N: int) -> int:
    """Hankel (N^2) + triangular Toeplitz (N(N+1)/2) products per prime."""
    return K * (N * N + N * (N + 1) // 2)


def contract_imad(m, n, degs_f, degs_g, K, N, C, L) -> int:
    r = m + n
    E = eval_products(degs_f, degs_g)
    w = K * N * (E + 4 * r * (r + 1)) + K * N * N + N * K * (K - 1) // 2 + C * L * K
    return 3 * w

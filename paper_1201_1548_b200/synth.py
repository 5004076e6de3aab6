"""Synthetic bivariate inputs for the benchmark configurations.

Restates the generator of SURVEY.md §8(d) / BASELINE.md §2: for a seed, draw
every monomial x^i y^j with i + j <= d (i-major), coefficient uniform in
[-(2^b - 1), 2^b - 1] with zeros redrawn; f first, then g from the same
stream.  cfg3 uses g = df/dy.  Polynomials are returned as plain term dicts
``{(i, j): c}`` (the key layout of ``curvekit.bivpoly.BivPoly``,
reference ``pkg/src/curvekit/bivpoly.py:18-26``).
"""

from __future__ import annotations

import random

# name -> (degree, coefficient bits, kind); kind "pair" = (f, g), "fy" = (f, f_y)
CONFIGS = {
    "cfg1": (6, 10, "pair"),
    "cfg2": (20, 32, "pair"),
    "cfg3": (24, 64, "fy"),
    "cfg4": (40, 64, "pair"),
    "cfg5": (64, 256, "pair"),
    # structured (not a BASELINE config): f = F(x, y^2), g = G(x, y^2), total degree 40, 64-bit -- every
    # image's remainder sequence drops the y-degree by 2 (systematically non-generic)
    "sparse": (40, 64, "even"),
}


def random_dense_terms(rng: random.Random, d: int, bits: int) -> dict:
    hi = (1 << bits) - 1
    terms = {}
    for i in range(d + 1):
        for j in range(d + 1 - i):
            c = 0
            while c == 0:
                c = rng.randint(-hi, hi)
            terms[(i, j)] = c
    return terms


def random_even_terms(rng: random.Random, d: int, bits: int) -> dict:
    """Dense in x and y^2: every x^i y^(2j) with i + 2j <= d."""
    hi = (1 << bits) - 1
    terms = {}
    for i in range(d + 1):
        for j in range(0, d + 1 - i, 2):
            c = 0
            while c == 0:
                c = rng.randint(-hi, hi)
            terms[(i, j)] = c
    return terms


def diff_y(terms: dict) -> dict:
    out = {}
    for (i, j), c in terms.items():
        if j:
            out[(i, j - 1)] = out.get((i, j - 1), 0) + j * c
    return {k: v for k, v in out.items() if v}


def make_pair(config: str, seed: int = 0):
    """(f_terms, g_terms) for a named configuration and seed."""
    d, bits, kind = CONFIGS[config]
    rng = random.Random(seed)
    f = random_dense_terms(rng, d, bits)
    if kind == "fy":
        return f, diff_y(f)
    if kind == "even":
        rng = random.Random(seed)
        return random_even_terms(rng, d, bits), random_even_terms(rng, d, bits)
    g = random_dense_terms(rng, d, bits)
    return f, g

"""Drop-in B200 replacement for ``curvekit.modpoly`` (the reference hot path).

Same public names, argument meaning, return types and exceptions as
pkg/src/curvekit/modpoly.py; every modular computation runs in
libcurvekit_b200.so (include/curvekit_b200.h) on the GPU.  There is no CPU
fallback: without the library or a CUDA device these functions raise.

What stays on the host is what the reference itself does outside its modular
loops: argument checks, the degenerate branches of ``biv_resultant``
(modpoly.py:363-369), primitive parts and the exact trial division that
verifies a modular gcd (:337-340), and the conversion of the GPU's output limbs
into Python ints.  ``prime_table``/``prime_stream`` are the reference's own
(host constants, :31-73); the GPU pipeline draws its primes from
``primes30.PRIMES30`` because the result does not depend on the primes.
"""

from __future__ import annotations

import ctypes
import random
from dataclasses import dataclass
from functools import lru_cache
from math import gcd as int_gcd

import numpy as np

from . import _lib
from .bivpoly import as_biv
from .planner import (ints_to_limbs, limbs_to_ints, pack_grid, pack_terms, plan_packed, plan_resultant)
from .primes30 import PRIMES30

ctypes_ptr = ctypes.c_void_p

__all__ = [
    "UnluckyPrime", "prime_table", "prime_stream", "ModPoly", "ResidueSystem",
    "ModularSubresultantProfile", "zp_resultant_uni", "zp_resultant_batch", "zp_interpolate",
    "zp_gcd_sylvester", "crt_reconstruct", "int_gcd_uni", "biv_resultant",
    "modular_subres_profile",
]


class UnluckyPrime(Exception):
    """Raised when a chosen prime degenerates the leading coefficients."""


# ---------------------------------------------------------------------------
# prime table (host constants; restated from modpoly.py:29-73)
# ---------------------------------------------------------------------------

_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37)


def _is_prime(n: int) -> bool:
    if n < 2:
        return False
    for b in _MR_BASES:
        if n % b == 0:
            return n == b
    d, s = n - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for b in _MR_BASES:
        x = pow(b, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(s - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


@lru_cache(maxsize=8)
def prime_table(bits: int = 31, count: int = 4096) -> tuple:
    """The ``count`` largest primes below 2**bits, descending (modpoly.py:57-66)."""
    out = []
    n = (1 << bits) - 1
    while len(out) < count and n > 2:
        if _is_prime(n):
            out.append(n)
        n -= 2
    return tuple(out)


def prime_stream(seed: int = 0, bits: int = 31):
    """Deterministic enumeration of the prime table in seeded order (:69-73)."""
    table = list(prime_table(bits))
    random.Random(seed).shuffle(table)
    return iter(table)


# ---------------------------------------------------------------------------
# value types (modpoly.py:80-99, :258-261, :421-425)
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class ModPoly:
    p: int
    coeffs: tuple  # residues in [0, p), lowest degree first, no trailing zeros

    @staticmethod
    def make(coeffs, p: int) -> "ModPoly":
        c = [x % p for x in coeffs]
        while c and c[-1] == 0:
            c.pop()
        return ModPoly(p, tuple(c))

    def degree(self) -> int:
        return len(self.coeffs) - 1

    def is_zero(self) -> bool:
        return not self.coeffs


@dataclass(frozen=True)
class ResidueSystem:
    primes: tuple
    residues: tuple


@dataclass(frozen=True)
class ModularSubresultantProfile:
    prime: int
    chain_degrees: tuple
    factor_degrees: tuple


def _same_type_modpoly(like, p: int, coeffs) -> object:
    """Return a ModPoly of the caller's class (reference or ours)."""
    cls = type(like) if hasattr(like, "coeffs") and hasattr(like, "p") else ModPoly
    c = list(coeffs)
    while c and c[-1] == 0:
        c.pop()
    return cls(p, tuple(int(x) for x in c))


def _trim(c: list) -> list:
    while c and c[-1] == 0:
        c.pop()
    return c


# ---------------------------------------------------------------------------
# univariate kernels mod p (batched on the GPU)
# ---------------------------------------------------------------------------

def _check_prime_word(p: int):
    if not (3 <= p < 2 ** 31) or p % 2 == 0:
        raise ValueError("the GPU kernels need an odd prime 3 <= p < 2^31")


def _prime_index(ps):
    uniq = sorted(set(ps))
    for p in uniq:
        _check_prime_word(p)
    pos = {p: i for i, p in enumerate(uniq)}
    return np.array(uniq, dtype=np.uint32), np.array([pos[p] for p in ps], dtype=np.int32)


def zp_resultant_batch(triples) -> list:
    """res(a, b) mod p for a batch of (a, b, p) low-first residue lists.

    Semantics of ``_zp_resultant`` (modpoly.py:132-153) for each triple,
    one GPU thread per pair.
    """
    triples = list(triples)
    if not triples:
        return []
    lib = _lib.lib()
    B = len(triples)
    A = [_trim([x % p for x in a]) for a, _, p in triples]
    Bb = [_trim([x % p for x in b]) for _, b, p in triples]
    W = max(1, max(max(len(a), len(b)) for a, b in zip(A, Bb)))
    fa = np.zeros((B, W), dtype=np.uint32)
    gb = np.zeros((B, W), dtype=np.uint32)
    for i, (a, b) in enumerate(zip(A, Bb)):
        fa[i, :len(a)] = a
        gb[i, :len(b)] = b
    da = np.array([len(a) - 1 for a in A], dtype=np.int32)
    db = np.array([len(b) - 1 for b in Bb], dtype=np.int32)
    primes, pidx = _prime_index([p for _, _, p in triples])
    out = np.empty(B, dtype=np.uint32)
    _lib.check(lib.ckb_uni_resultant_batch(_lib.ptr(fa), _lib.ptr(da), _lib.ptr(gb), _lib.ptr(db), W,
                                           _lib.ptr(primes), len(primes), _lib.ptr(pidx), B, _lib.ptr(out)),
               "ckb_uni_resultant_batch")
    return [int(v) for v in out]


def zp_resultant_uni(f, g) -> int:
    """modpoly.py:156-161."""
    if f.p != g.p:
        raise ValueError("mismatched primes")
    if f.is_zero() or g.is_zero():
        raise ValueError("zero polynomial")
    return zp_resultant_batch([(list(f.coeffs), list(g.coeffs), f.p)])[0]


def zp_interpolate_batch(problems) -> list:
    """Coefficient lists for a batch of (points, values, p) (modpoly.py:164-185)."""
    problems = list(problems)
    if not problems:
        return []
    lib = _lib.lib()
    for pts, vals, p in problems:
        if len(vals) != len(pts):
            raise ValueError("points/values length mismatch")
        if len(set(pts)) != len(pts):
            raise ValueError("duplicate interpolation points")
    B = len(problems)
    W = max(1, max(len(pts) for pts, _, _ in problems))
    xs = np.zeros((B, W), dtype=np.uint32)
    vs = np.zeros((B, W), dtype=np.uint32)
    ns = np.zeros(B, dtype=np.int32)
    for i, (pts, vals, p) in enumerate(problems):
        xs[i, :len(pts)] = [x % p for x in pts]
        vs[i, :len(vals)] = [v % p for v in vals]
        ns[i] = len(pts)
    primes, pidx = _prime_index([p for _, _, p in problems])
    out = np.zeros((B, W), dtype=np.uint32)
    _lib.check(lib.ckb_interp_points(_lib.ptr(xs), _lib.ptr(vs), _lib.ptr(ns), W, _lib.ptr(primes), len(primes),
                                     _lib.ptr(pidx), B, _lib.ptr(out)), "ckb_interp_points")
    return [_trim([int(v) for v in out[i, :ns[i]]]) for i in range(B)]


def zp_interpolate_arrays(xs: np.ndarray, vals: np.ndarray, primes) -> np.ndarray:
    """Array form of a batch of _zp_interp problems (modpoly.py:164-185) sharing
    one point set per prime: xs [k][n] distinct points mod primes[k], vals
    [k][r][n] -> coefficients [k][r][n] (low first, canonical residues)."""
    lib = _lib.lib()
    k, r, n = vals.shape
    B = k * r
    xsb = np.ascontiguousarray(np.repeat(xs.astype(np.uint32), r, axis=0))
    vsb = np.ascontiguousarray(vals.reshape(B, n).astype(np.uint32))
    ns = np.full(B, n, dtype=np.int32)
    parr, pidx = _prime_index([p for p in primes for _ in range(r)])
    out = np.zeros((B, n), dtype=np.uint32)
    _lib.check(lib.ckb_interp_points(_lib.ptr(xsb), _lib.ptr(vsb), _lib.ptr(ns), n, _lib.ptr(parr), len(parr),
                                     _lib.ptr(pidx), B, _lib.ptr(out)), "ckb_interp_points")
    return out.reshape(k, r, n)


def zp_interpolate(points, values, p: int):
    """modpoly.py:188-189."""
    points, values = list(points), list(values)
    if len(values) != len(points):
        raise ValueError("points/values length mismatch")
    if len(set(points)) != len(points):
        raise ValueError("duplicate interpolation points")
    if not points:
        return ModPoly(p, ())
    return ModPoly.make(zp_interpolate_batch([(points, values, p)])[0], p)


def zp_gcd_batch(triples) -> list:
    """Monic gcds mod p of (a, b, p) triples (``_zp_gcd``, modpoly.py:115-122)."""
    triples = list(triples)
    if not triples:
        return []
    lib = _lib.lib()
    B = len(triples)
    A = [_trim([x % p for x in a]) for a, _, p in triples]
    Bb = [_trim([x % p for x in b]) for _, b, p in triples]
    Wf = max(1, max(len(a) for a in A))
    Wg = max(1, max(len(b) for b in Bb))
    fa = np.zeros((B, Wf), dtype=np.uint32)
    gb = np.zeros((B, Wg), dtype=np.uint32)
    for i, (a, b) in enumerate(zip(A, Bb)):
        fa[i, :len(a)] = a
        gb[i, :len(b)] = b
    da = np.array([len(a) - 1 for a in A], dtype=np.int32)
    db = np.array([len(b) - 1 for b in Bb], dtype=np.int32)
    primes, pidx = _prime_index([p for _, _, p in triples])
    Wo = max(Wf, Wg)
    out = np.zeros((B, Wo), dtype=np.uint32)
    odeg = np.zeros(B, dtype=np.int32)
    _lib.check(lib.ckb_gcd_mod_batch(_lib.ptr(fa), _lib.ptr(da), Wf, _lib.ptr(gb), _lib.ptr(db), Wg,
                                     _lib.ptr(primes), len(primes), _lib.ptr(pidx), B, _lib.ptr(out), Wo,
                                     _lib.ptr(odeg)), "ckb_gcd_mod_batch")
    return [[int(v) for v in out[i, :odeg[i] + 1]] for i in range(B)]


def _zp_gcd(a: list, b: list, p: int) -> list:
    """modpoly.py:115-122 (GPU batch of one)."""
    return zp_gcd_batch([(a, b, p)])[0]


def zp_gcd_sylvester(f, g):
    """Monic gcd mod p (modpoly.py:192-244).

    The reference reads it off the row-echelon Sylvester matrix (Thm.,
    PAPER.md:1469-1474); the division-free elimination on the Sylvester
    generators computes the same monic polynomial.
    """
    if f.p != g.p:
        raise ValueError("mismatched primes")
    p = f.p
    fa, gb = list(f.coeffs), list(g.coeffs)
    if not fa or not gb:
        raise ValueError("zero polynomial")
    if len(fa) == 1 or len(gb) == 1:
        return _same_type_modpoly(f, p, [1])
    gm = _zp_gcd(fa, gb, p)
    if len(gm) <= 1:
        gm = [1]
    return _same_type_modpoly(f, p, gm)


# ---------------------------------------------------------------------------
# Chinese remaindering (modpoly.py:258-300)
# ---------------------------------------------------------------------------

def crt_lift(residues: np.ndarray, primes) -> list:
    """Symmetric CRT of K x N residues (rows = primes) -> N Python ints."""
    lib = _lib.lib()
    primes = [int(p) for p in primes]
    K = len(primes)
    res = np.ascontiguousarray(residues, dtype=np.uint32).reshape(K, -1)
    N = res.shape[1]
    mod = 1
    for p in primes:
        mod *= p
    LW = (mod.bit_length() + 31) // 32
    parr = np.array(primes, dtype=np.uint32)
    out = np.empty(N * LW, dtype=np.uint32)
    _lib.check(lib.ckb_crt_lift(_lib.ptr(res), K, N, _lib.ptr(parr), LW, _lib.ptr(out)), "ckb_crt_lift")
    return limbs_to_ints(out, N, LW)


def crt_reconstruct(rs) -> int:
    """The unique representative in (-M/2, M/2] congruent to every residue."""
    if len(set(rs.primes)) != len(rs.primes):
        raise ValueError("primes must be pairwise distinct")
    if not rs.primes:
        return 0
    for p in rs.primes:
        _check_prime_word(p)
    res = np.array([[r % p] for p, r in zip(rs.primes, rs.residues)], dtype=np.uint32)
    return crt_lift(res, rs.primes)[0]


# ---------------------------------------------------------------------------
# integer univariate gcd (modpoly.py:307-341)
# ---------------------------------------------------------------------------

def _content(p: list) -> int:
    g = 0
    for a in p:
        g = int_gcd(g, a)
    return g


def _primitive(p: list) -> list:
    """upoly.primitive (upoly.py:88-95)."""
    if not p:
        return []
    c = _content(p)
    if p[-1] < 0:
        c = -c
    return [a // c for a in p]


def _divexact(p: list, d: list):
    """upoly.divexact (upoly.py:98-118): exact quotient over Z or None."""
    if not d:
        raise ZeroDivisionError
    if not p:
        return []
    if len(p) < len(d):
        return None
    r = list(p)
    q = [0] * (len(p) - len(d) + 1)
    lead = d[-1]
    for k in range(len(q) - 1, -1, -1):
        c = r[k + len(d) - 1]
        if c % lead:
            return None
        c //= lead
        q[k] = c
        if c:
            for j, b in enumerate(d):
                r[k + j] -= c * b
    return _trim(q) if not any(r[: len(d) - 1]) else None


def _reduce_many(polys: list, primes: list) -> list:
    """Residues of each integer polynomial mod each prime: [K] x [poly] lists (K1 on the GPU)."""
    lib = _lib.lib()
    flat = [c for poly in polys for c in poly]
    limbs, L = ints_to_limbs(flat)
    C = len(flat)
    parr = np.array(primes, dtype=np.uint32)
    K = len(primes)
    out = np.empty((K, C), dtype=np.uint32)
    _lib.check(lib.ckb_reduce(_lib.ptr(limbs), C, L, _lib.ptr(parr), K, _lib.ptr(out)), "ckb_reduce")
    return out


def int_gcd_uni(f, g, seed: int = 0):
    """Primitive gcd over Z with positive leading coefficient (modpoly.py:307-341).

    Per-prime Euclid runs on the GPU for a batch of primes at once (the
    reference's incremental loop, made speculative); the
    CRT of the surviving images runs on the GPU; the candidate is verified by
    exact trial division exactly as in the reference.  ``seed`` is accepted
    for API parity (the result does not depend on it).
    """
    f = _trim(list(f))
    g = _trim(list(g))
    if not f and not g:
        raise ValueError("gcd of two zero polynomials")
    if not f:
        return _primitive(g)
    if not g:
        return _primitive(f)
    fp, gp = _primitive(f), _primitive(g)
    if len(fp) == 1 or len(gp) == 1:
        return [1]
    gamma = int_gcd(fp[-1], gp[-1])
    lf, lg = fp[-1], gp[-1]
    best = None
    acc_p, acc_r = [], []
    idx = 0
    batch = 2
    while True:
        primes = []
        while len(primes) < batch:
            if idx >= len(PRIMES30):
                raise ArithmeticError("prime table exhausted in gcd computation")
            p = PRIMES30[idx][0]
            idx += 1
            if lf % p and lg % p:
                primes.append(p)
        red = _reduce_many([fp, gp], primes)
        nf = len(fp)
        gms = zp_gcd_batch([(red[i, :nf].tolist(), red[i, nf:].tolist(), p) for i, p in enumerate(primes)])
        for p, gm in zip(primes, gms):
            d = len(gm) - 1
            if d == 0:
                return [1]
            if best is None or d < best:
                best = d
                acc_p, acc_r = [], []
            elif d > best:
                continue
            gmod = (np.array(gm, dtype=np.uint64) * (gamma % p)) % p
            acc_p.append(p)
            acc_r.append(gmod.astype(np.uint32))
        if acc_p:
            vals = crt_lift(np.stack(acc_r), acc_p)
            cand = _primitive(_trim(vals))
            if len(cand) - 1 == best and _divexact(fp, cand) is not None and \
                    _divexact(gp, cand) is not None:
                return cand
        batch = min(2 * batch, 64)


def int_gcd_uni_batch(pairs) -> list:
    """[int_gcd_uni(f, g) for (f, g) in pairs] with the first modular round of
    every pair in one GPU batch: a pair whose images have degree 0 is coprime
    (the common case) and is done; the others run int_gcd_uni."""
    out = [None] * len(pairs)
    todo = []
    for i, (f, g) in enumerate(pairs):
        f, g = _trim(list(f)), _trim(list(g))
        if not f or not g or len(_primitive(f)) == 1 or len(_primitive(g)) == 1:
            out[i] = int_gcd_uni(f, g)
        else:
            todo.append((i, _primitive(f), _primitive(g)))
    triples, owners = [], []
    for i, fp, gp in todo:
        picked = [p for p, _ in PRIMES30[:16] if fp[-1] % p and gp[-1] % p][:2]
        for p in picked:
            triples.append(([a % p for a in fp], [a % p for a in gp], p))
            owners.append(i)
    gms = zp_gcd_batch(triples)
    coprime = {i for i, gm in zip(owners, gms) if len(gm) == 1}
    for i, fp, gp in todo:
        out[i] = [1] if i in coprime else int_gcd_uni(fp, gp)
    return out


# ---------------------------------------------------------------------------
# bivariate resultants (modpoly.py:348-394)
# ---------------------------------------------------------------------------

def _mul(p: list, q: list) -> list:
    if not p or not q:
        return []
    out = [0] * (len(p) + len(q) - 1)
    for i, a in enumerate(p):
        if a:
            for j, b in enumerate(q):
                out[i + j] += a * b
    return _trim(out)


def _pow(p: list, k: int) -> list:
    out = [1]
    for _ in range(k):
        out = _mul(out, p)
    return out


def biv_resultant(f, g, var: str = "y", seed: int = 0) -> list:
    """Resultant of f and g with respect to ``var``, exactly over Z.

    Equals the determinant of the Sylvester matrix of f and g viewed as
    polynomials in ``var``; the result is a polynomial in the other variable
    (lowest degree first), ``[]`` if it vanishes.  Every modular step (K1
    reduce, plan, fused evaluation + resultant per (prime, point), geometric
    interpolation, mixed-radix CRT with limbs out) runs in one call of
    ``ckb_biv_resultant`` on the GPU.
    """
    # plain term dicts go straight to the limb grid (one C pass, no coeffs_wrt_y)
    pk = pack_terms(f, g, var == "x") if var in ("x", "y") else None
    if pk is not None and pk.m > 0 and pk.n > 0:
        return _biv_resultant_gpu(None, None, pk.tdf, pk.tdg, pk)[0]
    f, g = as_biv(f), as_biv(g)
    if f.is_zero() or g.is_zero():
        raise ValueError("resultant of zero polynomial")
    if var == "x":
        f, g = f.swap(), g.swap()
    elif var != "y":
        raise ValueError("var must be 'x' or 'y'")
    fc = f.coeffs_wrt_y()
    gc = g.coeffs_wrt_y()
    m, n = len(fc) - 1, len(gc) - 1
    if m == 0 and n == 0:
        return [1]
    if m == 0:
        return _pow(fc[0], n)
    if n == 0:
        return _pow(gc[0], m)
    res, _ = _biv_resultant_gpu(fc, gc, f.total_degree(), g.total_degree())
    return res


def _biv_resultant_gpu(fc, gc, tdf: int, tdg: int, packed=None):
    """One ckb_biv_resultant call; ``packed`` from pack_terms replaces fc/gc."""
    lib = _lib.lib()
    if packed is None:
        packed = pack_grid(fc, gc)
    m, n = packed.m, packed.n
    start = 0
    for _attempt in range(4):
        if packed.norms is not None:
            plan = plan_packed(packed, start)
        else:
            plan = plan_resultant(fc, gc, tdf, tdg, packed.dfx, packed.dgx, start)
        K, N, LW = len(plan.primes), plan.N, plan.LW
        out = _lib.pinned.get("biv_out", N * LW)  # page-locked: the result lands here directly
        status = np.zeros(1, dtype=np.uint32)
        ms = np.zeros(1, dtype=np.float32)
        G = min(_lib.n_devices(), K, N)
        if G > 1:  # primes sharded over the device contexts, one residue exchange
            rc = _lib.check(lib.ckb_biv_resultant_multi(
                _lib.ptr(packed.limbs), packed.C, packed.L, _lib.ptr(packed.degs), m, n, packed.dfx, packed.dgx,
                _lib.ptr(plan.primes), _lib.ptr(plan.gens), K, N, LW, G, _lib.ptr(out), _lib.ptr(status),
                _lib.ptr(ms)), "ckb_biv_resultant_multi")
        else:
            rc = _lib.check(lib.ckb_biv_resultant(
                _lib.ptr(packed.limbs), packed.C, packed.L, _lib.ptr(packed.degs), m, n, packed.dfx, packed.dgx,
                _lib.ptr(plan.primes), _lib.ptr(plan.gens), K, N, LW, _lib.ptr(out), _lib.ptr(status),
                _lib.ptr(ms)), "ckb_biv_resultant")
        if rc == 0:
            vals = _trim(limbs_to_ints(out, N, LW))
            return vals, {"K": K, "N": N, "LW": LW, "device_ms": float(ms[0]),
                          "bound_bits": plan.bound_bits, "modulus_bits": plan.modulus_bits}
        start += K  # a prime had no admissible point set: use the next primes
    raise ArithmeticError("no admissible evaluation points after re-planning")


def biv_resultant_batch(problems, seed: int = 0) -> list:
    """[biv_resultant(f, g, var) for (f, g, var) in problems], the GPU problems
    of the list in ONE library call (ckb_biv_resultant_batch, up to 4 per call,
    each pipeline on its own stream so their kernels overlap) — SURVEY.md §8(f) #1,
    bisolve.biproject's two resultants (bisolve.py:107-108).  Errors and
    degenerate branches are those of biv_resultant, problem by problem."""
    results = [None] * len(problems)
    gpu = []
    for i, (f, g, var) in enumerate(problems):
        pk = pack_terms(f, g, var == "x") if var in ("x", "y") else None
        if pk is not None and pk.m > 0 and pk.n > 0:
            gpu.append((i, None, None, pk.tdf, pk.tdg, pk))
            continue
        f, g = as_biv(f), as_biv(g)
        if f.is_zero() or g.is_zero():
            raise ValueError("resultant of zero polynomial")
        if var == "x":
            f, g = f.swap(), g.swap()
        elif var != "y":
            raise ValueError("var must be 'x' or 'y'")
        fc, gc = f.coeffs_wrt_y(), g.coeffs_wrt_y()
        m, n = len(fc) - 1, len(gc) - 1
        if m == 0 and n == 0:
            results[i] = [1]
        elif m == 0:
            results[i] = _pow(fc[0], n)
        elif n == 0:
            results[i] = _pow(gc[0], m)
        else:
            gpu.append((i, fc, gc, f.total_degree(), g.total_degree(), None))
    lib = _lib.lib()
    for a in range(0, len(gpu), 4):
        chunk = gpu[a:a + 4]
        P = len(chunk)
        packs = [pk if pk is not None else pack_grid(fc, gc) for _, fc, gc, _, _, pk in chunk]
        plans = [plan_packed(pk) if pk.norms is not None else plan_resultant(fc, gc, tdf, tdg, pk.dfx, pk.dgx)
                 for (_, fc, gc, tdf, tdg, _), pk in zip(chunk, packs)]
        outs = [_lib.pinned.get(f"biv_out{j}", pl.N * pl.LW) for j, pl in enumerate(plans)]
        status = np.zeros(P, dtype=np.uint32)

        def ptrs(arrs):
            return (ctypes_ptr * P)(*[_lib.ptr(x) for x in arrs])

        def ints(vals):
            return np.array(vals, dtype=np.int32)

        cs, ls = ints([pk.C for pk in packs]), ints([pk.L for pk in packs])
        ms, ns = ints([pk.m for pk in packs]), ints([pk.n for pk in packs])
        dfs, dgs = ints([pk.dfx for pk in packs]), ints([pk.dgx for pk in packs])
        ks, nn = ints([len(pl.primes) for pl in plans]), ints([pl.N for pl in plans])
        lws = ints([pl.LW for pl in plans])
        rc = _lib.check(lib.ckb_biv_resultant_batch(
            P, ptrs([pk.limbs for pk in packs]), _lib.ptr(cs), _lib.ptr(ls), ptrs([pk.degs for pk in packs]),
            _lib.ptr(ms), _lib.ptr(ns), _lib.ptr(dfs), _lib.ptr(dgs), ptrs([pl.primes for pl in plans]),
            ptrs([pl.gens for pl in plans]), _lib.ptr(ks), _lib.ptr(nn), _lib.ptr(lws), ptrs(outs),
            _lib.ptr(status)), "ckb_biv_resultant_batch")
        for j, (i, fc, gc, tdf, tdg, _) in enumerate(chunk):
            if status[j]:  # a prime had no admissible point set: the single call re-plans
                results[i], _ = _biv_resultant_gpu(fc, gc, tdf, tdg, packs[j])
            else:
                results[i] = _trim(limbs_to_ints(outs[j], plans[j].N, plans[j].LW))
        del rc
    return results


# ---------------------------------------------------------------------------
# modular subresultant degree profiles (modpoly.py:421-526)
# ---------------------------------------------------------------------------

def _mod_list(xs, p: int) -> list:
    try:
        from .ckb_limbs import mod_list
    except ImportError:  # the host helper is optional glue
        return [c % p for c in xs]
    return mod_list(list(xs), p)


def modular_subres_profile(f, g, rstar, p: int):
    """Degree profile of the subresultant gcd chain of f, g mod p (modpoly.py:428-474).

    ``rstar`` is the square-free part of res(f, g; y) over Z; the chain is
    S_0 = rstar mod p, S_i = gcd(S_{i-1}, psc_i mod p), with psc_i the i-th
    principal subresultant coefficient of f and g with respect to y.  On the
    GPU: the residues (K1), then ONE library call (ckb_subres_profile) for the
    reference's points, every psc_i at every point (one remainder sequence per
    point instead of a determinant per (point, i)), the batched interpolation
    of every psc_i and the gcd chain.
    """
    lib = _lib.lib()
    f, g = as_biv(f), as_biv(g)
    _check_prime_word(p)
    fci, gci = f.coeffs_wrt_y(), g.coeffs_wrt_y()
    if not fci or not gci:
        raise UnluckyPrime(p)
    # one prime: residues on the host (C helper over CPython's digits) instead of
    # packing every coefficient -- rstar's ~5 kbit ones at cfg4 -- into limbs for K1
    fc = [_mod_list(col, p) for col in fci]
    gc = [_mod_list(col, p) for col in gci]
    rmod = _mod_list(rstar, p)
    if not _trim(list(fc[-1])) or not _trim(list(gc[-1])):
        raise UnluckyPrime(p)  # modpoly.py:437-439
    m, n = len(fc) - 1, len(gc) - 1
    if m < n:
        fc, gc, m, n = gc, fc, n, m
    dmax = max(f.deg_x(), g.deg_x(), 0)
    rlen_int = len(_trim(list(rstar)))
    if n == 0:
        # no psc to interpolate: the chain is S_0 alone (modpoly.py:462-474)
        s0 = zp_gcd_batch([(rmod, [], p)])[0] if _trim(list(rmod)) else []
        if len(s0) - 1 != rlen_int - 1:
            raise UnluckyPrime(p)
        return ModularSubresultantProfile(p, (len(s0) - 1,), ())
    dfx = max(0, max(len(c) - 1 for c in fc))
    dgx = max(0, max(len(c) - 1 for c in gc))
    fg = np.zeros((m + 1, dfx + 1), dtype=np.uint32)
    gg = np.zeros((n + 1, dgx + 1), dtype=np.uint32)
    for j, col in enumerate(fc):
        fg[j, :len(col)] = col
    for j, col in enumerate(gc):
        gg[j, :len(col)] = col
    fdeg = np.array([len(_trim(list(c))) - 1 for c in fc], dtype=np.int16)
    gdeg = np.array([len(_trim(list(c))) - 1 for c in gc], dtype=np.int16)
    rm = np.array(rmod, dtype=np.uint32)
    chain = np.zeros(n + 1, dtype=np.int32)
    rc = _lib.check(lib.ckb_subres_profile(_lib.ptr(fg), _lib.ptr(fdeg), m, dfx, _lib.ptr(gg), _lib.ptr(gdeg), n,
                                           dgx, _lib.ptr(rm), len(rmod), rlen_int, dmax, p, _lib.ptr(chain)),
                    "ckb_subres_profile")
    if rc == 2:
        raise UnluckyPrime(p)  # modpoly.py:450-451, :462-463
    chain = [int(v) for v in chain]
    d = [chain[i - 1] - chain[i] for i in range(1, n + 1)]
    return ModularSubresultantProfile(p, tuple(chain), tuple(d))

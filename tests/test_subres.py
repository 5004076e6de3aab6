"""psc values from one remainder sequence per point (ckb_psc.cu) against the
reference's determinant definition (_psc_det, pkg/src/curvekit/modpoly.py:477-501).

CPU: the fundamental-theorem formula the kernel evaluates, restated in Python,
equals _psc_det on random dense, sparse and common-factor inputs.  GPU:
ckb_psc_values equals _psc_det at every candidate point of random bivariate
pairs; the full profile is pinned by the goldens in test_gpu_parity.py."""

import random

import numpy as np
import pytest


def _mul(x, y, p):
    o = [0] * (len(x) + len(y) - 1)
    for i, u in enumerate(x):
        for j, w in enumerate(y):
            o[i + j] = (o[i + j] + u * w) % p
    return o


def psc_from_prs(a, b, p, M):
    """psc_1..psc_n of a (deg m) and b (deg n), m >= n >= 1, lc's nonzero."""
    m, n = len(a) - 1, len(b) - 1
    out = {i: 0 for i in range(1, n + 1)}
    degs, lcs, R = [m, n], [a[-1], b[-1]], [list(a), list(b)]
    acc, i = 1, 1
    while True:
        ni = degs[i]
        tau = sum((degs[l - 1] - ni) * (degs[l] - ni) for l in range(1, i)) % 2
        v = pow(lcs[i], degs[i - 1] - ni, p) * acc % p
        if tau:
            v = -v % p
        if ni >= 1:
            out[ni] = v
        if ni == 0:
            break
        r = M._zp_rem(R[i - 1], R[i], p)
        if not r:
            break
        R.append(r)
        degs.append(len(r) - 1)
        lcs.append(r[-1])
        acc = acc * pow(lcs[i], degs[i - 1] - degs[i + 1], p) % p
        i += 1
    return out


def _random_pair(rng, p):
    m = rng.randint(1, 10)
    n = rng.randint(1, m)
    dens = rng.choice([1.0, 0.6, 0.3])
    a = [rng.randrange(p) if rng.random() < dens else 0 for _ in range(m + 1)]
    b = [rng.randrange(p) if rng.random() < dens else 0 for _ in range(n + 1)]
    a[-1] = rng.randrange(1, p)
    b[-1] = rng.randrange(1, p)
    if rng.random() < 0.25 and n >= 2:  # a planted common factor
        c = [rng.randrange(p), 1]
        a = _mul(a[:-1], c, p)
        b = _mul(b[:-1], c, p)
        if a[-1] == 0 or b[-1] == 0:
            return None
    if len(b) > len(a):
        a, b = b, a
    return a, b


def test_prs_formula_equals_reference_determinants(curvekit_mod):
    M = curvekit_mod.modpoly
    rng = random.Random(1)
    for p in (7, 1009, 1073692673):
        for _ in range(700):
            pr = _random_pair(rng, p)
            if pr is None:
                continue
            a, b = pr
            got = psc_from_prs(a, b, p, M)
            for i in range(1, len(b)):
                assert got[i] == M._psc_det(a, b, i, p), (a, b, i, p)


@pytest.mark.gpu
def test_gpu_psc_values_equal_reference_determinants(curvekit_mod):
    from paper_1201_1548_b200 import _lib
    M = curvekit_mod.modpoly
    lib = _lib.lib()
    rng = random.Random(7)
    for trial in range(30):
        p = rng.choice([101, 1009, 1073692673, 2147483629])
        m = rng.randint(1, 9)
        n = rng.randint(1, m)
        dfx, dgx = rng.randint(0, 5), rng.randint(0, 5)
        dens = rng.choice([1.0, 0.5, 0.25])
        fg = np.array([[rng.randrange(p) if rng.random() < dens else 0 for _ in range(dfx + 1)]
                       for _ in range(m + 1)], dtype=np.uint32)
        gg = np.array([[rng.randrange(p) if rng.random() < dens else 0 for _ in range(dgx + 1)]
                       for _ in range(n + 1)], dtype=np.uint32)
        fg[m, 0] = fg[m, 0] or 1
        gg[n, 0] = gg[n, 0] or 1

        def deg(r):
            nz = np.nonzero(r)[0]
            return int(nz[-1]) if len(nz) else -1
        fdeg = np.array([deg(r) for r in fg], dtype=np.int16)
        gdeg = np.array([deg(r) for r in gg], dtype=np.int16)
        ncand = 60
        out = np.zeros((n, ncand), dtype=np.uint32)
        valid = np.zeros(ncand, dtype=np.uint8)
        _lib.check(lib.ckb_psc_values(_lib.ptr(fg), _lib.ptr(fdeg), m, dfx, _lib.ptr(gg), _lib.ptr(gdeg), n, dgx, p,
                                      ncand, _lib.ptr(out), _lib.ptr(valid)), "ckb_psc_values")
        for t in range(ncand):
            fu = [M._zp_eval([int(v) for v in row], t, p) for row in fg]
            gu = [M._zp_eval([int(v) for v in row], t, p) for row in gg]
            ok = fu[-1] != 0 and gu[-1] != 0
            assert bool(valid[t]) == ok
            if not ok:
                continue
            for i in range(1, n + 1):
                assert int(out[i - 1, t]) == M._psc_det(fu, gu, i, p), (trial, t, i)

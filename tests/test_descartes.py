"""Descartes test of real-root isolation: upoly._variations_on
(pkg/src/curvekit/upoly.py:338-346) on the GPU against the reference's own
recorded counts and isolating intervals (tests/golden/descartes.json.gz)."""

import random
from dataclasses import dataclass

import pytest

from conftest import ints_in, load_golden


@dataclass(frozen=True)
class Dy:  # the two fields of curvekit.dyadic.Dyadic the test reads
    man: int
    exp: int


@pytest.fixture(scope="module")
def gold():
    return load_golden("descartes.json.gz")


def _poly(gold, c):
    return ints_in(c["p"]) if "p" in c else ints_in(gold["polys"][c["name"]])


def test_oracle_matches_reference_counts(gold):
    from oracle import oracle
    for c in gold["cases"]:
        p = _poly(gold, c)
        if len(p) > 100:
            continue  # the degree-400 cases are checked on the GPU
        assert oracle.variations_on(p, int(c["am"]), c["ae"], int(c["bm"]), c["be"]) == c["v"], c


@pytest.mark.gpu
def test_gpu_variations_match_reference(gold):
    from paper_1201_1548_b200.upoly import variations_on
    polys = {}
    for c in gold["cases"]:
        key = c["name"] if "p" not in c else None
        p = polys.setdefault(key, _poly(gold, c)) if key else _poly(gold, c)
        v = variations_on(p, Dy(int(c["am"]), c["ae"]), Dy(int(c["bm"]), c["be"]))
        assert v == c["v"], (c["name"], c["am"], c["ae"], c["bm"], c["be"])


@pytest.mark.gpu
def test_gpu_variations_random_vs_oracle():
    from oracle import oracle
    from paper_1201_1548_b200.upoly import variations_on
    rng = random.Random(5)
    for _ in range(25):
        deg = rng.randint(1, 70)
        p = [rng.randint(-2 ** 60, 2 ** 60) for _ in range(deg + 1)]
        p[-1] = p[-1] or 3
        if rng.random() < 0.3:
            p[0] = 0
        a = Dy(rng.randint(-2 ** 40, 2 ** 40), rng.randint(-60, 5))
        b = Dy(rng.randint(-2 ** 40, 2 ** 40), rng.randint(-60, 5))
        want = oracle.variations_on(p, a.man, a.exp, b.man, b.exp)
        assert variations_on(p, a, b) == want




@pytest.mark.gpu
def test_isolation_matches_reference(gold, curvekit_mod):
    """descartes_isolate of the unmodified reference, with install() routing its
    Descartes tests (and square-free check) to the GPU: identical isolating
    intervals for every recorded polynomial, the degree-400 cfg2 resultant
    included (53 s in the reference)."""
    import time

    import curvekit.upoly as U

    import paper_1201_1548_b200 as pkg
    saved = pkg.install()
    try:
        from paper_1201_1548_b200 import upoly as ours
        assert U._variations_on is ours.variations_on
        for iso in gold["isolations"]:
            p = ints_in(iso["p"])
            t0 = time.time()
            roots = U.descartes_isolate(p)
            dt = time.time() - t0
            got = [[str(r.interval.lo.man), r.interval.lo.exp, str(r.interval.hi.man), r.interval.hi.exp]
                   for r in roots]
            assert got == iso["roots"], iso["name"]
            print(iso["name"], "%.3f s (reference %.1f s)" % (dt, iso["seconds"]))
    finally:
        pkg.uninstall(saved)


@pytest.mark.gpu
def test_cfg3_isolation_matches_reference(curvekit_mod):
    """cfg3's degree-552 resultant: the reference's isolation takes ~170 s on one
    core; through install() the same intervals come back in about a second."""
    import math
    import time

    import curvekit.upoly as U

    import paper_1201_1548_b200 as pkg
    gold = load_golden("cfg3_seed0.json.gz")
    want = load_golden("descartes_cfg3.json")
    r = [int(c, 16) for c in gold["res"]]
    c = 0
    for v in r:
        c = math.gcd(c, v)
    p = [v // c for v in r]
    saved = pkg.install()
    try:
        t0 = time.time()
        roots = U.descartes_isolate(p)
        dt = time.time() - t0
    finally:
        pkg.uninstall(saved)
    got = [[str(x.interval.lo.man), x.interval.lo.exp, str(x.interval.hi.man), x.interval.hi.exp] for x in roots]
    assert got == want["roots"]
    print("cfg3 isolation %.2f s (reference %.1f s)" % (dt, want["seconds"]))


@pytest.mark.gpu
def test_batched_variations_and_breadth_first_isolation(gold, curvekit_mod):
    """variations_batch (one launch for many intervals) equals the single-interval
    test, and the breadth-first descartes_isolate that install() binds returns the
    brackets of the reference's depth-first loop (run here with the GPU test)."""
    import curvekit.upoly as U

    import paper_1201_1548_b200 as pkg
    from paper_1201_1548_b200 import upoly as ours
    polys = {}
    for c in gold["cases"]:
        key = c["name"] if "p" not in c else repr(c["p"])[:64]
        polys.setdefault(key, []).append(c)
    for key, cases in polys.items():
        p = _poly(gold, cases[0])
        ivs = [(Dy(int(c["am"]), c["ae"]), Dy(int(c["bm"]), c["be"])) for c in cases]
        assert ours.variations_batch(p, ivs) == [c["v"] for c in cases], key
    saved = pkg.install()
    try:
        assert U.descartes_isolate is ours.descartes_isolate
        dfs = saved[("curvekit.upoly", "descartes_isolate")]  # the reference's own loop
        for iso in gold["isolations"]:
            p = ints_in(iso["p"])
            a = [(str(r.interval.lo.man), r.interval.lo.exp, str(r.interval.hi.man), r.interval.hi.exp, r.multiplicity)
                 for r in ours.descartes_isolate(p, multiplicity=2)]
            b = [(str(r.interval.lo.man), r.interval.lo.exp, str(r.interval.hi.man), r.interval.hi.exp, r.multiplicity)
                 for r in dfs(p, multiplicity=2)]
            assert a == b, iso["name"]
        with pytest.raises(ValueError):
            ours.descartes_isolate([])
        with pytest.raises(ValueError):
            ours.descartes_isolate([1, -2, 1])  # (x - 1)^2 is not square-free
        assert [r.exact for r in ours.descartes_isolate([0, 1])] == [0]
    finally:
        pkg.uninstall(saved)


@pytest.mark.gpu
def test_variations_batch_chunking_vs_oracle():
    """More intervals than one library call takes (chunks of <= 256), mixed widths
    and exponents (different prime counts per interval within a chunk)."""
    from oracle import oracle
    from paper_1201_1548_b200.upoly import variations_batch
    rng = random.Random(23)
    for deg in (7, 33):
        p = [rng.randint(-2 ** 50, 2 ** 50) for _ in range(deg + 1)]
        p[-1] = p[-1] or 5
        ivs = []
        for _ in range(600):
            a = Dy(rng.randint(-2 ** 30, 2 ** 30), rng.randint(-70, 3))
            b = Dy(a.man * 2 ** max(0, a.exp - (a.exp - 1)) + rng.randint(1, 2 ** 20), a.exp)
            ivs.append((a, b))
        want = [oracle.variations_on(p, a.man, a.exp, b.man, b.exp) for a, b in ivs]
        assert variations_batch(p, ivs) == want


def test_breadth_first_walk_matches_reference_loop(curvekit_mod, monkeypatch):
    """CPU: the breadth-first isolation (one batched call per subdivision level,
    split points checked modulo 2^61 - 1 first) returns the reference's own
    descartes_isolate brackets, with the reference's CPU Descartes test standing
    in for the GPU batch — the walk and the split points are what is checked."""
    import curvekit.upoly as U

    import paper_1201_1548_b200 as pkg
    from paper_1201_1548_b200 import upoly as ours
    ref_loop = pkg._ORIGINALS.get(("curvekit.upoly", "descartes_isolate"), U.descartes_isolate)
    assert ref_loop is not ours.descartes_isolate

    def cpu_batch(p, intervals, pbits=None):
        return [U._variations_on(p, a, b) for a, b in intervals]

    monkeypatch.setattr(ours, "variations_batch", cpu_batch)
    rng = random.Random(11)
    n = 0
    for _ in range(8):  # products of linear factors with close rational roots, times a random factor
        p = [1]
        for _ in range(rng.randint(2, 6)):
            num, den = rng.randint(-40, 40), rng.choice([1, 3, 7, 64, 1000])
            p = [a - b for a, b in zip([0] + [den * c for c in p], [num * c for c in p] + [0])]
        q = [rng.randint(-9, 9) for _ in range(rng.randint(1, 5))] + [1]
        p = [sum(p[i] * q[j - i] for i in range(len(p)) if 0 <= j - i < len(q)) for j in range(len(p) + len(q) - 1)]
        try:
            want = ref_loop(p)
        except ValueError:  # not square-free
            continue
        got = ours.descartes_isolate(p, check_squarefree=False)
        assert [(r.interval.lo, r.interval.hi) for r in got] == [(r.interval.lo, r.interval.hi) for r in want]
        n += 1
    assert n >= 3

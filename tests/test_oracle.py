"""Pin the CPU oracle against the reference's golden vectors (CPU only).

The fixtures in tests/golden/ were produced by the unmodified reference
(tests/golden/make_golden.py); the oracle is a restatement of
pkg/src/curvekit/modpoly.py, so it must reproduce every one of them.
"""

import hashlib

import pytest

from conftest import ints_in, load_golden, terms_in


def test_oracle_resultant_cases(small, oracle_mod):
    for case in small["resultant_cases"]:
        got = oracle_mod.biv_resultant(terms_in(case["f"]), terms_in(case["g"]), case["var"])
        assert got == ints_in(case["res"]), case


def test_oracle_random50_both_directions(small, oracle_mod):
    # test_modpoly.py:41-48 (Bareiss-checked in make_golden.py) plus res_x
    for case in small["random50"]:
        f, g = terms_in(case["f"]), terms_in(case["g"])
        assert oracle_mod.biv_resultant(f, g, "y") == ints_in(case["res_y"])
        assert oracle_mod.biv_resultant(f, g, "x") == ints_in(case["res_x"])


def test_oracle_zp_resultant(small, oracle_mod):
    for case in small["zp_resultant"]:
        assert oracle_mod.zp_resultant(case["f"], case["g"], case["p"]) == case["res"]


def test_oracle_zp_interpolate(small, oracle_mod):
    for case in small["zp_interpolate"]:
        assert oracle_mod.zp_interp(case["x"], case["v"], case["p"]) == case["c"]
    with pytest.raises(ValueError):
        oracle_mod.zp_interp([1, 1], [0, 0], 5)


def test_oracle_crt(small, oracle_mod):
    for case in small["crt"]:
        assert oracle_mod.crt_reconstruct(case["primes"], case["res"]) == int(case["x"])


def test_oracle_int_gcd(small, oracle_mod):
    for case in small["int_gcd"]:
        assert oracle_mod.int_gcd_uni(ints_in(case["f"]), ints_in(case["g"])) == ints_in(case["gcd"])


def test_oracle_zp_gcd_matches_reference_euclid(small, oracle_mod):
    for case in small["zp_gcd_sylvester"]:
        if "euclid" in case:
            assert oracle_mod.zp_gcd(case["f"], case["g"], case["p"]) == case["euclid"]


def test_oracle_prime_table(small, oracle_mod):
    pt = small["prime_table"]
    t = oracle_mod.prime_table()
    assert len(t) == pt["count"] and list(t[:8]) == pt["first"] and list(t[-8:]) == pt["last"]
    assert list(oracle_mod._stream(0)[:8]) == pt["stream0_8"]
    assert list(oracle_mod._stream(7)[:8]) == pt["stream7_8"]


def test_oracle_cfg4_one_prime(oracle_mod):
    # one prime of the reference loop body at cfg4 (modpoly.py:376-391)
    from paper_1201_1548_b200.synth import make_pair
    gold = load_golden("cfg4_prime0.json.gz")
    f, g = make_pair("cfg4", 0)
    fc, gc = oracle_mod.coeffs_wrt_y(f), oracle_mod.coeffs_wrt_y(g)
    (rc, poly), = oracle_mod.prime_images(fc, gc, [gold["p"]], 1601)
    assert rc >= 0 and poly == gold["poly"]


def test_oracle_cfg2_full():
    from oracle import oracle
    from paper_1201_1548_b200.synth import make_pair
    gold = load_golden("cfg2_seed0.json.gz")
    f, g = make_pair("cfg2", 0)
    got = oracle.biv_resultant(f, g, "y")
    assert got == [int(c, 16) for c in gold["res"]]
    assert hashlib.sha256(repr(got).encode()).hexdigest()[:16] == gold["sha16_repr"] == "e19abb8388d2a501"


def test_cfg4_full_golden_matches_reference_prime():
    """The oracle's full cfg4 resultant (tests/golden/cfg4_full.json.gz) reduced
    modulo the reference loop's own prime equals the polynomial the UNMODIFIED
    reference interpolated at that prime (cfg4_prime0.json.gz), and its bit
    length stays inside the reference's coefficient bound (modpoly.py:397-414)."""
    gold = load_golden("cfg4_full.json.gz")
    one = load_golden("cfg4_prime0.json.gz")
    res = [int(c, 16) for c in gold["res"]]
    assert hashlib.sha256(repr(res).encode()).hexdigest() == gold["sha256_repr"]
    p = one["p"]
    assert [c % p for c in res] == one["poly"] + [0] * (len(res) - len(one["poly"]))
    assert max(abs(c).bit_length() for c in res) == gold["max_bits"] <= 5765

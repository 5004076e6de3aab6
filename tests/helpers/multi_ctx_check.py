"""Run in a subprocess by tests/test_multi_device.py with CKB_DEVICES set
(e.g. "0,0,0": three device contexts sharing GPU 0).  Every res_y of the
drop-in then goes through ckb_biv_resultant_multi (primes sharded over the
contexts, the residue exchange, coefficient-sharded CRT); the results must be
bit-identical to the goldens and the oracle."""

import hashlib
import json
import os
import random
import sys

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))

from conftest import load_golden, terms_in, ints_in  # noqa: E402
from oracle import oracle  # noqa: E402
from paper_1201_1548_b200 import _lib, modpoly  # noqa: E402
from paper_1201_1548_b200.synth import make_pair  # noqa: E402

n = _lib.n_devices()
want = len(os.environ["CKB_DEVICES"].split(","))
assert n == want, (n, want)
oracle.build()
report = {"contexts": n, "nccl": _lib.uses_nccl()}
launches0 = _lib.launch_count()
small = load_golden("small.json")
for case in small["random50"][:20]:
    f, g = terms_in(case["f"]), terms_in(case["g"])
    assert modpoly.biv_resultant(f, g, "y") == ints_in(case["res_y"])
    assert modpoly.biv_resultant(f, g, "x") == ints_in(case["res_x"])
rng = random.Random(3)
for _ in range(10):
    d1, d2 = rng.randint(2, 9), rng.randint(2, 9)
    f = {(i, j): rng.randint(-2 ** 40, 2 ** 40) or 1 for i in range(d1 + 1) for j in range(d1 + 1 - i)}
    g = {(i, j): rng.randint(-2 ** 40, 2 ** 40) or 1 for i in range(d2 + 1) for j in range(d2 + 1 - i)}
    assert modpoly.biv_resultant(f, g, "y") == oracle.biv_resultant(f, g, "y")
for cfg in ("cfg2", "cfg3"):
    gold = load_golden(f"{cfg}_seed0.json.gz")
    f, g = make_pair(cfg, 0)
    got = modpoly.biv_resultant(f, g, "y")
    assert got == [int(c, 16) for c in gold["res"]], cfg
gold = load_golden("cfg4_full.json.gz")
f, g = make_pair("cfg4", 0)
for _ in range(3):  # eager, captured, replayed
    got = modpoly.biv_resultant(f, g, "y")
    assert hashlib.sha256(repr(got).encode()).hexdigest() == gold["sha256_repr"]
report["launches"] = _lib.launch_count() - launches0
report["exchange"] = _lib.last_exchange()
print(json.dumps(report))

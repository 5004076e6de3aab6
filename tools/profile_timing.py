"""Wall time of modpoly.modular_subres_profile (GeoTop's N^- test) at cfg2/cfg3/cfg4,
one prime of the reference's table, rstar = the primitive part of res_y (square-free
for these random inputs); cfg3 checked against the reference's recorded profile."""
import math
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from conftest import load_golden  # noqa: E402
from paper_1201_1548_b200 import modpoly as mp  # noqa: E402
from paper_1201_1548_b200.synth import make_pair  # noqa: E402

for cfg in ("cfg2", "cfg3", "cfg4"):
    f, g = make_pair(cfg, 0)
    r = mp.biv_resultant(f, g, "y")
    c = 0
    for v in r:
        c = math.gcd(c, v)
    rs = [v // c for v in r]
    p = mp.prime_table()[0]
    if cfg == "cfg3":
        gold = load_golden("cfg3_seed0.json.gz")
        p = gold["profile"]["p"]
    t = time.perf_counter()
    pr = mp.modular_subres_profile(f, g, rs, p)
    cold = time.perf_counter() - t
    ws = []
    for _ in range(5):
        t = time.perf_counter()
        pr = mp.modular_subres_profile(f, g, rs, p)
        ws.append(time.perf_counter() - t)
    if cfg == "cfg3":
        assert list(pr.chain_degrees) == gold["profile"]["chain"] and list(pr.factor_degrees) == gold["profile"]["d"]
    print(f"{cfg} profile cold {cold * 1e3:.2f} ms warm {statistics.median(ws) * 1e3:.2f} ms "
          f"chain {pr.chain_degrees[:4]} sum d {sum(pr.factor_degrees)}", flush=True)

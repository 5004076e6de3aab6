import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, math
from paper_1201_1548_b200 import modpoly as mp
from paper_1201_1548_b200.synth import make_pair
for cfg in ("cfg2", "cfg4"):
    f, g = make_pair(cfg, 0)
    r = mp.biv_resultant(f, g, "y")
    c = 0
    for v in r:
        c = math.gcd(c, v)
    rs = [v // c for v in r]
    p = mp.prime_table()[0]
    t = time.time(); pr = mp.modular_subres_profile(f, g, rs, p); t1 = time.time() - t
    t = time.time(); pr = mp.modular_subres_profile(f, g, rs, p); t2 = time.time() - t
    print(cfg, "profile cold %.3f s warm %.3f s" % (t1, t2), pr.chain_degrees[:4], sum(pr.factor_degrees))

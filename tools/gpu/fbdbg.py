import os, sys
sys.path.insert(0, os.getcwd())
from paper_1201_1548_b200 import modpoly as mp, _lib
from paper_1201_1548_b200.synth import make_pair
for cfg in ("sparse", "cfg4"):
    f, g = make_pair(cfg, 0)
    for i in range(3):
        mp.biv_resultant(f, g, "y")
        print(cfg, i, _lib.last_fallback(), flush=True)

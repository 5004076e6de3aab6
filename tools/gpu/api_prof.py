import os, sys, time, cProfile, pstats
sys.path.insert(0, os.getcwd())
from paper_1201_1548_b200 import modpoly as mp, _lib
from paper_1201_1548_b200.planner import limbs_to_ints
from paper_1201_1548_b200.synth import make_pair
import numpy as np
f, g = make_pair("cfg4", 0)
for _ in range(5): mp.biv_resultant(f, g, "y")
t = time.perf_counter()
for _ in range(20): mp.biv_resultant(f, g, "y")
print("api ms %.3f" % ((time.perf_counter() - t) / 20 * 1e3))
cProfile.run("for _ in range(20): mp.biv_resultant(f, g, 'y')", "/tmp/ap")
pstats.Stats("/tmp/ap").sort_stats("tottime").print_stats(12)

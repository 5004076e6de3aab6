import math, os, sys, time
sys.path.insert(0, os.getcwd())
from paper_1201_1548_b200 import modpoly as mp, _lib
from paper_1201_1548_b200.bivpoly import as_biv
from paper_1201_1548_b200.synth import make_pair
f, g = make_pair("cfg4", 0)
r = mp.biv_resultant(f, g, "y")
c = 0
for v in r: c = math.gcd(c, v)
rs = [v // c for v in r]
p = mp.prime_table()[0]
mp.modular_subres_profile(f, g, rs, p)
t = time.perf_counter(); F, G = as_biv(f), as_biv(g); t1 = time.perf_counter() - t
t = time.perf_counter(); fci, gci = F.coeffs_wrt_y(), G.coeffs_wrt_y(); t2 = time.perf_counter() - t
t = time.perf_counter(); rm = [x % p for x in rs]; t3 = time.perf_counter() - t
t = time.perf_counter(); mp.modular_subres_profile(f, g, rs, p); t4 = time.perf_counter() - t
import cProfile, pstats
cProfile.run("mp.modular_subres_profile(f, g, rs, p)", "/tmp/pp")
pstats.Stats("/tmp/pp").sort_stats("tottime").print_stats(8)
print("as_biv %.2f ms coeffs %.2f ms rstar%%p %.2f ms total %.2f ms" % (t1*1e3, t2*1e3, t3*1e3, t4*1e3))

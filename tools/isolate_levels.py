import math, os, sys, time
REPO="/root/repo"; sys.path.insert(0, REPO); sys.path.insert(0, os.path.join(REPO, "baseline", "_ref"))
import curvekit.upoly as U
import paper_1201_1548_b200 as pkg
from paper_1201_1548_b200 import modpoly as mp, upoly as ours
from paper_1201_1548_b200.synth import make_pair
orig = ours.variations_batch
log = []
def wrapped(p, ivs):
    t = time.perf_counter(); r = orig(p, ivs); log.append((len(ivs), time.perf_counter() - t)); return r
ours.variations_batch = wrapped
saved = pkg.install()
for cfg in ["cfg3", "cfg3", "cfg3"]:
    f, g = make_pair(cfg, 0)
    r = mp.biv_resultant(f, g, "y")
    c = 0
    for v in r: c = math.gcd(c, v)
    p = [v // c for v in r]
    log.clear()
    t0 = time.time(); roots = U.descartes_isolate(p); dt = time.time() - t0
    print(cfg, len(roots), "%.2f s" % dt, "levels", len(log), "batch time %.2f s" % sum(x[1] for x in log))
    print("  ", [(n, round(t * 1e3, 1)) for n, t in log])

import math, os, sys, time
sys.path.insert(0, "/root/repo")
from dataclasses import dataclass
from paper_1201_1548_b200 import modpoly as mp, upoly as ours, _lib
from paper_1201_1548_b200.synth import make_pair
@dataclass(frozen=True)
class Dy:
    man: int
    exp: int
f, g = make_pair("cfg2", 0)
r = mp.biv_resultant(f, g, "y")
c = 0
for v in r: c = math.gcd(c, v)
p = [v // c for v in r]
for (a, b) in [(Dy(-1, 30), Dy(1, 30)), (Dy(1, -20), Dy(3, -21)), (Dy(12345, -40), Dy(12347, -40))]:
    v = ours.variations_on(p, a, b)
    t = time.perf_counter()
    for _ in range(20):
        ours.variations_on(p, a, b)
    dt = (time.perf_counter() - t) / 20
    e = min(a.exp, b.exp, 0)
    print("interval", a, b, "v", v, "%.3f ms" % (dt * 1e3))

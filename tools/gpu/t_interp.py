import random, sys
sys.path.insert(0, '/root/repo')
from paper_1201_1548_b200.modpoly import zp_interpolate
rng = random.Random(1)
p = 1073692673
for n in (5, 100, 700, 3000, 5000, 13000):
    for cons in (False, True):
        pts = list(range(n)) if cons else rng.sample(range(1, p), n)
        vals = [rng.randrange(p) for _ in range(n)]
        try:
            zp_interpolate(pts, vals, p)
            print(n, cons, "ok", flush=True)
        except Exception as e:
            print(n, cons, "ERR", e, flush=True)

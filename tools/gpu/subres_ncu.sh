timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_subres_launches.csv python tools/profile_timing.py > /dev/null 2>&1; echo ncu=$?
python - <<'PY'
import cProfile, pstats, sys, os, math
sys.path.insert(0, '.')
from paper_1201_1548_b200 import modpoly as mp
from paper_1201_1548_b200.synth import make_pair
f, g = make_pair("cfg4", 0)
r = mp.biv_resultant(f, g, "y")
c = 0
for v in r: c = math.gcd(c, v)
rs = [v // c for v in r]
p = mp.prime_table()[0]
mp.modular_subres_profile(f, g, rs, p)
cProfile.run("for _ in range(5): mp.modular_subres_profile(f, g, rs, p)", "/tmp/prof")
pstats.Stats("/tmp/prof").sort_stats("cumulative").print_stats(12)
PY

"""Run one configuration's res_y a few times through the Python API (for ncu captures)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_1201_1548_b200 import modpoly  # noqa: E402
from paper_1201_1548_b200.synth import make_pair  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
f, g = make_pair(cfg, 0)
for _ in range(reps):
    r = modpoly.biv_resultant(f, g, "y")
print(cfg, "deg", len(r) - 1)

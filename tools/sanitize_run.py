"""One small res_y per pipeline shape for compute-sanitizer (no CUDA graphs, so
every kernel launch is visible to the tool): cfg2 (register images kernel,
tensor-core interpolation + CRT), a sparse curve pair (fallback warp kernel),
a modular gcd batch and a Descartes test."""
import os
import sys

os.environ["CKB_NO_GRAPHS"] = "1"
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_1201_1548_b200 import modpoly, upoly  # noqa: E402
from paper_1201_1548_b200.synth import make_pair  # noqa: E402

f, g = make_pair("cfg2", 0)
r = modpoly.biv_resultant(f, g, "y")
assert len(r) == 401
circle = {(2, 0): 1, (0, 2): 1, (0, 0): -1}
assert modpoly.biv_resultant(circle, {(0, 1): 2}) == [-4, 0, 4]
cusp = {(0, 2): 1, (3, 0): -1}
assert modpoly.biv_resultant(cusp, {(0, 1): 2}) == [0, 0, 0, -4]
p = 1073692673
print(modpoly.zp_gcd_batch([([1, 2, 1], [1, 1], p)]))


class Dy:
    def __init__(self, m, e):
        self.man, self.exp = m, e


print(upoly.variations_batch([-2, 0, 1], [(Dy(0, 0), Dy(2, 0))]))
print("sanitize run ok")

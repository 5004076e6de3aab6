import os, sys
sys.path.insert(0, "/root/repo")
from paper_1201_1548_b200 import modpoly as mp
from paper_1201_1548_b200.synth import make_pair
for cfg in ("cfg2", "cfg3", "cfg4"):
    f, g = make_pair(cfg, 0)
    r, info = mp._biv_resultant_gpu(mp.as_biv(f).coeffs_wrt_y(), mp.as_biv(g).coeffs_wrt_y(), mp.as_biv(f).total_degree(), mp.as_biv(g).total_degree())
    mb = max(abs(c).bit_length() for c in r)
    print(cfg, "max bits", mb, "bound bits", info["bound_bits"], "modulus bits", info["modulus_bits"], "K", info["K"])

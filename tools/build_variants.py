"""Build tuning variants of the library into build/variants/ (experiments only).

    python tools/build_variants.py NAME=DEF1,DEF2 ...
Run one with CKB_LIB=build/variants/libNAME.so python bench.py ...
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1201_1548_b200 import build  # noqa: E402

out_dir = os.path.join(build.REPO, "build", "variants")
os.makedirs(out_dir, exist_ok=True)
for arg in sys.argv[1:]:
    name, _, defs = arg.partition("=")
    build.build(out=os.path.join(out_dir, f"lib{name}.so"), defines=[d for d in defs.split(",") if d])

import cProfile
import os
import pstats
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.argv = ["isolate_timing.py", "cfg3"]
code = compile(open(os.path.join(HERE, "isolate_timing.py")).read(), "isolate_timing.py", "exec")
cProfile.run(code, "/tmp/iso.prof")
pstats.Stats("/tmp/iso.prof").sort_stats("tottime").print_stats(14)

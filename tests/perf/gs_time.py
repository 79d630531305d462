import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from tests.perf import stencil_bench as sb
for n, reps in ((1024, 10), (2048, 5)):
    r = sb.gramschmidt(n, reps)
    print("GS", n, round(r["ms"], 4), round(r["us_per_step"], 3))

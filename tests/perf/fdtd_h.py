import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from tests.perf import stencil_bench as sb
r = sb.fdtd(1024, 500, 10)
print("H", os.environ.get("PB_FDTD_H", "8"), round(r["us_per_step"], 3), r["bitwise_f32"])

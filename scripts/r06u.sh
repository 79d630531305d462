make -j8 > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_stencil.py -q -m gpu --timeout 120 -x -k "fdtd" 2>&1 | tail -1
python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
r = sb.fdtd(1024, 500, 10)
print("T1024", round(r["us_per_step"], 3), r["bitwise_f32"])
PY

make -j8 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_stencil.py -q -m gpu --timeout 120 -x -k "gramschmidt or fdtd" 2>&1 | tail -2
python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
print(json.dumps(sb.gramschmidt(1024, 10)))
print(json.dumps(sb.gramschmidt(2048, 5)))
r = sb.fdtd(1024, 500, 10); print("fdtd", round(r["us_per_step"], 3), r["bitwise_f32"])
PY

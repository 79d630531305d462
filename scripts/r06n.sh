make -j8 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_stencil.py -q -m gpu --timeout 120 -x -k "fdtd" 2>&1 | tail -3
python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
print(json.dumps(sb.fdtd(1024, 500, 10)))
PY
PB_FDTD_STEPS=1 python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
print("steps", json.dumps(sb.fdtd(1024, 500, 10)))
PY

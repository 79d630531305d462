make -j8 > /dev/null 2>&1
for h in 4 8 16; do
PB_FDTD_H=$h timeout 300 python -m pytest tests/test_gpu_stencil.py -q -m gpu --timeout 120 -x -k "fdtd" 2>&1 | tail -1
PB_FDTD_H=$h python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
r = sb.fdtd(1024, 500, 10)
print("H", os.environ["PB_FDTD_H"], round(r["us_per_step"], 3), r["bitwise_f32"])
PY
done

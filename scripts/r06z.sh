make -j8 > /dev/null 2>&1
for r in 1 2; do
PB_C3_RPW=$r timeout 300 python -m pytest tests/test_gpu_stencil.py -q -m gpu --timeout 120 -x -k "conv3d" 2>&1 | tail -1
PB_C3_RPW=$r python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
for n in (1024, 512):
    r = sb.conv3d(n, 10)
    print("RPW", os.environ["PB_C3_RPW"], n, round(r["ms"], 4), round(r["frac"], 4))
PY
done

mkdir -p gpurun_out
make -j8 > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_stencil.py -q -m gpu --timeout 120 -x -k "conv" 2>&1 | tail -2
python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
print(json.dumps(sb.conv3d(1024, 10)))
print(json.dumps(sb.conv2d(16384, 10)))
print(json.dumps(sb.conv2d(4096, 10)))
print(json.dumps(sb.conv3d(512, 10)))
PY
PB_C3_ROWS=16 python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
print("rows16", json.dumps(sb.conv3d(1024, 10)))
PY

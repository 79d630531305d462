make -j8 > /dev/null 2>&1
timeout 300 python -m pytest tests/test_gpu_stencil.py -q -m gpu --timeout 120 -x -k "conv" 2>&1 | tail -2
python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
for f, n in ((sb.conv3d, 1024), (sb.conv3d, 512), (sb.conv2d, 16384), (sb.conv2d, 4096)):
    r = f(n, 10)
    print(r["kernel"], n, round(r["ms"], 4), round(r["frac"], 4))
PY

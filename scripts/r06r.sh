make -j8 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_stencil.py -q -m gpu --timeout 60 -x -k "gramschmidt" 2>&1 | tail -3
timeout 300 python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
print(json.dumps(sb.gramschmidt(1024, 10)))
print(json.dumps(sb.gramschmidt(2048, 5)))
PY

make -j8 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_stencil.py -q -m gpu --timeout 120 -x -k "fdtd" 2>&1 | tail -3
python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
print(json.dumps(sb.fdtd(1024, 500, 10)))
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:march -s 2 -c 1 -o gpurun_out/r06_conv3d_v3 -f python scripts/stencil_one.py conv3d 3 > /dev/null 2>&1; ls gpurun_out | grep v3

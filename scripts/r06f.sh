set -x
mkdir -p gpurun_out
make -j8 > /dev/null 2>&1
python - <<'PY'
import sys, os, json, statistics
sys.path.insert(0, "scripts")
import stencil_bench as sb
print(json.dumps(sb.conv3d(1024, 10)))
PY
PB_C3_ROWS=16 python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
print("rows16", json.dumps(sb.conv3d(1024, 10)))
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:march -s 2 -c 1 -o gpurun_out/r06_conv3d_v2 -f python scripts/stencil_one.py conv3d 3 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gs_kernel -s 1 -c 1 -o gpurun_out/r06_gs -f python scripts/stencil_one.py gramschmidt 2 > /dev/null 2>&1
ls gpurun_out | grep -E "conv3d_v2|r06_gs"

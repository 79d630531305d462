make -j8 > /dev/null 2>&1
for h in 0 8 9; do
PB_ST_L2=$h python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
r = sb.conv3d(1024, 10)
print("exp", os.environ["PB_ST_L2"], round(r["ms"], 4), round(r["frac"], 4))
PY
PB_ST_L2=$h timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum -k regex:march -s 2 -c 1 python scripts/stencil_one.py conv3d 3 2>&1 | grep -E "dram|gpu__"
done

mkdir -p gpurun_out
make -j8 > /dev/null 2>&1
for o in 0 1; do for h in 0 1 2; do
PB_ST_ORDER=$o PB_ST_L2=$h python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
r = sb.conv3d(1024, 10)
print("order", os.environ["PB_ST_ORDER"], "hint", os.environ["PB_ST_L2"], round(r["ms"], 4), round(r["frac"], 4))
PY
done; done
PB_ST_ORDER=1 PB_ST_L2=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_op_read_hit_rate.pct -k regex:march -s 2 -c 1 python scripts/stencil_one.py conv3d 3 2>&1 | grep -E "dram|gpu__|hit"

mkdir -p gpurun_out
make -j8 > /dev/null 2>&1
for h in 0 1 2; do
PB_ST_L2=$h python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
print("hint", os.environ["PB_ST_L2"], json.dumps(sb.conv3d(1024, 10)), json.dumps(sb.conv2d(16384, 10)), json.dumps(sb.conv2d(4096, 10)))
PY
done
PB_ST_L2=1 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_op_read_hit_rate.pct -k regex:march -s 2 -c 1 python scripts/stencil_one.py conv3d 3 2>&1 | grep -E "dram|gpu__|hit"

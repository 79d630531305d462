# r2u: raster group size in the power-capped suite (bench) and DRAM bytes of syr2k / syrk
mkdir -p gpurun_out
make -j8 > gpurun_out/r2u_make.log 2>&1 || tail -20 gpurun_out/r2u_make.log
for gm in 8 16 8 16; do
  PB_GROUP_M=$gm timeout 900 python bench.py --no-cpu --no-e2e --no-next > gpurun_out/r2u_bench_gm$gm.json 2>/dev/null
  python - "$gm" <<'PY'
import json, sys
l = [x for x in open(f"gpurun_out/r2u_bench_gm{sys.argv[1]}.json") if x.startswith('{')][-1]
d = json.loads(l)
print("gm", sys.argv[1], d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"], {k: v["frac"] for k, v in d["kernels"].items()})
PY
done
for gm in 8 16 12; do
  for k in "syr2k 8192" "syrk 8192" "3mm 4096"; do
    PB_GROUP_M=$gm timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:umma3x -c 1 --csv python scripts/time_calls.py $k 1 2>&1 | grep -E "umma3x" | awk -F'","' '{print $(NF-2), $NF}' | sed "s/^/gm=$gm $k /"
  done
done

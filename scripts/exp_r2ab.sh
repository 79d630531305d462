# r2ab: suite order — atax after bicg/mvt (clock recovery after syr2k) vs the current order
mkdir -p gpurun_out
make -j8 > gpurun_out/r2ab_make.log 2>&1 || tail -20 gpurun_out/r2ab_make.log
A=gemm,covariance,correlation,2mm,3mm,syrk,syr2k,atax,bicg,mvt,gesummv
B=gemm,covariance,correlation,2mm,3mm,syrk,syr2k,bicg,mvt,atax,gesummv
for rep in 1 2; do for o in A B; do
  eval ks=\$$o
  timeout 900 python bench.py --no-cpu --no-e2e --no-next --kernels $ks > gpurun_out/r2ab_$o$rep.json 2>/dev/null
  python - "$o$rep" <<'PY'
import json, sys
l = [x for x in open(f"gpurun_out/r2ab_{sys.argv[1]}.json") if x.startswith('{')][-1]
d = json.loads(l)
print(sys.argv[1], d["value"], d["ms_per_step"], d["clocks"]["sm_mhz"], {k: v["frac"] for k, v in d["kernels"].items()})
PY
done; done

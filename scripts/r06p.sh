make -j8 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_stencil.py -q -m gpu --timeout 120 -x -k "fdtd" 2>&1 | tail -3
python - <<'PY'
import sys, os, json
sys.path.insert(0, "scripts")
import stencil_bench as sb
print(json.dumps(sb.fdtd(1024, 500, 10)))
PY
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r06_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-next --graphs 0 > /dev/null 2>&1; wc -l gpurun_out/r06_launches.csv

#!/bin/bash
# config-matrix parity + compute-sanitizer on tests/perf/sanitize_r2.py (default plan)
mkdir -p gpurun_out
T=${TAG:-sn}
make -j8 > gpurun_out/${T}_make.log 2>&1 || tail -20 gpurun_out/${T}_make.log
[ -n "$CONFIGS" ] && timeout 1200 python -m pytest -x -q -m gpu tests/test_gpu_configs.py > gpurun_out/${T}_configs.log 2>&1; echo configs rc=$?; tail -3 gpurun_out/${T}_configs.log
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python tests/perf/sanitize_r2.py > gpurun_out/${T}_sanitizer_${tool}.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|True|False" gpurun_out/${T}_sanitizer_${tool}.log | head -12
done

# r2y: gram cluster barrier split (phase 0 before the cluster wait) — parity + timing
mkdir -p gpurun_out
make -j8 > gpurun_out/r2y_make.log 2>&1 || tail -20 gpurun_out/r2y_make.log
timeout 900 python -m pytest tests/test_gpu_gram_fused.py tests/test_gpu_fullsize.py -q -x --timeout 300 -k "gram or cov or corr" > gpurun_out/r2y_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r2y_pytest.log
for rep in 1 2 3; do for k in covariance correlation; do
  PB_FLUSH=1 timeout 300 python scripts/time_calls.py $k 2048 60 2>&1 >> gpurun_out/r2y_times.log
done; done
PB_GRAM_TIMING=1 timeout 300 python scripts/gram_timing.py > gpurun_out/r2y_stamps.log 2>&1
cat gpurun_out/r2y_times.log; grep -A14 "covariance call 2" gpurun_out/r2y_stamps.log | head -16

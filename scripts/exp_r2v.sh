# r2v: cov/corr split-K partner values by bulk copy (PB_GRAM_XBULK) — parity + timing
mkdir -p gpurun_out
make -j8 > gpurun_out/r2v_make.log 2>&1 || tail -20 gpurun_out/r2v_make.log
timeout 900 python -m pytest tests/test_gpu_gram_fused.py tests/test_gpu_fullsize.py -q -x --timeout 300 -k "gram or cov or corr" > gpurun_out/r2v_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r2v_pytest.log
for xb in 0 1 0 1; do
  for k in covariance correlation; do
    PB_FLUSH=1 PB_GRAM_XBULK=$xb timeout 300 python scripts/time_calls.py $k 2048 30 2>&1 | sed "s/^/xbulk=$xb /" >> gpurun_out/r2v_times.log
  done
done
PB_GRAM_TIMING=1 PB_GRAM_XBULK=1 timeout 300 python scripts/gram_timing.py > gpurun_out/r2v_stamps.log 2>&1
cat gpurun_out/r2v_times.log; grep -A14 "covariance call 2" gpurun_out/r2v_stamps.log | head -16

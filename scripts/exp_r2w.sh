# r2w: gram flags one 128-B line each vs packed
mkdir -p gpurun_out
make -j8 > gpurun_out/r2w_make.log 2>&1 || tail -20 gpurun_out/r2w_make.log
timeout 900 python -m pytest tests/test_gpu_gram_fused.py tests/test_gpu_fullsize.py -q -x --timeout 300 -k "gram or cov or corr" > gpurun_out/r2w_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r2w_pytest.log
for fs in 1 32 1 32; do
  for k in covariance correlation; do
    PB_FLUSH=1 PB_GRAM_FLAG_STRIDE=$fs timeout 300 python scripts/time_calls.py $k 2048 40 2>&1 | sed "s/^/fs=$fs /" >> gpurun_out/r2w_times.log
  done
done
for fs in 1 32; do PB_GRAM_TIMING=1 PB_GRAM_FLAG_STRIDE=$fs timeout 300 python scripts/gram_timing.py > gpurun_out/r2w_stamps_fs$fs.log 2>&1; done
cat gpurun_out/r2w_times.log; for fs in 1 32; do echo fs=$fs; grep -A4 "covariance call 2" gpurun_out/r2w_stamps_fs$fs.log; done

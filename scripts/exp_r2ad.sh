# r2ad: gram flag-release fence: fence.acq_rel.gpu (default) vs __threadfence (fence.sc)
mkdir -p gpurun_out
make -j8 > gpurun_out/r2ad_make.log 2>&1 || tail -20 gpurun_out/r2ad_make.log
timeout 900 python -m pytest tests/test_gpu_gram_fused.py tests/test_gpu_fullsize.py -q -x --timeout 300 -k "gram or cov or corr" > gpurun_out/r2ad_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r2ad_pytest.log
for rep in 1 2 3; do for sc in 0 1; do for k in covariance correlation; do
  PB_FLUSH=1 PB_GRAM_FENCE_SC=$sc timeout 300 python scripts/time_calls.py $k 2048 60 2>&1 | sed "s/^/sc=$sc /" >> gpurun_out/r2ad_times.log
done; done; done
sort gpurun_out/r2ad_times.log

# r2aa: split-K posts by bulk copy (PB_GRAM_XPOST) — parity + interleaved timing
mkdir -p gpurun_out
make -j8 > gpurun_out/r2aa_make.log 2>&1 || tail -20 gpurun_out/r2aa_make.log
PB_GRAM_XPOST=1 timeout 900 python -m pytest tests/test_gpu_gram_fused.py tests/test_gpu_fullsize.py -q -x --timeout 300 -k "gram or cov or corr" > gpurun_out/r2aa_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r2aa_pytest.log
for rep in 1 2 3; do for xp in 0 1; do for k in covariance correlation; do
  PB_FLUSH=1 PB_GRAM_XPOST=$xp timeout 300 python scripts/time_calls.py $k 2048 60 2>&1 | sed "s/^/xpost=$xp /" >> gpurun_out/r2aa_times.log
done; done; done
sort gpurun_out/r2aa_times.log

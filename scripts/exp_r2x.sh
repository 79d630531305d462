# r2x: xbulk x flag stride, interleaved repetitions
mkdir -p gpurun_out
make -j8 > gpurun_out/r2x_make.log 2>&1 || tail -20 gpurun_out/r2x_make.log
for rep in 1 2 3; do
  for xb in 0 1; do for fs in 1 32; do
    PB_FLUSH=1 PB_GRAM_XBULK=$xb PB_GRAM_FLAG_STRIDE=$fs timeout 300 python scripts/time_calls.py covariance 2048 60 2>&1 | sed "s/^/xb=$xb fs=$fs /" >> gpurun_out/r2x_times.log
  done; done
done
sort gpurun_out/r2x_times.log

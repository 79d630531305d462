# fused cov/corr: parity tests, phase stamps, graph-replay timing vs the 3-launch path
set -x
mkdir -p gpurun_out
make -j8 > gpurun_out/g1_make.log 2>&1 || tail -20 gpurun_out/g1_make.log
timeout 300 python -m pytest tests/test_gpu_gram_fused.py -x -q --timeout 120 > gpurun_out/g1_fused.log 2>&1; echo fused rc=$?
tail -30 gpurun_out/g1_fused.log
if ! grep -q " passed" gpurun_out/g1_fused.log || grep -q failed gpurun_out/g1_fused.log; then
  PB_GRAM_MNSWAP=1 timeout 300 python -m pytest tests/test_gpu_gram_fused.py -x -q --timeout 120 > gpurun_out/g1_fused_swap.log 2>&1; echo fused swap rc=$?
  tail -30 gpurun_out/g1_fused_swap.log
fi
PB_GRAM_TIMING=1 timeout 60 python scripts/gram_timing.py 2>&1 | tail -12
for k in covariance correlation; do
  PB_FLUSH=1 timeout 60 python scripts/time_calls.py $k 2048 30
  PB_GRAM_FUSED=0 PB_FLUSH=1 timeout 60 python scripts/time_calls.py $k 2048 30
done

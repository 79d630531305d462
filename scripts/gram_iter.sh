# one tuning iteration of the fused cov/corr kernel: parity, stamps, timing, ncu capture
mkdir -p gpurun_out
make -j8 > gpurun_out/g_make.log 2>&1 || tail -20 gpurun_out/g_make.log
for t in ${TMAS:-0}; do
echo "=== PB_GRAM_TMA=$t"
export PB_GRAM_TMA=$t
timeout 300 python -m pytest tests/test_gpu_gram_fused.py -q --timeout 120 > gpurun_out/g_fused_$t.log 2>&1; echo fused rc=$?
grep -E "passed|failed|Error" gpurun_out/g_fused_$t.log | tail -3
PB_GRAM_TIMING=1 timeout 60 python scripts/gram_timing.py 2>&1 | tail -12
for k in covariance correlation; do PB_FLUSH=1 timeout 60 python scripts/time_calls.py $k 2048 30; done
done
if [ -n "$NCU" ]; then bash scripts/gram_ncu.sh ${TAG:-g3} > /dev/null 2>&1; ls gpurun_out | grep ncu-rep; fi

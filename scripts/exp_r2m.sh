# r2m: per-rank 2mm / gemm (512 rows) plan variants
mkdir -p gpurun_out
make -j8 > gpurun_out/r2m_make.log 2>&1 || tail -20 gpurun_out/r2m_make.log
for v in "" "PB_UMMA_TILE=3 PB_UMMA_KSPLIT=2" "PB_UMMA_TILE=3 PB_UMMA_KSPLIT=3" "PB_STREAMK=1" "PB_UMMA_TILE=2 PB_UMMA_KSPLIT=2"; do
  for k in "2mm 512x4096" "gemm 512x4096x4096" "gemm 1024x4096x4096"; do
    env $v PB_FLUSH=1 timeout 300 python scripts/time_calls.py $k 10 2>&1 | sed "s/^/[$v] /" >> gpurun_out/r2m_times.log
  done
done
cat gpurun_out/r2m_times.log

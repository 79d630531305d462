# Experiments (r2h): cov stamps + clock in context; syr2k DRAM bytes vs split-K ordering.
mkdir -p gpurun_out
make -j8 > gpurun_out/r2h_make.log 2>&1 || tail -20 gpurun_out/r2h_make.log
PB_GRAM_TIMING=1 timeout 300 python scripts/cov_context.py > gpurun_out/r2h_cov_ctx_stamps.log 2>&1; echo ctx rc=$?
timeout 300 python scripts/cov_context.py > gpurun_out/r2h_cov_ctx.log 2>&1; echo ctx2 rc=$?
for ks in 0 1; do
  PB_UMMA_KSPLIT=$ks timeout 300 python scripts/time_calls.py syr2k 8192 5 > gpurun_out/r2h_syr2k_ks$ks.log 2>&1
  PB_UMMA_KSPLIT=$ks timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:umma3x -c 2 --csv python scripts/time_calls.py syr2k 8192 1 > gpurun_out/r2h_syr2k_ks${ks}_ncu.csv 2>&1
done
tail -3 gpurun_out/r2h_*.log

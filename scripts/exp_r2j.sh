# r2j: raster group and tail split-K cap for syr2k/syrk; cov flush variants; bench with write+read flush
mkdir -p gpurun_out
make -j8 > gpurun_out/r2j_make.log 2>&1 || tail -20 gpurun_out/r2j_make.log
timeout 300 python scripts/cov_context.py > gpurun_out/r2j_cov_ctx.log 2>&1; echo ctx rc=$?
for gm in 8 4 16; do for sm in 4 8; do
  for k in "syr2k 8192" "syrk 8192"; do
    PB_FLUSH=1 PB_GROUP_M=$gm PB_KSPLIT_MAX=$sm timeout 300 python scripts/time_calls.py $k 6 2>&1 | sed "s/^/gm=$gm smax=$sm /" >> gpurun_out/r2j_times.log
  done
done; done
for gm in 4 16; do
  PB_GROUP_M=$gm timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:umma3x -c 1 --csv python scripts/time_calls.py syr2k 8192 1 2>&1 | grep -E "umma3x" | awk -F'","' '{print $(NF-2), $NF}' | sed "s/^/gm=$gm /" >> gpurun_out/r2j_ncu.log
done
timeout 900 python bench.py > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err; echo bench rc=$?
cat gpurun_out/r2j_times.log gpurun_out/r2j_ncu.log; tail -4 gpurun_out/r2j_cov_ctx.log

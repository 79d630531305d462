# r2l: chained 2mm at per-rank shapes vs separate launches
mkdir -p gpurun_out
make -j8 > gpurun_out/r2l_make.log 2>&1 || tail -20 gpurun_out/r2l_make.log
for r in 512 1024 2048 4096; do
  for c in 0 1; do
    PB_FLUSH=1 PB_CHAIN=$c timeout 300 python scripts/time_calls.py 2mm ${r}x4096 10 2>&1 | sed "s/^/chain=$c /" >> gpurun_out/r2l_times.log
  done
done
cat gpurun_out/r2l_times.log

# r2ac: per-rank syrk/syr2k with stream-K (single-wave per-rank shapes) vs the default plan
mkdir -p gpurun_out
make -j8 > gpurun_out/r2ac_make.log 2>&1 || tail -20 gpurun_out/r2ac_make.log
for sk in 0 1; do
  PB_STREAMK=$sk timeout 900 python scripts/rank_shapes.py --only-syrk gpurun_out/r2ac_sk$sk.json > gpurun_out/r2ac_sk$sk.log 2>&1
  echo sk=$sk; tail -5 gpurun_out/r2ac_sk$sk.log
done

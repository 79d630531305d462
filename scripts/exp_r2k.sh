# r2k: per-rank proxy with split-last, and the syrk/syr2k partition cost ratio RHO
mkdir -p gpurun_out
make -j8 > gpurun_out/r2k_make.log 2>&1 || tail -20 gpurun_out/r2k_make.log
timeout 900 python scripts/rank_shapes.py gpurun_out/r2k_rank_shapes.json > gpurun_out/r2k_rank.log 2>&1; echo rank rc=$?
for rho in 120 165 210; do
  PB_RHO=$rho timeout 900 python scripts/rank_shapes.py --only-syrk gpurun_out/r2k_rank_rho$rho.json > gpurun_out/r2k_rank_rho$rho.log 2>&1; echo rho $rho rc=$?
done
tail -2 gpurun_out/r2k_rank*.log

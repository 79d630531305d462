# r2o: reproduce the PB_UMMA_TILE=1 config failure
mkdir -p gpurun_out
make -j8 > gpurun_out/r2o_make.log 2>&1 || tail -20 gpurun_out/r2o_make.log
PB_UMMA_TILE=1 timeout 600 python -m pytest -q -m gpu -x -p no:cacheprovider tests/test_gpu_parity.py -k "(gemm or 2mm or 3mm or syrk or syr2k or cov or corr) and not row_sharded and not discriminator and not listing8 and not variants" --timeout 120 > gpurun_out/r2o_tile1.log 2>&1; echo tile1 rc=$?
tail -60 gpurun_out/r2o_tile1.log
PB_SPLIT_FIRST=1 PB_UMMA_TILE=1 timeout 600 python -m pytest -q -m gpu -x -p no:cacheprovider tests/test_gpu_parity.py -k "(gemm or 2mm or 3mm or syrk or syr2k or cov or corr) and not row_sharded and not discriminator and not listing8 and not variants" --timeout 120 > gpurun_out/r2o_tile1_sf.log 2>&1; echo tile1sf rc=$?
tail -5 gpurun_out/r2o_tile1_sf.log

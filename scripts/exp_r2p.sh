# r2p: split -> GEMM overlap (PDL + panel counters): GEMM-family parity + timings on/off
mkdir -p gpurun_out
make -j8 > gpurun_out/r2p_make.log 2>&1 || tail -20 gpurun_out/r2p_make.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_configs.py -q -x --timeout 900 -k "gemm or 2mm or 3mm or syrk or syr2k or config" > gpurun_out/r2p_pytest.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/r2p_pytest.log
for ov in 0 1; do
  for k in "syr2k 8192" "syrk 8192" "2mm 4096" "3mm 4096" "gemm 4096"; do
    PB_FLUSH=1 PB_SPLIT_OVERLAP=$ov timeout 300 python scripts/time_calls.py $k 10 2>&1 | sed "s/^/ov=$ov /" >> gpurun_out/r2p_times.log
  done
done
cat gpurun_out/r2p_times.log

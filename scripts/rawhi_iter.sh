make -j8 > gpurun_out/rh_make.log 2>&1 || tail -20 gpurun_out/rh_make.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_configs.py tests/test_gpu_chain.py tests/test_gpu_streamk.py tests/test_gpu_dist.py tests/test_gpu_polybench_init.py -q -x --timeout 600 > gpurun_out/rh_tests.log 2>&1; echo tests rc=$?
grep -E "passed|failed|^E  " gpurun_out/rh_tests.log | head -8
for k in 2mm 3mm; do PB_FLUSH=1 timeout 120 python scripts/time_calls.py $k 4096 10; done
PB_FLUSH=1 timeout 120 python scripts/time_calls.py gemm 4096 10
PB_FLUSH=1 timeout 120 python scripts/time_calls.py syr2k 8192 5

mkdir -p gpurun_out
make -j8 > gpurun_out/r2t_make.log 2>&1 || tail -20 gpurun_out/r2t_make.log
PB_TRACE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 -k mixed > gpurun_out/r2t_mixed.log 2>&1; echo mixed rc=$?; grep "umma3x" gpurun_out/r2t_mixed.log | head -3; tail -2 gpurun_out/r2t_mixed.log
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x --timeout 300 > gpurun_out/r2t_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r2t_pytest.log

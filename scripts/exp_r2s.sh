mkdir -p gpurun_out
make -j8 > gpurun_out/r2s_make.log 2>&1 || tail -20 gpurun_out/r2s_make.log
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x --timeout 900 > gpurun_out/r2s_pytest.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/r2s_pytest.log

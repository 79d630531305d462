set -x
mkdir -p gpurun_out
make -j8 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_stencil.py -q -m gpu --timeout 120 -x > gpurun_out/r06e_pytest.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/r06e_pytest.log
timeout 600 python scripts/stencil_bench.py gpurun_out/r06e_stencil.json 2>&1 | tail -10

set -x
mkdir -p gpurun_out
make -j8 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_stencil.py -q -m gpu --timeout 120 -x -k gramschmidt > gpurun_out/r06d_pytest_gs.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/r06d_pytest_gs.log
timeout 600 python scripts/stencil_bench.py gpurun_out/r06d_stencil.json 2>&1 | tail -10

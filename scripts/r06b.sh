set -x
mkdir -p gpurun_out
make -j8 > gpurun_out/r06b_make.log 2>&1 || tail -20 gpurun_out/r06b_make.log
timeout 900 python -m pytest tests/test_gpu_stencil.py -q -m gpu --timeout 300 -x > gpurun_out/r06b_pytest_stencil.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/r06b_pytest_stencil.log
timeout 600 python scripts/stencil_bench.py gpurun_out/r06b_stencil.json 2>&1 | tail -10
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -4

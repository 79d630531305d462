set -x
mkdir -p gpurun_out
make -j8 > gpurun_out/r06_make.log 2>&1 || tail -20 gpurun_out/r06_make.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/r06_pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/r06_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r06_smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/r06_smoke.log
timeout 900 python bench.py > gpurun_out/r06_bench_default.json 2> gpurun_out/r06_bench.err; echo bench rc=$?
tail -c 3000 gpurun_out/r06_bench_default.json

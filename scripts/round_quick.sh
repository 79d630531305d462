# Quick GPU check (usage: TAG=r07 bash scripts/round_quick.sh under gpurun): GPU suite, smoke, bench.
set -x
mkdir -p gpurun_out
make -j8 > gpurun_out/${TAG:-r06}_make.log 2>&1 || tail -20 gpurun_out/${TAG:-r06}_make.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/${TAG:-r06}_pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/${TAG:-r06}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG:-r06}_smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/${TAG:-r06}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG:-r06}_bench_default.json 2> gpurun_out/${TAG:-r06}_bench.err; echo bench rc=$?
tail -c 3000 gpurun_out/${TAG:-r06}_bench_default.json

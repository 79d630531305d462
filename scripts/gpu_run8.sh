timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x -k atax 2>&1 | tail -2
PB_ATAX_CLUSTER=4 timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x -k atax 2>&1 | tail -2
PB_TRACE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --kernels atax 2>&1 | tail -2 | cut -c1-400
PB_TRACE=1 PB_ATAX_CLUSTER=4 timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --kernels atax 2>&1 | tail -2 | cut -c1-400

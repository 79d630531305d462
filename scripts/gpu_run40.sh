set -e
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_fullsize.py -q -x -k "cov or corr" 2>&1 | tail -2
for k in covariance correlation; do timeout 120 python scripts/time_calls.py $k 2048 30; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --kernels covariance,correlation 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"

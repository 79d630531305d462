set -e
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "cov or corr or gemm or mm" 2>&1 | tail -2
for k in covariance correlation; do timeout 120 python scripts/time_calls.py $k 2048 30; done
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step']); print({k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"

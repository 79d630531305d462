set -e
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "gemm" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu --kernels gemm 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"
ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --kernels gemm --graphs 0 2>/dev/null | grep small_gemm | tail -2 | awk -F'","' '{print $NF}'

timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k atax 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --kernels atax,bicg 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --kernels syr2k,atax 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:(v['ms'],v['frac']) for k,v in d['kernels'].items()}, d['clocks'])"

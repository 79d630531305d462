timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
PB_UMMA_KSPLIT=2 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "gemm or 2mm or 3mm or syr or cov or corr" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x 2>&1 | tail -1
PB_TRACE=1 timeout 100 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --kernels covariance,2mm,3mm,syrk,syr2k --graphs 0 2>&1 | grep "^\[pb\]" | sort | uniq -c
timeout 900 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['clocks']); print({k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"

timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x 2>&1 | tail -3
PB_UMMA_KSPLIT=3 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x -k "gemm or 2mm or 3mm or syrk or syr2k or cov or corr" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu --timeout 600 -x 2>&1 | tail -3
PB_TRACE=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --kernels covariance,correlation,2mm,3mm,syrk,syr2k 2>&1 | grep -v "^\[pb\]" | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:(v['ms'],v['frac']) for k,v in d['kernels'].items()}, d['clocks'])"
PB_TRACE=1 timeout 100 python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --kernels covariance,correlation,2mm,3mm,syrk,syr2k --graphs 0 2>&1 | grep "^\[pb\]" | sort | uniq -c
PB_UMMA_KSPLIT=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --kernels covariance,correlation,2mm,3mm,syrk,syr2k 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ks1', {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()}, d['clocks'])"

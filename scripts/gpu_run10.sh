timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x 2>&1 | tail -4
for t in 1 2 3; do PB_UMMA_TILE=$t timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x -k "gemm or 2mm or 3mm or syrk or syr2k or cov or corr or row_sharded" 2>&1 | tail -2; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu --timeout 600 -x 2>&1 | tail -3
for t in 0 2 3; do PB_UMMA_TILE=$t timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --kernels covariance,correlation,2mm,3mm,syrk,syr2k 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($t, {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()}, d['clocks'])"; done

timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu --timeout 600 -x 2>&1 | tail -5
for cg in 1 2; do PB_UMMA_CG=$cg timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --kernels covariance,correlation,2mm,3mm,syrk,syr2k 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($cg, {k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"; done

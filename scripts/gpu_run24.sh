timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 3 --cpu-budget 10 2>&1 | tail -1 > gpurun_out/bench24.json; python -c "import json; d=json.load(open('gpurun_out/bench24.json')); print(d['value'], d['ms_per_step'], d['clocks'], d.get('e2e',{}).get('value'), d['roofline']); print({k:(v['ms'],v['frac']) for k,v in d['kernels'].items()})"

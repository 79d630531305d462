make -j8 > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -m gpu --timeout 120 -x -k "cov or corr" 2>&1 | tail -2
for i in 1 2; do
python bench.py --kernels covariance,correlation --no-e2e --no-cpu --no-next --steps 30 --warmup 5 | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print({k:(v['ms'],v['ms_median'],v['frac']) for k,v in d['kernels'].items()}, d['clocks']['sm_mhz'])"
done

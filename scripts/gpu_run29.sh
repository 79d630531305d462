timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "cov or corr" 2>&1 | tail -3
timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -k "cov or corr" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
for k in covariance correlation; do timeout 120 python scripts/time_calls.py $k 2048 2>&1 | tail -1; done
timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l29.csv python bench.py --kernels covariance --steps 1 --warmup 3 --no-e2e --no-cpu --graphs 0 > /dev/null 2>&1

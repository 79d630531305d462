timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "cov or corr" 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -k "cov or corr" 2>&1 | tail -1
for f in 0 1; do for k in covariance correlation; do PB_COV_FUSED=$f timeout 120 python scripts/time_calls.py $k 2048 2>&1 | tail -1; done; done

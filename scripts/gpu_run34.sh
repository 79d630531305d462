timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -k "cov or corr" 2>&1 | tail -1

timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "atax" 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -k "atax" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_dist.py -q -m gpu 2>&1 | tail -1

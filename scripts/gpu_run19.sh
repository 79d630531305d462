for ks in 1 2; do PB_UMMA_TILE=3 PB_UMMA_KSPLIT=$ks timeout 120 python scripts/time_calls.py gemm 2048; done
PB_UMMA_TILE=3 PB_UMMA_KSPLIT=2 timeout 120 python scripts/time_calls.py covariance 2048
PB_UMMA_TILE=3 PB_UMMA_KSPLIT=4 timeout 120 python scripts/time_calls.py gemm 1024
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "gemm or cov or corr" 2>&1 | tail -1
PB_UMMA_KSPLIT=2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "gemm or cov or corr or syr" 2>&1 | tail -1

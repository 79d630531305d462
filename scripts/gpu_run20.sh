for ks in 1 2; do PB_UMMA_TIMING=1 PB_UMMA_TILE=3 PB_UMMA_KSPLIT=$ks timeout 120 python scripts/time_calls.py gemm 2048 2>&1 | tail -2; done
PB_UMMA_TIMING=1 PB_UMMA_TILE=3 PB_UMMA_KSPLIT=1 timeout 120 python scripts/time_calls.py gemm 4096 2>&1 | tail -2
PB_UMMA_TIMING=1 PB_UMMA_TILE=2 PB_UMMA_KSPLIT=1 timeout 120 python scripts/time_calls.py covariance 2048 2>&1 | tail -2
PB_UMMA_TIMING=1 PB_UMMA_TILE=3 PB_UMMA_KSPLIT=2 timeout 120 python scripts/time_calls.py covariance 2048 2>&1 | tail -2

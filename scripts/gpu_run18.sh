for ks in 1 2; do PB_UMMA_TILE=3 PB_UMMA_KSPLIT=$ks timeout 120 python scripts/time_calls.py gemm 2048; done
PB_UMMA_DEBUG=1 PB_UMMA_TILE=3 PB_UMMA_KSPLIT=2 timeout 120 python scripts/time_calls.py gemm 2048
for ks in 1 4; do PB_UMMA_TILE=3 PB_UMMA_KSPLIT=$ks timeout 120 python scripts/time_calls.py gemm 1024; done
PB_UMMA_DEBUG=1 PB_UMMA_TILE=3 PB_UMMA_KSPLIT=4 timeout 120 python scripts/time_calls.py gemm 1024
PB_UMMA_DEBUG=1 PB_UMMA_TILE=3 PB_UMMA_KSPLIT=2 timeout 120 python scripts/time_calls.py covariance 2048
PB_UMMA_TILE=2 PB_UMMA_KSPLIT=1 timeout 120 python scripts/time_calls.py covariance 2048

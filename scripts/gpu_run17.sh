for t in 2 3; do for ks in 1 2 4; do PB_UMMA_TILE=$t PB_UMMA_KSPLIT=$ks timeout 120 python scripts/time_calls.py covariance 2048; done; done
for t in 3; do for ks in 1 2; do PB_UMMA_TILE=$t PB_UMMA_KSPLIT=$ks timeout 120 python scripts/time_calls.py gemm 4096; done; done
PB_UMMA_TILE=2 PB_UMMA_KSPLIT=1 timeout 120 python scripts/time_calls.py gemm 4096

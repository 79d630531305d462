for t in 3; do for ks in 2 3 4; do PB_UMMA_TIMING=1 PB_UMMA_TILE=$t PB_UMMA_KSPLIT=$ks timeout 120 python scripts/time_calls.py covariance 2048 2>&1 | grep -v "^$" | tail -2; done; done
PB_UMMA_TIMING=1 timeout 120 python scripts/time_calls.py covariance 2048 2>&1 | grep -v "^$" | tail -2
timeout 120 python scripts/time_calls.py correlation 2048 2>&1 | tail -1
for ks in 2 3; do PB_UMMA_KSPLIT=$ks timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "cov or corr" 2>&1 | tail -1; done
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l21.csv python bench.py --kernels covariance --steps 1 --warmup 3 --no-e2e --no-cpu --graphs 0 > /dev/null 2>&1

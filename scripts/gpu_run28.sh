PB_UMMA_TIMING=1 timeout 120 python scripts/time_calls.py 2mm 4096 2>&1 | grep -v "^$" | tail -3
PB_UMMA_TIMING=1 timeout 120 python scripts/time_calls.py gemm 4096 2>&1 | grep -v "^$" | tail -2
timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l28.csv python scripts/time_calls.py 2mm 4096 3 > /dev/null 2>&1

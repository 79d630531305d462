for sh in 1024 256x4096x4096 512x4096x4096 768x4096x4096 2048; do timeout 60 python scripts/time_calls.py gemm $sh 10 | tail -1; PB_TRACE=1 timeout 60 python scripts/time_calls.py gemm $sh 2 2>&1 | grep umma3x | sort -u | head -1; done
for sh in 4096 512x4096; do timeout 60 python scripts/time_calls.py 2mm $sh 10 | tail -1; done

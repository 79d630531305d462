# umma_plan tuning: default plan vs forced tile/split-K on medium (per-rank) shapes
for sh in 256x4096x4096 512x4096x4096 768x4096x4096 1024x4096x4096 2048x4096x4096 512x8192x8192 1024x8192x8192; do
  d=$(timeout 60 python scripts/time_calls.py gemm $sh 10 | tail -1 | awk '{print $5}')
  line="$sh default=$d"
  for t in 1 2 3; do for ks in 1 2; do
    v=$(PB_UMMA_TILE=$t PB_UMMA_KSPLIT=$ks timeout 60 python scripts/time_calls.py gemm $sh 10 | tail -1 | awk '{print $5}')
    line="$line t${t}k${ks}=$v"
  done; done
  echo $line
  PB_TRACE=1 timeout 60 python scripts/time_calls.py gemm $sh 2 2>&1 | grep umma3x | sort -u | head -1
done

PB_UMMA_KSPLIT=1 timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:umma3x -s 6 -c 1 -o gpurun_out/prof_2mm_c3 -f \
   python bench.py --kernels 2mm --steps 1 --warmup 3 --no-e2e --no-cpu --graphs 0 > /dev/null 2>&1
PB_UMMA_KSPLIT=1 timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:umma3x -s 3 -c 1 -o gpurun_out/prof_gram_c3 -f \
   python bench.py --kernels covariance --steps 1 --warmup 3 --no-e2e --no-cpu --graphs 0 > /dev/null 2>&1
ls gpurun_out

for ks in 1 2; do
PB_UMMA_KSPLIT=$ks timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l15_$ks.csv \
   python bench.py --kernels covariance,2mm --steps 1 --warmup 3 --no-e2e --no-cpu --graphs 0 > /dev/null 2>&1
done
PB_UMMA_TILE=2 PB_UMMA_KSPLIT=1 timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/l15_t2.csv \
   python bench.py --kernels covariance --steps 1 --warmup 3 --no-e2e --no-cpu --graphs 0 > /dev/null 2>&1
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:stats_split -s 3 -c 1 -o gpurun_out/prof_stats -f \
   python bench.py --kernels covariance --steps 1 --warmup 3 --no-e2e --no-cpu --graphs 0 > /dev/null 2>&1
ls gpurun_out

timeout 600 ncu --cache-control none --metrics gpu__time_duration.sum,sm__cycles_active.avg,gpc__cycles_elapsed.max --clock-control none --csv --log-file gpurun_out/launches_cov3.csv \
   python bench.py --kernels covariance,correlation --steps 2 --warmup 3 --no-e2e --no-cpu --graphs 0 > /dev/null 2>&1
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:umma3x -s 4 -c 1 -o gpurun_out/prof_cov -f \
   python bench.py --kernels covariance --steps 1 --warmup 3 --no-e2e --no-cpu --graphs 0 > /dev/null 2>&1
ls gpurun_out

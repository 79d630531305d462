set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x 2>&1 | tail -15
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu --timeout 600 -k "atax or covariance or correlation or 2mm" 2>&1 | tail -8
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --kernels atax,covariance,correlation,gemm 2>&1 | tail -2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:atax -s 3 -c 1 -o gpurun_out/prof_atax2 -f \
   python bench.py --kernels atax --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cov2.csv \
   python bench.py --kernels covariance,correlation,gemm --steps 2 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ls gpurun_out

set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 2>&1 | tail -8
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -m gpu --timeout 600 2>&1 | tail -8
timeout 900 python bench.py --steps 10 --warmup 3 --cpu-budget 10 2>&1 | tail -3
# launch list of the bench command (cold, serialised: compare shares)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
   python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_bench.log 2>&1; tail -2 gpurun_out/ncu_bench.log
# full captures of the hot kernels (one launch each, after warm-up launches)
timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma3x -s 3 -c 1 -o gpurun_out/prof_syr2k -f \
   python bench.py --kernels syr2k --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:mvmt -s 3 -c 1 -o gpurun_out/prof_bicg -f \
   python bench.py --kernels bicg --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rowdot -s 3 -c 1 -o gpurun_out/prof_gesummv -f \
   python bench.py --kernels gesummv --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:umma3x -s 3 -c 1 -o gpurun_out/prof_2mm -f \
   python bench.py --kernels 2mm --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1
ls -la gpurun_out/

# r2r: atax_tm row slice as 1/2/4/8/16 bulk copies
mkdir -p gpurun_out
make -j8 > gpurun_out/r2r_make.log 2>&1 || tail -20 gpurun_out/r2r_make.log
for c in 1 2 4 8 16 1 4 8; do
  PB_ATAX_CHUNKS=$c timeout 300 python scripts/time_calls.py atax 32768 20 2>&1 | sed "s/^/chunks=$c /" >> gpurun_out/r2r_times.log
done
PB_ATAX_CHUNKS=8 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k atax > gpurun_out/r2r_pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/r2r_pytest.log
cat gpurun_out/r2r_times.log

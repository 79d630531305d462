# NEXT-4 chain fusion: 2mm/3mm parity (small, ragged, full size) and timing chained vs separate launches
make -j8 > gpurun_out/c_make.log 2>&1 || tail -20 gpurun_out/c_make.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -k "2mm or 3mm" --timeout 600 > gpurun_out/c_parity.log 2>&1; echo parity rc=$?
grep -E "passed|failed|^E  " gpurun_out/c_parity.log | head -8
for k in 2mm 3mm; do for n in 1024 4096; do
  PB_FLUSH=1 timeout 120 python scripts/time_calls.py $k $n 10
  PB_CHAIN=0 PB_FLUSH=1 timeout 120 python scripts/time_calls.py $k $n 10
done; done

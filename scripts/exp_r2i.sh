# r2i: split-last unit order — GEMM-family parity + timing/DRAM vs PB_SPLIT_FIRST=1
mkdir -p gpurun_out
make -j8 > gpurun_out/r2i_make.log 2>&1 || tail -20 gpurun_out/r2i_make.log
timeout 1200 python -m pytest tests -q -m gpu -x --timeout 600 -k "gemm or 2mm or 3mm or syrk or syr2k or chain or config or streamk or dist or fullsize" > gpurun_out/r2i_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/r2i_pytest.log
for sf in 1 0; do
  for k in "syr2k 8192" "syrk 8192" "2mm 4096" "3mm 4096" "gemm 4096"; do
    PB_FLUSH=1 PB_SPLIT_FIRST=$sf timeout 300 python scripts/time_calls.py $k 10 >> gpurun_out/r2i_times_sf$sf.log 2>&1
  done
  for k in "syr2k 8192" "syrk 8192" "2mm 4096"; do
    PB_SPLIT_FIRST=$sf timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:umma3x -c 2 --csv python scripts/time_calls.py $k 1 2>&1 | grep -E "umma3x" | awk -F'","' '{print $(NF-2), $NF}' >> gpurun_out/r2i_ncu_sf$sf.log
  done
done
cat gpurun_out/r2i_times_sf*.log gpurun_out/r2i_ncu_sf*.log

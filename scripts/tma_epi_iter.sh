#!/bin/bash
# A/B of the GEMM engine's staged TMA-store epilogue (PB_TMA_EPI=0: per-thread row stores).
mkdir -p gpurun_out
T=${TAG:-te}
make -j8 > gpurun_out/${T}_make.log 2>&1 || tail -20 gpurun_out/${T}_make.log
timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_streamk.py tests/test_gpu_chain.py > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/${T}_pytest.log
for cfg in "gemm 4096" "2mm 4096" "3mm 4096" "syrk 8192" "syr2k 8192" "2mm 1024" "3mm 1024" "gemm 1024" "2mm 512x4096" "syrk 2048"; do
  for e in 1 0; do
    PB_TMA_EPI=$e PB_FLUSH=1 timeout 120 python scripts/time_calls.py $cfg 30 2>&1 | tail -1 | sed "s/^/tma=$e /"
  done
done | tee gpurun_out/${T}_ab.log

set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 -x 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu --timeout 600 -k "atax or gemm" 2>&1 | tail -4
timeout 600 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu --kernels atax,gemm 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kernels'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:atax -s 3 -c 1 -o gpurun_out/prof_atax3 -f \
   python bench.py --kernels atax --steps 1 --warmup 3 --no-e2e --no-cpu > /dev/null 2>&1

# Round-2 evidence on one B200: GPU suite, smoke, default bench line, launch list of the
# bench step, ncu captures of the top kernels, per-rank proxy, cov phase stamps, and the
# N = 2 launch path (two ranks sharing the GPU). compute-sanitizer is closed on this pool.
set -x
mkdir -p gpurun_out
T=${TAG:-r2h}
make -j8 > gpurun_out/${T}_make.log 2>&1 || tail -20 gpurun_out/${T}_make.log
timeout 1800 python -m pytest tests -q -m gpu --timeout 900 > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench.err; echo bench rc=$?
tail -c 2500 gpurun_out/${T}_bench_default.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-next > /dev/null 2>&1; echo launches rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:gram_fused -s 2 -c 1 -o gpurun_out/${T}_cov_gram -f python scripts/gram_timing.py > /dev/null 2>&1; echo ncu gram rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:atax_tm -s 1 -c 1 -o gpurun_out/${T}_atax -f python scripts/time_calls.py atax 32768 2 > /dev/null 2>&1; echo ncu atax rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:umma3x -c 1 -o gpurun_out/${T}_syr2k_gemm -f python scripts/time_calls.py syr2k 8192 2 > /dev/null 2>&1; echo ncu syr2k rc=$?
timeout 900 ncu --set full --import-source on --clock-control none -k regex:umma3x -c 1 -o gpurun_out/${T}_2mm_gemm -f python scripts/time_calls.py 2mm 4096 2 > /dev/null 2>&1; echo ncu 2mm rc=$?
timeout 900 python scripts/rank_shapes.py gpurun_out/${T}_rank_shapes.json > gpurun_out/${T}_rank.log 2>&1; echo rank rc=$?
PB_GRAM_TIMING=1 timeout 300 python scripts/cov_context.py > gpurun_out/${T}_cov_stamps.log 2>&1; echo stamps rc=$?
PB_SHARE_GPU=1 PB_TRANSPORT=local timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29641 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu > gpurun_out/${T}_bench_share2.json 2> gpurun_out/${T}_bench_share2.err; echo share2 rc=$?
tail -c 1200 gpurun_out/${T}_bench_share2.json
ls gpurun_out | grep ${T}

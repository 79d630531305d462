# r2n: observation-split cov/corr (pb_<k>_dist) — dist tests + forced-dist bench
mkdir -p gpurun_out
make -j8 > gpurun_out/r2n_make.log 2>&1 || tail -20 gpurun_out/r2n_make.log
timeout 1500 python -m pytest tests/test_gpu_dist.py -q -x --timeout 900 > gpurun_out/r2n_pytest.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/r2n_pytest.log
PB_FORCE_DIST=1 MASTER_ADDR=127.0.0.1 MASTER_PORT=29631 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu --no-e2e --kernels covariance,correlation > gpurun_out/r2n_bench_forced.json 2> gpurun_out/r2n_bench_forced.err; echo bench rc=$?
tail -c 1500 gpurun_out/r2n_bench_forced.json; tail -5 gpurun_out/r2n_bench_forced.err

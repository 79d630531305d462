# r2q: bench with the isolated cov/corr replays in the aux line
mkdir -p gpurun_out
make -j8 > gpurun_out/r2q_make.log 2>&1 || tail -20 gpurun_out/r2q_make.log
timeout 900 python bench.py > gpurun_out/r2q_bench.json 2> gpurun_out/r2q_bench.err; echo bench rc=$?
head -c 1500 gpurun_out/r2q_bench.json; tail -c 1200 gpurun_out/r2q_bench.json

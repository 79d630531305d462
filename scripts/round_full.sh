# Round-end evidence on one B200 (usage: TAG=r07 bash scripts/round_full.sh under gpurun):
# full GPU suite, smoke, default bench line, NEXT-3 timings and ncu captures of their kernels.
set -x
mkdir -p gpurun_out
make -j8 > gpurun_out/${TAG:-r06}_make.log 2>&1 || tail -20 gpurun_out/${TAG:-r06}_make.log
timeout 1500 python -m pytest tests -q -m gpu --timeout 300 > gpurun_out/${TAG:-r06}_pytest_gpu.log 2>&1; echo pytest rc=$?
tail -5 gpurun_out/${TAG:-r06}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG:-r06}_smoke.log 2>&1; echo smoke rc=$?; tail -3 gpurun_out/${TAG:-r06}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG:-r06}_bench_default.json 2> gpurun_out/${TAG:-r06}_bench.err; echo bench rc=$?
tail -c 1500 gpurun_out/${TAG:-r06}_bench_default.json
timeout 600 python -m tests.perf.stencil_bench gpurun_out/${TAG:-r06}_stencil.json > /dev/null 2>&1
true
for k in conv2d conv3d fdtd_2d gramschmidt; do
  case $k in conv2d|conv3d) re=march;; fdtd_2d) re=fdtd_persist;; gramschmidt) re=gs_kernel;; esac
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$re -s 1 -c 1 -o gpurun_out/${TAG:-r06}_next_${k} -f python scripts/stencil_one.py $k 2 > /dev/null 2>&1
done
ls gpurun_out | grep r06

# bench + per-rank proxy + chain A/B (after the raw-hi split)
make -j8 > /dev/null 2>&1
timeout 900 python bench.py --no-cpu --no-next > gpurun_out/${TAG:-r2d}_bench.json 2> gpurun_out/${TAG:-r2d}_bench.err; echo bench rc=$?
tail -1 gpurun_out/${TAG:-r2d}_bench.json | python -c "import json,sys; r=json.loads(sys.stdin.read()); print(r['value'], r['ms_per_step'], r['clocks']['sm_mhz'], {k: v['frac'] for k, v in r['kernels'].items()})"
timeout 600 python scripts/rank_shapes.py gpurun_out/${TAG:-r2d}_rank_shapes.json 2>&1 | tail -1
for k in 2mm 3mm; do PB_FLUSH=1 timeout 120 python scripts/time_calls.py $k 4096 10; PB_CHAIN=1 PB_FLUSH=1 timeout 120 python scripts/time_calls.py $k 4096 10; done

#!/bin/bash
# atax variants: parity (PB_ATAX_VARIANT) + standalone timing + the suite's atax line.
mkdir -p gpurun_out
T=${TAG:-ax}
V=${V:-3}
make -j8 > gpurun_out/${T}_make.log 2>&1 || tail -20 gpurun_out/${T}_make.log
PB_ATAX_VARIANT=$V timeout 600 python -m pytest -x -q -m gpu tests/test_gpu_parity.py tests/test_gpu_fullsize.py -k "atax" > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/${T}_pytest.log
for v in 2 $V 2 $V; do PB_ATAX_VARIANT=$v PB_FLUSH=1 timeout 120 python scripts/time_calls.py atax 32768 30 2>&1 | tail -1 | sed "s/^/v=$v /"; done
for v in 2 $V 2 $V; do
  PB_ATAX_VARIANT=$v timeout 600 python bench.py --steps 30 --warmup 3 > gpurun_out/${T}_bench_v$v.log 2>&1
  python - "$v" gpurun_out/${T}_bench_v$v.log <<'PY'
import json,sys
v=sys.argv[1]
for l in open(sys.argv[2]):
    if l.startswith('{') and '"metric"' in l:
        d=json.loads(l); k=d["kernels"]
        print("v=%s bench atax %.4f ms frac %.3f | mvt %.3f bicg %.3f | clock %s value %.1f" % (v, k["atax"]["ms"], k["atax"]["frac"], k["mvt"]["frac"], k["bicg"]["frac"], d["clocks"]["sm_mhz"], d["value"]))
PY
done

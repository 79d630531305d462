set -x
nproc; free -g | head -2
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 2>&1 | tail -25
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -15
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --cpu-budget 10 2>&1 | tail -5
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -m gpu --timeout 600 2>&1 | tail -25

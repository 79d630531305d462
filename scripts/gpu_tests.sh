set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
python -c "import torch;print(torch.cuda.get_device_properties(0))"
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu --timeout 120 -k "pbgen or test_gemm" 2>&1 | tail -30
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu --timeout 120 2>&1 | tail -40

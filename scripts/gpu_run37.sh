PB_SPLIT_RAWHI=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "syrk or gemm_precision or gemm_integer or test_gemm" 2>&1 | grep -E "passed|failed|assert|Error" | head -12

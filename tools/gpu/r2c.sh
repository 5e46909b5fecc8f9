timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q -x 2>&1 | tail -30
timeout 1500 python -m pytest tests/test_parity_scale.py -m gpu -q -s -k "scale" 2>&1 | grep -E "parity|passed|failed|Error|assert" | tail -40

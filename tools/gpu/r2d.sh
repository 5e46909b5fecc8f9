rm -f gpurun_out/parity_scale.jsonl
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q 2>&1 | tail -30
timeout 2400 python -m pytest tests/test_parity_scale.py -m gpu -q -s -k "scale" 2>&1 | grep -E "passed|failed|Error|assert" | tail -20

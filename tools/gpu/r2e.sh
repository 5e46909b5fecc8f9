timeout 300 python tools/op_check.py mobilenet_v3_small_s50 reorder 2 2>&1 | grep -E "<<<|FAULT|Error" | head -20
timeout 300 python tools/op_check.py efficientnet_v2_s_s50 baseline 2 2>&1 | grep -E "<<<|FAULT|Error" | head -20
timeout 900 python -m pytest tests/test_engine_gpu.py tests/test_output_mode.py -m gpu -q 2>&1 | tail -8

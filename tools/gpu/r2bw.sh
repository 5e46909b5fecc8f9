timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q -x -k "direct or mobilenet or efficientnet" 2>&1 | grep -E "FAILED|passed|failed|Error" | head -8
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | cut -c1-700
UB_DIRECT_NOTMA=1 timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | cut -c1-700
timeout 300 python tools/sweep.py --set mobilenet 2>&1 | cut -c1-140

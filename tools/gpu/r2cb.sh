timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q -x -k "dwconv or depthwise or efficientnet or mobilenet or se_" 2>&1 | tail -2
python tools/one_conv.py dw 256 14 730 3 1
python tools/one_conv.py dw 256 28 387 3 2
python tools/one_conv.py dw 256 7 1159 3 1
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | cut -c1-500

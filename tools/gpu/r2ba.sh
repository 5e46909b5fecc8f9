timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py tests/test_parity_scale.py -m gpu -q -x -k "dwconv or depthwise or se_gate or mobilenet or efficientnet or effnet" 2>&1 | tail -3
python tools/one_conv.py dw 256 14 730 3 1
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | cut -c1-700
UB_SE_NOFUSEPOOL=1 timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | cut -c1-300
timeout 900 python tools/sweep.py --set mobilenet 2>&1 | cut -c1-400 | tail -6

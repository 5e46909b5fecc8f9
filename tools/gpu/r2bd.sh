timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q -x -k "direct or mobilenet or efficientnet or depthwise" 2>&1 | tail -4
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | cut -c1-800
python tools/op_times.py mobilenet_v3_small_s50 1 reorder fused 4 2>&1 | cut -c1-300

timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "halo" 2>&1 | tail -4
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 12 2>&1 | cut -c1-300

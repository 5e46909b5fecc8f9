timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "conv_matches" 2>&1 | tail -1
UB_HALO_MT4=1 timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "conv_matches and halo" 2>&1 | tail -1
python tools/bench_conv.py l1_conv2_3x3 2>&1 | tail -1
UB_HALO_MT4=1 python tools/bench_conv.py l1_conv2_3x3 2>&1 | tail -1
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | grep -o '"conv_halo3_kernel": {[^}]*}'
UB_HALO_MT4=1 timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | grep -o '"conv_halo3_kernel": {[^}]*}'

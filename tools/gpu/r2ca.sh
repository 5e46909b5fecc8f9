timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q -x -k "activation or eltwise or dwconv or efficientnet or se_" 2>&1 | tail -2
UB_BENCH_ACT=silu python tools/bench_conv.py eff_s5_expand eff_s6_expand eff_s4_expand 2>&1 | tail -3
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | cut -c1-500

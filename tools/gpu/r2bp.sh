for v in 0 1 2; do echo "variant $v"; UB_VARIANT=$v UB_BENCH_ACT=silu python tools/bench_conv.py eff_s5_expand eff_s6_expand eff_s4_expand; done
UB_BENCH_ACT=hardswish python tools/bench_conv.py eff_s5_expand
python tools/bench_conv.py eff_s5_expand l3_conv3_1016
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "activation" 2>&1 | tail -2
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | cut -c1-400

python tools/bench_conv.py eff_s5_expand eff_s5_expand_dense eff_s6_expand eff_s4_expand l3_conv3_1016
UB_BENCH_ACT=silu python tools/bench_conv.py eff_s5_expand eff_s5_expand_dense eff_s6_expand eff_s4_expand
for v in 1 2 3 5 17 21 65 69 81 8193; do echo "variant $v"; UB_VARIANT=$v UB_BENCH_ACT=silu python tools/bench_conv.py eff_s5_expand 2>&1 | tail -1; done

mkdir -p gpurun_out
N="ncu --set full --import-source on --clock-control none -c 1"
$N -k regex:dwconv -o gpurun_out/r2bv_dw python tools/one_conv.py dw 256 14 730 3 1 > gpurun_out/r2bv.log 2>&1
$N -k regex:gate_mul -s 3 -o gpurun_out/r2bv_mul python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 >> gpurun_out/r2bv.log 2>&1
$N -k regex:conv_direct -o gpurun_out/r2bv_direct python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 >> gpurun_out/r2bv.log 2>&1
UB_STEM_COUT=32 $N -k regex:stem_pool -o gpurun_out/r2bv_stemquad python tools/bench_stem.py --pool-only >> gpurun_out/r2bv.log 2>&1
UB_BENCH_ACT=silu $N -k regex:conv_tc -o gpurun_out/r2bv_silu python tools/bench_conv.py eff_s5_expand --once >> gpurun_out/r2bv.log 2>&1
ls gpurun_out/r2bv_*

mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:conv_tc -c 1 -o gpurun_out/r2bu_relu python tools/bench_conv.py eff_s5_expand --once > gpurun_out/r2bu.log 2>&1
UB_BENCH_ACT=hardswish ncu --set full --import-source on --clock-control none -k regex:conv_tc -c 1 -o gpurun_out/r2bu_hsw python tools/bench_conv.py eff_s5_expand --once >> gpurun_out/r2bu.log 2>&1
tail -2 gpurun_out/r2bu.log

mkdir -p gpurun_out
UB_BENCH_ACT=silu ncu --set full --import-source on --clock-control none -k regex:conv_tc -c 1 -o gpurun_out/r2bn_silu python tools/bench_conv.py eff_s5_expand --once > gpurun_out/r2bn.log 2>&1
tail -1 gpurun_out/r2bn.log

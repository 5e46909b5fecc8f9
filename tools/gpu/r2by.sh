mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:conv_halo -c 1 -o gpurun_out/r2by_halo python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 > gpurun_out/r2by.log 2>&1
tail -1 gpurun_out/r2by.log

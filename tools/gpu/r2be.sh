mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:dwconv -c 1 -o gpurun_out/r2be_dw python tools/one_conv.py dw 256 14 730 3 1 > gpurun_out/r2be.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:conv_direct -c 1 -o gpurun_out/r2be_direct python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 >> gpurun_out/r2be.log 2>&1
tail -3 gpurun_out/r2be.log

mkdir -p gpurun_out
ncu --set full --clock-control none -k regex:dwconv -c 1 -o gpurun_out/r2ay_dw python tools/one_conv.py dw 256 14 730 3 1 > gpurun_out/r2ay.log 2>&1
tail -3 gpurun_out/r2ay.log

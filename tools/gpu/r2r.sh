python tools/profile_step.py resnet50_s50 256 1 > gpurun_out/r2r_plain.log 2>&1 && \
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "step/" --set full --clock-control none --import-source on -k regex:conv_tc -s 2 -c 1 -o gpurun_out/r2r_top python tools/profile_step.py resnet50_s50 256 1 > gpurun_out/r2r_ncu.log 2>&1
tail -2 gpurun_out/r2r_ncu.log

timeout 600 python -m pytest tests/test_engine_gpu.py -m gpu -q -x -k "apply_plan_twin" 2>&1 | tail -2
python tools/profile_step.py resnet50_s50 256 1 > gpurun_out/r2af_plain.log 2>&1 && \
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "step/" --set full --clock-control none -k regex:conv_halo3 -s 9 -c 3 -o gpurun_out/r2af_halo python tools/profile_step.py resnet50_s50 256 1 > gpurun_out/r2af_ncu.log 2>&1
tail -2 gpurun_out/r2af_ncu.log

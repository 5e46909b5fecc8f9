python tools/profile_step.py resnet50_s50 1 3 > gpurun_out/r2t_plain.log 2>&1 && \
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2t_launches.csv python tools/profile_step.py resnet50_s50 1 1 > gpurun_out/r2t_ncu.log 2>&1
tail -2 gpurun_out/r2t_ncu.log

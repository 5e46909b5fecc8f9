mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/r2cm_plain.json 2>&1 && \
/usr/local/cuda/bin/ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2cm_launches.csv python bench.py --steps 2 --warmup 3 --no-extras --no-cpu-baseline > gpurun_out/r2cm_ncu.log 2>&1
tail -2 gpurun_out/r2cm_ncu.log

mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:gather_rows -c 1 -o gpurun_out/r2cq_g python /tmp/g.py > gpurun_out/r2cq.log 2>&1
tail -1 gpurun_out/r2cq.log

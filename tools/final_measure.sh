set -x
timeout 400 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 400 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_final.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv_tc -c 1 -o gpurun_out/full_l1c3 python tools/bench_conv.py l1_conv3 > gpurun_out/ncu_full1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:conv_tc -c 1 -o gpurun_out/full_fc python tools/bench_conv.py fc_dense > gpurun_out/ncu_full2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:avgpool_gather -c 1 -o gpurun_out/full_apg python -m pytest tests/test_kernels_gpu.py -q -k "avgpool_gather and 49-1816" > gpurun_out/ncu_full3.log 2>&1
ls gpurun_out

mkdir -p gpurun_out
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 200 > gpurun_out/r2bi_ops.jsonl 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:gate_mul -s 3 -c 1 -o gpurun_out/r2bi_mul python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 > gpurun_out/r2bi_ncu.log 2>&1
tail -1 gpurun_out/r2bi_ncu.log

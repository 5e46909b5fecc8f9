mkdir -p gpurun_out
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 200 > gpurun_out/r2bb_ops.jsonl 2>&1
timeout 600 ncu --set full --clock-control none -k regex:se_gate -s 20 -c 2 -o gpurun_out/r2bb_se python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 > gpurun_out/r2bb_ncu.log 2>&1
tail -2 gpurun_out/r2bb_ncu.log

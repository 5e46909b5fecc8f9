mkdir -p gpurun_out
timeout 300 python tools/op_times.py resnet50_s50 256 reorder fused 80 > gpurun_out/r2az_ops.jsonl 2>&1
tail -2 gpurun_out/r2az_ops.jsonl | cut -c1-200

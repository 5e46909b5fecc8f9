timeout 300 python tools/op_times.py densenet121_s50 128 reorder fused 40 > gpurun_out/r2cn_ops.jsonl 2>&1

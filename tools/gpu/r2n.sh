timeout 300 python tools/op_times.py densenet121_s50 128 reorder fused 40 2>&1 | tail -41

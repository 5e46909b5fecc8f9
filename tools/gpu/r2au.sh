timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | cut -c1-700

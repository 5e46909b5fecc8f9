timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 2>&1 | tail -28
timeout 300 python tools/op_times.py densenet121_s50 128 2>&1 | tail -28
timeout 300 python tools/op_times.py mobilenet_v3_small_s50 1 2>&1 | tail -28

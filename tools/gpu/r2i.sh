timeout 300 python tools/bench_gather.py 2>&1 | tail -8
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 2>&1 | head -1

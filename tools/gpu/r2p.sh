timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q -x 2>&1 | tail -3
timeout 300 python tools/bench_gather.py 2>&1 | tail -6
timeout 300 python tools/op_times.py densenet121_s50 128 reorder fused 3 2>&1 | head -1

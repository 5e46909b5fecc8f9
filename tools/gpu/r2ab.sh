timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "gather" 2>&1 | tail -2
timeout 300 python tools/bench_gather.py 2>&1 | tail -6
timeout 300 python tools/op_times.py densenet121_s50 128 reorder fused 1 2>&1 | head -1 | cut -c1-300

python tools/bench_se.py
UB_SE_WARPROWS=1 python tools/bench_se.py
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "se_gate or se_pool" 2>&1 | tail -2

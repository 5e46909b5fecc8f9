timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q -x -k "linear or mobilenet or se_" 2>&1 | tail -2
timeout 900 python tools/sweep.py --set mobilenet 2>&1 | cut -c1-170

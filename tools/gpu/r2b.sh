timeout 1500 python -m pytest tests/test_parity_scale.py tests/test_kernels_gpu.py -m gpu -q -s -k "scale or variant or production" 2>&1 | grep -v "^$" | tail -40

timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q -x -k "dwconv or depthwise" 2>&1 | tail -2
python tools/one_conv.py dw 256 14 730 3 1
python tools/one_conv.py dw 256 28 256 3 1
python tools/one_conv.py dw 256 56 96 3 2
python tools/one_conv.py dw 1 56 72 5 2

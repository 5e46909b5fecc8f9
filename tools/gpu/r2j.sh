timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "direct or dwconv or gather or linear or avgpool" 2>&1 | tail -4
timeout 900 python -m pytest tests/test_engine_gpu.py -m gpu -q -x -k "depthwise or densenet or resnet18" 2>&1 | tail -4
timeout 300 python tools/bench_gather.py 2>&1 | tail -6
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 2>&1 | head -16
timeout 300 python tools/op_times.py densenet121_s50 128 2>&1 | head -1

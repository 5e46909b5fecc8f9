python /tmp/g.py 2>/dev/null || true
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py tests/test_output_mode.py -m gpu -q -x -k "gather or densenet or output or join" 2>&1 | tail -2
timeout 300 python tools/op_times.py densenet121_s50 128 reorder fused 1 2>&1 | head -1 | cut -c1-300

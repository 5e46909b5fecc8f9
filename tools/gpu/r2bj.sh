timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q -x -k "eltwise or efficientnet or mobilenet or densenet or output_mode or join" 2>&1 | tail -2
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 200 > /tmp/ops.jsonl 2>&1
head -1 /tmp/ops.jsonl | cut -c1-700
grep '"mul' /tmp/ops.jsonl | cut -c1-60 | head -8

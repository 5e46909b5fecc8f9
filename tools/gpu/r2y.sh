timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q -x -k "se_gate or depthwise" 2>&1 | tail -2
timeout 600 python tools/sweep.py --set mobilenet 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['upscale']['ms'], d['baseline_copy']['ms'], d['upscale_speedup'], d['upscale']['launches'])"
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | cut -c1-700

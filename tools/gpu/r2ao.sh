timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q -x -k "halo or activation or depthwise or conv_matches" 2>&1 | tail -2
timeout 900 python tools/sweep.py --set config5 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['upscale']['ms'], d['upscale']['images_per_s'], d['upscale']['roofline_frac'], d['baseline_copy']['images_per_s'], d['upscale_speedup'])"

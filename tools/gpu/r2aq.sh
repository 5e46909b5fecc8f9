timeout 900 python -m pytest tests/test_engine_gpu.py -m gpu -q -x 2>&1 | tail -2
timeout 900 python tools/sweep.py --set config5 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['upscale']['ms'], d['upscale']['images_per_s'], d['upscale']['roofline_frac'], d['baseline_copy']['images_per_s'], d['upscale_speedup'])"
timeout 600 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('R50', d['value'], d['ms_per_step'])"

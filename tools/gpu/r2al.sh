timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "stem" 2>&1 | tail -2
python tools/bench_stem.py 2>&1 | head -1
timeout 600 python tools/sweep.py --set mobilenet 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'], d['upscale']['ms'], d['baseline_copy']['ms'], d['upscale_speedup'])"
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('R50', d['value'], d['b1_latency_ms'], d['b1_baseline_export_ms'])"

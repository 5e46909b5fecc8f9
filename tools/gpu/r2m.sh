for i in 1 2; do
  (cd _ab/r2a && timeout 600 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('OLD', d['value'], d['ms_per_step'], d['roofline']['eager_sum_ms'])")
  timeout 600 python bench.py --steps 30 --warmup 5 --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('NEW', d['value'], d['ms_per_step'], d['roofline']['eager_sum_ms'])"
done
timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "activation or conv_matches or halo" 2>&1 | tail -2

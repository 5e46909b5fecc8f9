timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q -x -k "stem or resnet50 or densenet" 2>&1 | tail -1
for f in 0 128; do echo "flags $f"; UB_DEBUG_FLAGS=$f UB_STEM_COUT=64 python tools/bench_stem.py 2>/dev/null | head -1; UB_DEBUG_FLAGS=$f UB_STEM_COUT=48 python tools/bench_stem.py 2>/dev/null | head -1; done
for i in 1 2; do
timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('new', d['value'], d['ms_per_step'])"
UB_DEBUG_FLAGS=128 timeout 600 python bench.py --gpus 1 --steps 20 --warmup 5 --no-extras --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('old', d['value'], d['ms_per_step'])"
done

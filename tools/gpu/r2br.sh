timeout 600 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "stem" 2>&1 | tail -3
for c in 32 64; do echo "cout $c"; UB_STEM_COUT=$c timeout 120 python tools/bench_stem.py --pool-only; UB_SP_NOQUAD=1 UB_STEM_COUT=$c timeout 120 python tools/bench_stem.py --pool-only; done
timeout 300 python tools/op_times.py resnet50_s50 256 reorder fused 1 2>&1 | tail -1 | cut -c1-200

timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "conv_matches or activation" 2>&1 | tail -2
python tools/bench_conv.py l1_conv2_3x3 l2_conv2_3x3 l3_conv2_3x3 l4_conv2_3x3 2>&1 | tail -4
UB_HALO_NOEPI4=1 python tools/bench_conv.py l1_conv2_3x3 l2_conv2_3x3 l3_conv2_3x3 l4_conv2_3x3 2>&1 | tail -4
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | cut -c1-600
UB_HALO_NOEPI4=1 timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | cut -c1-600
timeout 600 python bench.py --gpus 1 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"
UB_HALO_NOEPI4=1 timeout 600 python bench.py --gpus 1 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"

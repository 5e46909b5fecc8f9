UB_BENCH_ACT=silu python tools/bench_conv.py eff_s5_expand 2>&1 | tail -1
python tools/bench_conv.py eff_s5_expand l1_conv3 l3_conv3_1016 l3_conv2_3x3 2>&1 | tail -4
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | cut -c1-500
timeout 600 python bench.py --gpus 1 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['b1_latency_ms'])"

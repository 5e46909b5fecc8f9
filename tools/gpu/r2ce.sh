python tools/bench_conv.py r50_l4_2_conv1 l3_conv1_cover r50_l2_3_conv1 l1_conv1_slice r50_l1_0_conv1 eff_s5_expand 2>&1 | tail -6
UB_CONV_EPI4_ALL=1 python tools/bench_conv.py r50_l4_2_conv1 l3_conv1_cover r50_l2_3_conv1 l1_conv1_slice r50_l1_0_conv1 eff_s5_expand 2>&1 | tail -6
timeout 600 python bench.py --gpus 1 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"
UB_CONV_EPI4_ALL=1 timeout 600 python bench.py --gpus 1 --steps 10 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"

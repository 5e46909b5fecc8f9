timeout 900 python -m pytest tests -m gpu -q -x --deselect tests/test_parity_scale.py 2>&1 | tail -15
timeout 300 python tools/op_times.py densenet121_s50 128 2>&1 | head -1
timeout 300 python tools/op_times.py mobilenet_v3_small_s50 1 2>&1 | head -8
timeout 300 python tools/sweep.py --set mobilenet 2>&1 | tail -6

timeout 300 python tools/op_times.py resnet101_s30 256 reorder fused 3 2>&1 | cut -c1-330

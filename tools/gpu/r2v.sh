python tools/one_conv.py dw 256 14 730 3 1
python tools/one_conv.py dw 256 28 256 3 1
python tools/one_conv.py dw 1 56 72 5 2
python tools/one_conv.py dw 256 14 730 3 1 && /usr/local/cuda/bin/ncu --set full --clock-control none -k regex:dwconv -s 3 -c 1 -o gpurun_out/r2v_dw python tools/one_conv.py dw 256 14 730 3 1 > /dev/null 2>&1
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 3 2>&1 | head -1 | cut -c1-600

timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_engine_gpu.py -m gpu -q -x -k "eltwise or direct or dwconv or depthwise or efficientnet or mobilenet" 2>&1 | tail -3
for v in "" 1; do
if [ -n "$v" ]; then export UB_DW_NOTMA=1; else unset UB_DW_NOTMA; fi; echo "NOTMA=$v"
python tools/one_conv.py dw 256 14 730 3 1
python tools/one_conv.py dw 256 28 256 3 1
python tools/one_conv.py dw 256 7 1159 3 1
python tools/one_conv.py dw 256 28 387 3 2
done
unset UB_DW_NOTMA
timeout 300 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 1 2>&1 | head -1 | cut -c1-800

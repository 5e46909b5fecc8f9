timeout 600 python -m pytest tests/test_kernels_gpu.py tests/test_output_mode.py -m gpu -q -x -k "eltwise or output or join" 2>&1 | tail -2
python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 200 | grep '"add' | cut -c1-60
UB_ELT_GENERIC_ADD=1 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 200 | grep '"add' | cut -c1-60

for cap in 0 4 8 16; do echo "cap $cap"; UB_ADD_CAP=$cap python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 200 | grep '"add' | cut -c1-60; done
UB_ELT_GENERIC=1 python tools/op_times.py efficientnet_v2_s_s50 256 reorder fused 200 | grep '"add' | cut -c1-60

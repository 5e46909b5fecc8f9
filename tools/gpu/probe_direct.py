import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2307_08771_b200 import _lib, kernels as K
cin, k, s, cout, H, W = map(int, sys.argv[1:7])
dev = "cuda"
x = torch.randn(2, 3, H, W, device=dev)
idx = torch.tensor([2, 0, 1][:cin], dtype=torch.int32, device=dev)
wd = torch.randn(k * k, cin, _lib.load().ub_conv_direct_wcols(cout), device=dev)
b = torch.randn(cout, device=dev)
Ho, Wo = (H + 2 * (k // 2) - k) // s + 1, (W + 2 * (k // 2) - k) // s + 1
y = K.empty_act(2, Ho, Wo, cout, dev)
K.conv_direct(x, idx, wd, b, cout, k, s, k // 2, 0, y)
torch.cuda.synchronize()
print("ok", sys.argv[1:])

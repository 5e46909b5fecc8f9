cat > /tmp/g.py <<'PY'
import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2307_08771_b200 import kernels as K
dev = "cuda"
N, H, C = 128, 56, 128
x = K.empty_act(N, H, H, C, dev); x.buf.normal_()
idx = torch.randperm(C)[:127].sort().values.to(torch.int32).to(dev)
y = K.empty_act(N, H // 2, H // 2, 128, dev)
sc = torch.rand(127, device=dev) + 0.5; sh = torch.randn(127, device=dev)
for _ in range(3):
    K.gather_rows_ex(x, idx, K.gather_window(idx.tolist()), 1, y, scale=sc, shift=sh, relu=True, pool2=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(20):
    K.gather_rows_ex(x, idx, K.gather_window(idx.tolist()), 1, y, scale=sc, shift=sh, relu=True, pool2=True)
b.record(); torch.cuda.synchronize()
print("pool2 gather 128x56x56x128 -> 28x28:", a.elapsed_time(b) / 20 * 1e3, "us")
PY
mkdir -p gpurun_out
ncu --set full --import-source on --clock-control none -k regex:gather_rows -c 1 -o gpurun_out/r2cq_g python /tmp/g.py > gpurun_out/r2cq.log 2>&1
tail -1 gpurun_out/r2cq.log

"""Per-tile event clocks of CTA 0 of conv_tc_kernel (dev tool; UB_CONV_TRACE=1).

python tools/conv_trace.py <bench_conv case> [variant]
columns: mma:start tempty_ok committed | epi:start tfull_ok tempty_arrive | prod:start done
"""
import os
import sys
from pathlib import Path

os.environ["UB_CONV_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import torch  # noqa: E402

from paper_2307_08771_b200 import _lib, kernels as K  # noqa: E402
import bench_conv  # noqa: E402


def main():
    name = sys.argv[1]
    variant = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    N, H, W, cs, coff, cin, cout, k, st, pad, ng, use_r, relu = bench_conv.CASES[name]
    dev = "cuda"
    x = K.Act(torch.randn(N * H * W, cs, device=dev).to(torch.bfloat16), N, H, W, cs).view(coff, cin)
    lead, cpad = _lib.conv_weight_layout(cin, coff, False, k, k)
    wg = K.permute_weights(torch.randn(cout, cin, k, k, device=dev), list(range(cout)), list(range(cin)),
                           layout="gemm", lead=lead, cpad=cpad, out_dtype=torch.bfloat16)
    Ho, Wo = (H + 2 * pad - k) // st + 1, (W + 2 * pad - k) // st + 1
    y = K.empty_act(N, Ho, Wo, cout, dev)
    res = K.empty_act(N, Ho, Wo, cout, dev) if use_r else None
    for _ in range(3):
        K.conv(x, wg, lead, cpad, cout, k, k, st, pad, y, bias=torch.zeros(cout, device=dev), relu=relu,
               residual=res, variant=variant)
    torch.cuda.synchronize()
    lib = _lib.load()
    import ctypes
    lib.ub_debug_conv_trace.restype = ctypes.c_void_p
    ptr = lib.ub_debug_conv_trace()
    t = torch.empty(64 * 8, dtype=torch.int64, device=dev)
    import cuda.bindings.runtime as rt
    rt.cudaMemcpy(t.data_ptr(), ptr, 64 * 8 * 8, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
    torch.cuda.synchronize()
    v = t.cpu().view(64, 8).tolist()
    t0 = v[0][0]
    print(__doc__.strip().splitlines()[-1])
    for i, r in enumerate(v[:24]):
        print(i, [x - t0 if x else None for x in r])


if __name__ == "__main__":
    main()

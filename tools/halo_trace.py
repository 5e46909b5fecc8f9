"""Per-tile event clocks of CTA 0 of the halo kernel (dev tool; UB_HALO_TRACE=1)."""
import ctypes
import os
import sys
from pathlib import Path

os.environ["UB_HALO_TRACE"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2307_08771_b200 import _lib, kernels as K  # noqa: E402


def main():
    # args: cin [H=W [cout [N]]]
    a = [int(v) for v in sys.argv[1:]]
    cin = a[0] if a else 32
    H = W = a[1] if len(a) > 1 else 56
    cout = a[2] if len(a) > 2 else 64
    N = a[3] if len(a) > 3 else 256
    dev = "cuda"
    x = K.Act(torch.randn(N * H * W, cin, device=dev).to(torch.bfloat16), N, H, W, cin)
    lead, cpad = _lib.conv_weight_layout(cin, 0, False, 3, 3)
    wg = K.permute_weights(torch.randn(cout, cin, 3, 3, device=dev), list(range(cout)), list(range(cin)),
                           layout="gemm", lead=lead, cpad=cpad, out_dtype=torch.bfloat16)
    y = K.empty_act(N, H, W, cout, dev)
    for _ in range(3):
        K.conv(x, wg, lead, cpad, cout, 3, 3, 1, 1, y, bias=torch.zeros(cout, device=dev), relu=True)
    torch.cuda.synchronize()
    lib = _lib.load()
    lib.ub_debug_halo_trace.restype = ctypes.c_void_p
    ptr = lib.ub_debug_halo_trace()
    t = torch.empty(64 * 16, dtype=torch.int64, device=dev)
    import cuda.bindings.runtime as rt
    rt.cudaMemcpy(t.data_ptr(), ptr, 64 * 16 * 8, rt.cudaMemcpyKind.cudaMemcpyDeviceToDevice)
    torch.cuda.synchronize()
    v = t.cpu().view(64, 16).tolist()
    t0 = v[0][0]
    print("tile  mma:start tempty_ok afull_ok issued | epi:start tfull_ok tempty_arr | prod:stage_free |"
          " epi warp0 per chunk: ld_done bulkwait_done emit_done store_issued (x2)")
    for i, r in enumerate(v[:40]):
        print(i, [x - t0 if x else None for x in r])


if __name__ == "__main__":
    main()

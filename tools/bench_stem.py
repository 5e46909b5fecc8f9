"""Time the space-to-depth stem launches separately (development tool).

python tools/bench_stem.py [N]
"""

import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_08771_b200 import _lib, kernels as K  # noqa: E402


def timeit(fn, reps=20):
    """Device time per call: `reps` calls captured in one CUDA graph (no host launch gaps)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    N = int(args[0]) if args else 256
    dev = "cuda"
    x = torch.randn(N, 3, 224, 224, device=dev)
    idx = torch.tensor([2, 0], dtype=torch.int32, device=dev)
    cout, k, pad = int(os.environ.get("UB_STEM_COUT", "64")), 7, 3  # ResNet-50 @ 50 %: 32 kept
    Wt = torch.randn(cout, 2, k, k, device=dev) / 10
    wg = K.permute_weights(Wt, list(range(cout)), [0, 1], layout="s2d", out_dtype=torch.bfloat16)
    bias = torch.randn(cout, device=dev)
    y = K.empty_act(N, 112, 112, cout, dev)
    sbuf = K.s2d_buffer(N, 224, 224, k, pad, dev)
    lib = _lib.load()

    def pack():
        _lib.check(lib.ub_stem_s2d_pack(K._p(x), N, 3, 224, 224, K._p(idx), 2, k, pad, K._p(sbuf), K._stream()))

    def conv():
        _lib.check(lib.ub_conv_s2d(K._p(sbuf), N, 224, 224, k, pad, K._p(wg), cout, K._p(bias), 1, K._p(y.buf),
                                   y.cstride, y.coff, K._stream()))

    yp = K.empty_act(N, 56, 56, cout, dev)

    def pool():
        _lib.check(lib.ub_conv_s2d_maxpool(K._p(sbuf), N, 224, 224, k, pad, K._p(wg), cout, K._p(bias), 1, 3, 2, 1,
                                           K._p(yp.buf), yp.cstride, yp.coff, K._stream()))

    if "--pack-only" in sys.argv:
        for _ in range(3):
            pack()
        torch.cuda.synchronize()
        return
    if "--pool-only" in sys.argv:
        for _ in range(3):
            pool()
        torch.cuda.synchronize()
        return
    tpool = timeit(pool)
    print(f"conv+maxpool {tpool:8.1f} us")
    tf = timeit(lambda: K.stem_maxpool(x, idx, wg, cout, k, pad, yp, bias=bias, relu=True))
    print(f"fused pack+conv+maxpool {tf:8.1f} us")
    tp, tc = timeit(pack), timeit(conv)
    out_b = N * 112 * 112 * cout * 2
    s_b = sbuf.numel() * 2
    in_b = N * 2 * 224 * 224 * 4
    print(f"pack {tp:8.1f} us  ({(in_b + s_b) / tp / 1e3:7.1f} GB/s)")
    print(f"conv {tc:8.1f} us  ({(s_b + out_b) / tc / 1e3:7.1f} GB/s, out {out_b / 1e6:.0f} MB)")
    print(f"both {timeit(lambda: (pack(), conv())):8.1f} us")


if __name__ == "__main__":
    main()

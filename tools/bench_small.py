"""Graph-timed small ops (dev tool): avgpool over [256, 7, 7, C], channel_gather_2d."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from paper_2307_08771_b200 import kernels as K  # noqa: E402
from bench_stem import timeit  # noqa: E402


def main():
    dev = "cuda"
    for C in (1816, 2048):
        x = K.empty_act(256, 7, 7, C, dev)
        x.buf.normal_()
        y = K.empty_act(256, 1, 1, C, dev)
        t = timeit(lambda: K.avgpool_global(x, y))
        print(f"avgpool 256x7x7x{C}: {t:7.1f} us  ({x.buf.numel() * 2 / t / 1e3:7.1f} GB/s)")
    x = K.empty_act(256, 14, 14, 1016, dev)
    x.buf.normal_()
    idx = torch.arange(0, 1016, 2, dtype=torch.int32, device=dev)
    for st in (1, 2):
        ho = (14 - 1) // st + 1
        y = K.empty_act(256, ho, ho, idx.numel(), dev)
        t = timeit(lambda: K.channel_gather_2d(x, idx, st, y))
        rd = 256 * ho * ho * 1016 * 2
        print(f"gather_2d 256x14x14x1016 -> 508 stride {st}: {t:7.1f} us  ({(rd + y.buf.numel() * 2) / t / 1e3:7.1f} GB/s)")


if __name__ == "__main__":
    main()

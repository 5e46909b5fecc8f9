"""B200-native (sm_100a) hot path for UPSCALE-exported pruned CNNs.

Drop-in for the reference `reslice` package's export + inference path:
masks -> `plan_model` (the reference's planner, or its committed plan files)
-> `export_model` (GPU permute kernel) -> `run` (tcgen05 implicit-GEMM convs).
"""

__version__ = "0.1.0"

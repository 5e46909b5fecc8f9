"""Parity at the bench configuration, at scale (>= 1024 images per export).

The engines are built exactly as bench.py builds them (batch 256, autotuned
variants, CUDA-graph replay, default torchvision BN -- the BASELINE.json
configs); four batches of 256 seeded standard-normal images run through the
graph and through the fp32 CPU oracle (oracle/spatial_ref.py over the same
exported graph, weights permuted by the numpy apply_plan restatement).

Gates (SURVEY.md 8d / north_star):
  * the reference's relative metric (interp.py:119-120) <= 2e-2 over all 1024 x 1000 logits,
    and the max error relative to the logits' own scale <= 2e-2 (the reference metric's
    max(1, |x|) floor makes it vacuous for tiny random-init logits);
  * top-1 agreement >= 99.9 % (at most one disagreement in 1024) -- where the model's
    logits are decisive.  Random-init ResNet-50/18 with default BN (the bench config) is
    NOT: its logits span |x| <= 0.12 with a median top-1/top-2 margin of 8e-4 (R50), so
    merely rounding the input and weights to bf16 and running the fp32 oracle on them (no
    GPU code at all) already flips 4.4 % of the top-1 classes.  There the gate is the
    CPU-only precision control: the fp32 oracle re-run with bf16 input, bf16 weights and
    every node's output rounded to bf16 (the reference at the GPU's storage precision);
    the engine must agree with the fp32 oracle at least as often as that control, within
    two binomial standard errors.  Well-conditioned instances (ResNet-101 and DenseNet-121
    with default BN; randomised-BN ResNet-50/18 with margins ~0.1) meet the absolute
    >= 99.9 % gate.
"""

import json
import os

import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle.apply_plan_ref import apply_plans_spatial  # noqa: E402
from oracle.spatial_ref import deviation, run_spatial, top1_agreement  # noqa: E402
from paper_2307_08771_b200 import engine as EN, export as E, plans as P  # noqa: E402
from paper_2307_08771_b200.configs import CONFIGS, build_spatial_model  # noqa: E402

TOL = 2e-2
TOP1 = 0.999
BATCH = 256
N_BATCHES = 4

_models = {}


def _model(cfg_name):
    if cfg_name not in _models:
        _models[cfg_name] = build_spatial_model(CONFIGS[cfg_name])
    return _models[cfg_name]


def _record(rec):
    print(json.dumps(rec))
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "parity_scale.jsonl"), "a") as f:
            f.write(json.dumps(rec) + "\n")


@pytest.mark.parametrize("cfg_name,strategy,gather_mode,rbn", [
    ("resnet50_s50", "reorder", "fused", False),    # the bench engine (north-star config)
    ("resnet50_s50", "baseline", "copy", False),    # the baseline-export arm (copy-then-conv)
    ("resnet50_s50", "baseline", "fused", False),   # baseline plans with the fused read plans
    ("resnet18_s50", "reorder", "fused", False),
    ("resnet101_s50", "reorder", "fused", False),
    ("resnet50_s50", "reorder", "fused", True),     # randomised BN: decisive logits
    ("resnet18_s50", "baseline", "copy", True),
    ("densenet121_s50", "reorder", "fused", False),  # config 4 (batch 128)
    ("densenet121_s50", "reorder", "fused", True),
    ("mobilenet_v3_small_s50", "reorder", "fused", False),  # config 2 model
    ("mobilenet_v3_small_s50", "baseline", "copy", False),
    ("mobilenet_v3_small_s50", "reorder", "fused", True),
    ("efficientnet_v2_s_s50", "reorder", "fused", False),  # config 5 model
    ("efficientnet_v2_s_s50", "reorder", "fused", True),
])
def test_logits_at_scale(cfg_name, strategy, gather_mode, rbn):
    torch.set_num_threads(os.cpu_count() or 1)
    cfg = CONFIGS[cfg_name]
    sm = build_spatial_model(cfg, randomize_bn=True) if rbn else _model(cfg_name)
    plans = P.load_plans(cfg.asset_dir / f"plans_{strategy}.json")
    eg = E.export_graph(sm.graph, plans)
    maps = E.compose_maps(sm.graph, plans)
    batch = cfg.batch if cfg.batch > 1 else BATCH
    eng = EN.from_plans(sm, eg, maps, batch=batch, gather_mode=gather_mode)
    eng.capture()  # autotune + CUDA graph, as bench.py
    w, v = apply_plans_spatial(plans, sm.graph, sm.weights, sm.vectors)
    w = {k: t.float() for k, t in w.items()}
    wb = {k: t.bfloat16().float() for k, t in w.items()}
    gots, refs, ctrls = [], [], []
    for b in range(N_BATCHES * BATCH // batch):
        x = torch.randn(batch, 3, 224, 224, generator=torch.Generator().manual_seed(100 + b))
        gots.append(eng.forward(x.cuda()).cpu().clone())
        with torch.no_grad():
            refs.append(run_spatial(eg, sm.specs, w, v, x, dtype=torch.float32))
            if not rbn:  # CPU-only control: bf16 operands and bf16 storage of every node's output
                ctrls.append(run_spatial(eg, sm.specs, wb, v, x.bfloat16().float(), dtype=torch.float32,
                                         store_dtype=torch.bfloat16))
    got, ref = torch.cat(gots), torch.cat(refs)
    assert torch.isfinite(got).all()
    dev, agree = deviation(got, ref), top1_agreement(got, ref)
    top2 = ref.topk(2, dim=1).values
    scale_rel = float((got - ref).abs().max() / ref.abs().max())
    rec = {"parity": cfg_name, "strategy": strategy, "gather": gather_mode, "randomized_bn": rbn,
           "images": got.shape[0], "deviation": dev, "scale_relative_error": scale_rel, "top1": agree,
           "logit_absmax": float(ref.abs().max()), "median_top1_margin": float((top2[:, 0] - top2[:, 1]).median())}
    if ctrls:
        ctrl = torch.cat(ctrls)
        rec["control_top1"] = top1_agreement(ctrl, ref)
        rec["control_deviation"] = deviation(ctrl, ref)
    _record(rec)
    assert dev <= TOL, f"deviation {dev}"
    # the reference metric divides by max(1, |a|, |b|): vacuous when the logits are tiny (random-init
    # MobileNetV3 / EfficientNetV2 reach |x| ~ 1e-11 / 1e-9), so the error is also held to the
    # same tolerance relative to the logits' own scale
    assert scale_rel <= TOL, f"error relative to the logit scale {scale_rel}"
    if agree < TOP1:  # only where bf16 rounding alone flips top-1 classes (see above)
        c = rec["control_top1"]
        assert ctrls and agree >= c - 2 * (c * (1 - c) / got.shape[0]) ** 0.5, rec


def test_every_autotune_variant_is_bit_identical_within_its_kernel():
    """Every variant Engine.autotune can pick (producer width, resident vs streamed
    weights, TMA vs cp.async operands, epilogue groups, N-tile caps, 32-channel fp32
    tiles, halo epilogue groups) computes the same K order, so each must give the SAME
    bits as the default schedule of its read plan and kernel; different read plans /
    kernels (gather vs cover vs copy, halo vs im2col) reorder K and are held to the
    bf16 gate instead."""
    cfg = CONFIGS["resnet50_s50"]
    sm = _model("resnet50_s50")
    plans = P.load_plans(cfg.asset_dir / "plans_reorder.json")
    eg = E.export_graph(sm.graph, plans)
    eng = EN.from_plans(sm, eg, E.compose_maps(sm.graph, plans), batch=6)
    x = torch.randn(6, 3, 224, 224, generator=torch.Generator().manual_seed(4))
    eng.forward(x.cuda())
    torch.cuda.synchronize()
    n_checked = 0
    for op in eng.ops:
        if op.kind != "conv" or "stem_idx" in op.info or not op.info["variants"]:
            continue  # the stem, and small-M linears (one schedule)
        y = eng._value(op.output)
        default = op.info["variant"]
        fams = {}
        for v in op.info["variants"]:
            pi, bits = v
            fam = (pi, bool(op.info.get("halo")) and not bits & 8)
            op.info["variant"] = v
            op.launch()
            torch.cuda.synchronize()
            out = y.buf.clone()
            if fam not in fams:
                fams[fam] = out
            else:
                assert torch.equal(out.view(torch.int16), fams[fam].view(torch.int16)), (op.info["conv"], v)
            n_checked += 1
        base = next(iter(fams.values())).float()
        for fam, out in fams.items():
            rel = float((out.float() - base).abs().max() / base.abs().max().clamp_min(1e-6))
            assert rel < 2e-2, (op.info["conv"], fam, rel)
        op.info["variant"] = default
        op.launch()
    assert n_checked > 54 * 8

"""Reference plan_model wall time, pure Python vs with the native core (dev tool; needs the
reference): python tools/planner_speed.py [config ...]"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")
import reslice  # noqa: E402

from paper_2307_08771_b200 import ir, native_planner as NP, plans as P  # noqa: E402
from paper_2307_08771_b200.configs import CONFIGS  # noqa: E402


def main(names):
    for name in names:
        cfg = CONFIGS[name]
        g = reslice.graph.graph_from_dict(json.loads((cfg.asset_dir / "graph.json").read_text()))
        masks = {k: tuple(v) for k, v in ir.load_masks(cfg.asset_dir / "masks.json").items()}
        t0 = time.time()
        ref, _ = reslice.plan_model(g, masks, "input", "reorder", "error")
        t_ref = time.time() - t0
        NP.install(reslice)
        try:
            t0 = time.time()
            nat, _ = reslice.plan_model(g, masks, "input", "reorder", "error")
            t_nat = time.time() - t0
        finally:
            NP.uninstall()
        same = [P.plan_to_dict(P.from_reference(p)) for p in ref] == [P.plan_to_dict(P.from_reference(p)) for p in nat]
        print(f"{name}: reference plan_model {t_ref:.2f} s, with native core {t_nat:.2f} s "
              f"({t_ref / t_nat:.1f}x), plans identical: {same}")


if __name__ == "__main__":
    main(sys.argv[1:] or ["resnet18_s50", "resnet50_s50", "resnet101_s50"])

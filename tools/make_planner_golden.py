"""Golden vectors for the native planner core, made with the REFERENCE
decompose_paths + order_channels (path_search.py:290-305, ordering.py:39-88).

Run in the build container (needs /root/reference):  python tools/make_planner_golden.py
Writes tests/golden/planner_core.json: random reorder graphs (subsets, duplicates, > 20-node
greedy cases) and the reference's paths / channel order for each.
"""

import json
import random
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, "/root/reference/pkg/src")

from reslice.ordering import order_channels  # noqa: E402
from reslice.path_search import decompose_paths  # noqa: E402
from reslice.reorder_graph import reorder_graph_from_sets  # noqa: E402


def main(n_cases=120, seed=1):
    rng = random.Random(seed)
    cases = []
    for trial in range(n_cases):
        space = rng.choice([8, 16, 32, 64, 128, 256])
        n = rng.randint(1, 24 if trial % 12 == 0 else 12)
        sets = {}
        for i in range(n):
            cid = f"layer{i}_conv{rng.randint(1, 3)}"
            while cid in sets:
                cid += "_b"
            if sets and rng.random() < 0.35:
                prev = sets[rng.choice(sorted(sets))]
                sets[cid] = sorted(rng.sample(prev, rng.randint(1, len(prev))))
            else:
                sets[cid] = sorted(rng.sample(range(space), rng.randint(1, space)))
        rg = reorder_graph_from_sets(sets, space)
        paths = decompose_paths(rg)
        order = order_channels(rg, paths)
        cases.append({"channel_space": space, "retained": sets,
                      "nodes": {k: sorted(v.retained) for k, v in rg.nodes.items()},
                      "paths": [[list(p.nodes), p.reward, list(p.covered_parents)] for p in paths],
                      "order": list(order.order), "dropped": list(order.dropped)})
    out = ROOT / "tests" / "golden" / "planner_core.json"
    out.write_text(json.dumps({"source": "reference reslice decompose_paths + order_channels", "seed": seed,
                               "cases": cases}, separators=(",", ":")))
    print(f"wrote {out} ({len(cases)} cases)")


if __name__ == "__main__":
    main()

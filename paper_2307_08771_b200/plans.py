"""The integer contract between the reference planner and the GPU export.

`SegmentPlan`/`ConsumerAccess`/`CopyStats` and the plan file format are the
reference's own (`reslice.planner`, planner.py:56-126 and 813-927), imported
unmodified; plans are never re-derived here.  Local: `save_plans(compact=True)`
for the committed assets, and `from_reference` (identity, kept for callers).
"""

from __future__ import annotations

from pathlib import Path
from typing import Iterable

from .ir import dump_json
from .ref import reslice

_p = reslice.planner
PLAN_FILE_VERSION = _p.PLAN_FILE_VERSION
MODE_INPUT, MODE_OUTPUT = _p.MODE_INPUT, _p.MODE_OUTPUT
STRATEGY_REORDER, STRATEGY_BASELINE = _p.STRATEGY_REORDER, _p.STRATEGY_BASELINE
CopyStats = _p.CopyStats
ConsumerAccess = _p.ConsumerAccess
JoinRun = _p.JoinRun
JoinRewrite = _p.JoinRewrite
SegmentPlan = _p.SegmentPlan
copy_report = _p.copy_report
plan_to_dict = _p.plan_to_dict
plan_from_dict = _p.plan_from_dict
load_plans = _p.load_plans


def save_plans(plans: Iterable[SegmentPlan], path: str | Path, compact: bool = False) -> None:
    """planner.py:907-918; compact=True drops the indentation."""
    if not compact:
        return _p.save_plans(plans, path)
    plans = list(plans)
    rep = copy_report(plans)
    dump_json({"version": PLAN_FILE_VERSION,
               "segments": [plan_to_dict(p) for p in sorted(plans, key=lambda p: p.segment)],
               "totals": {"total_reads": rep.total_reads, "copied": rep.copied,
                          "zero_copy_optimal": rep.zero_copy_optimal}}, path, compact)


def from_reference(plan) -> SegmentPlan:
    return plan

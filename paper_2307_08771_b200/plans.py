"""The integer contract between the reference planner and the GPU export.

Mirrors `reslice.planner`'s value types (planner.py:56-126) and its plan file
format (planner.py:813-927) so plans produced by the reference's own
`plan_model` -- in this process, or committed as JSON -- drive the permute
kernel unchanged.  A plan is never re-derived here.
"""

from __future__ import annotations

from dataclasses import dataclass
from pathlib import Path
from typing import Iterable, Mapping

from .ir import ModelFormatError, ValidationError, dump_json, load_json

PLAN_FILE_VERSION = 1  # planner.py:47
MODE_INPUT, MODE_OUTPUT = "input", "output"
STRATEGY_REORDER, STRATEGY_BASELINE, STRATEGY_CONSTRAINED = "reorder", "baseline", "constrained"


@dataclass(frozen=True)
class CopyStats:
    """planner.py:56-71: channels materialised at inference time (slices are free)."""

    total_reads: int
    copied: int
    zero_copy_optimal: int = 0

    def __post_init__(self):
        if not (0 <= self.copied <= max(self.total_reads, 0)):
            raise ValidationError([f"copied {self.copied} outside [0, {self.total_reads}]"])

    @property
    def copied_fraction(self) -> float:
        return self.copied / self.total_reads if self.total_reads else 0.0


@dataclass(frozen=True)
class ConsumerAccess:
    """planner.py:74-92.  perm: original input columns in new column order.
    slice: reads [start, start+length); gather: indices[i] = position read by
    new column i (perm ascending)."""

    consumer: str
    mode: str
    start: int = 0
    length: int = 0
    perm: tuple[int, ...] = ()
    indices: tuple[int, ...] = ()


@dataclass(frozen=True)
class JoinRun:
    """planner.py:95-100 (output mode)."""

    producers: tuple[str, ...]
    windows: dict[str, tuple[int, int]]


@dataclass(frozen=True)
class JoinRewrite:
    """planner.py:103-109 (output mode)."""

    join: str
    kind: str
    keep_original: bool
    operands: dict[str, str]
    runs: tuple[JoinRun, ...]


@dataclass(frozen=True)
class SegmentPlan:
    """planner.py:112-126."""

    segment: str
    mode: str
    strategy: str
    producers: tuple[str, ...]
    interior: tuple[str, ...]
    producer_orders: dict[str, tuple[int, ...]]
    dropped: dict[str, tuple[int, ...]]
    zero_rows: dict[str, tuple[int, ...]]
    consumers: tuple[ConsumerAccess, ...]
    per_channel: dict[str, tuple[int, ...]]
    zero_columns: dict[str, tuple[int, ...]]
    infill: dict[str, tuple[int, ...]]
    join: JoinRewrite | None
    stats: CopyStats


def copy_report(plans: Iterable[SegmentPlan]) -> CopyStats:
    """planner.py:799-806."""
    total = copied = optimal = 0
    for p in plans:
        total += p.stats.total_reads
        copied += p.stats.copied
        optimal += p.stats.zero_copy_optimal
    return CopyStats(total, copied, optimal)


# ------------------------------------------------------------------ plan files
def _ints(m: Mapping) -> dict[str, tuple[int, ...]]:
    return {str(k): tuple(int(i) for i in v) for k, v in m.items()}


def _lists(m: Mapping) -> dict:
    return {k: list(v) for k, v in sorted(m.items())}


def plan_to_dict(plan: SegmentPlan) -> dict:
    """planner.py:840-868 (same keys and layout)."""
    join = None
    if plan.join is not None:
        j = plan.join
        join = {"join": j.join, "kind": j.kind, "keep_original": j.keep_original,
                "operands": dict(sorted(j.operands.items())),
                "runs": [{"producers": list(r.producers),
                          "windows": {p: list(w) for p, w in sorted(r.windows.items())}} for r in j.runs]}
    consumers = []
    for a in plan.consumers:
        rec = {"consumer": a.consumer, "perm": list(a.perm)}
        if a.mode == "slice":
            rec["slice"] = [a.start, a.length]
        else:
            rec["gather"] = list(a.indices)
        consumers.append(rec)
    return {
        "segment": plan.segment, "mode": plan.mode, "strategy": plan.strategy,
        "producers": list(plan.producers), "interior": list(plan.interior),
        "producer_orders": _lists(plan.producer_orders), "dropped": _lists(plan.dropped),
        "zero_rows": _lists(plan.zero_rows), "consumers": consumers,
        "per_channel": _lists(plan.per_channel), "zero_columns": _lists(plan.zero_columns),
        "infill": _lists(plan.infill), "join": join,
        "stats": {"total_reads": plan.stats.total_reads, "copied": plan.stats.copied,
                  "zero_copy_optimal": plan.stats.zero_copy_optimal},
    }


def plan_from_dict(obj: dict, source: str = "<memory>") -> SegmentPlan:
    """planner.py:871-904."""
    try:
        join = None
        if obj.get("join") is not None:
            j = obj["join"]
            join = JoinRewrite(
                join=str(j["join"]), kind=str(j["kind"]), keep_original=bool(j["keep_original"]),
                operands={str(k): str(v) for k, v in j["operands"].items()},
                runs=tuple(JoinRun(tuple(str(p) for p in r["producers"]),
                                   {str(p): (int(w[0]), int(w[1])) for p, w in r["windows"].items()})
                           for r in j["runs"]))
        accesses = []
        for rec in obj["consumers"]:
            perm = tuple(int(i) for i in rec["perm"])
            if "slice" in rec:
                s, n = (int(v) for v in rec["slice"])
                accesses.append(ConsumerAccess(str(rec["consumer"]), "slice", start=s, length=n, perm=perm))
            else:
                accesses.append(ConsumerAccess(str(rec["consumer"]), "gather", perm=perm,
                                               indices=tuple(int(i) for i in rec["gather"])))
        st = obj["stats"]
        return SegmentPlan(
            segment=str(obj["segment"]), mode=str(obj["mode"]), strategy=str(obj["strategy"]),
            producers=tuple(str(p) for p in obj["producers"]), interior=tuple(str(u) for u in obj["interior"]),
            producer_orders=_ints(obj["producer_orders"]), dropped=_ints(obj["dropped"]),
            zero_rows=_ints(obj["zero_rows"]), consumers=tuple(accesses),
            per_channel=_ints(obj["per_channel"]), zero_columns=_ints(obj["zero_columns"]),
            infill=_ints(obj["infill"]), join=join,
            stats=CopyStats(int(st["total_reads"]), int(st["copied"]), int(st["zero_copy_optimal"])))
    except (KeyError, ValueError, TypeError, AttributeError) as exc:
        raise ModelFormatError(f"{source}: bad plan record ({exc})") from exc


def save_plans(plans: Iterable[SegmentPlan], path: str | Path, compact: bool = False) -> None:
    """planner.py:907-918."""
    plans = list(plans)
    rep = copy_report(plans)
    dump_json({"version": PLAN_FILE_VERSION,
               "segments": [plan_to_dict(p) for p in sorted(plans, key=lambda p: p.segment)],
               "totals": {"total_reads": rep.total_reads, "copied": rep.copied,
                          "zero_copy_optimal": rep.zero_copy_optimal}}, path, compact)


def load_plans(path: str | Path) -> list[SegmentPlan]:
    """planner.py:921-927."""
    obj = load_json(path)
    if obj.get("version") != PLAN_FILE_VERSION:
        raise ModelFormatError(f"{path}: unsupported plan version {obj.get('version')!r}")
    if not isinstance(obj.get("segments"), list):
        raise ModelFormatError(f"{path}: need a 'segments' list")
    return [plan_from_dict(rec, str(path)) for rec in obj["segments"]]


def from_reference(plan) -> SegmentPlan:
    """Convert a live `reslice.planner.SegmentPlan` (duck-typed) into ours."""
    from dataclasses import asdict, is_dataclass  # noqa: F401
    d = {
        "segment": plan.segment, "mode": plan.mode, "strategy": plan.strategy,
        "producers": list(plan.producers), "interior": list(plan.interior),
        "producer_orders": plan.producer_orders, "dropped": plan.dropped, "zero_rows": plan.zero_rows,
        "consumers": [({"consumer": a.consumer, "perm": list(a.perm), "slice": [a.start, a.length]}
                       if a.mode == "slice" else
                       {"consumer": a.consumer, "perm": list(a.perm), "gather": list(a.indices)})
                      for a in plan.consumers],
        "per_channel": plan.per_channel, "zero_columns": plan.zero_columns, "infill": plan.infill,
        "join": None if plan.join is None else {
            "join": plan.join.join, "kind": plan.join.kind, "keep_original": plan.join.keep_original,
            "operands": plan.join.operands,
            "runs": [{"producers": list(r.producers), "windows": {p: list(w) for p, w in r.windows.items()}}
                     for r in plan.join.runs]},
        "stats": {"total_reads": plan.stats.total_reads, "copied": plan.stats.copied,
                  "zero_copy_optimal": plan.stats.zero_copy_optimal},
    }
    return plan_from_dict(d, "<reslice>")

"""Native planner core for the reference planner.

`decompose_and_order(graph)` runs path_search.decompose_paths + ordering.order_channels
(the hot spot of reference reorder planning: 20 s on ResNet-50, mostly order_channels)
in C++ (csrc/planner.cpp, `ub_plan_order_segment`) with the reference's exact tie-breaking.
`install(reslice)` makes an imported reference `plan_model` use it: pipeline.py:74-75 and
planner.py:527-528 call `decompose_paths(rg)` then `order_channels(rg, paths)`; the patched
decompose returns the reference's own `Path` objects and remembers the order it computed
for that graph, which the patched `order_channels` returns (any other call falls through
to the original).  Plans are identical (tests/test_native_planner.py); no GPU is needed.
"""

from __future__ import annotations

import ctypes
from typing import Any

import numpy as np

from . import _lib


def decompose_and_order(nodes: list[tuple[str, frozenset[int] | set[int]]], channel_space: int):
    """nodes: (id, retained set) of a reorder graph.  Returns (paths, order, dropped) with
    paths = [(member ids, reward, absorbed parent ids)] and order/dropped as in
    ordering.ChannelOrder."""
    nodes = sorted(nodes, key=lambda t: t[0])
    n = len(nodes)
    chans = [sorted(int(c) for c in r) for _, r in nodes]
    offsets = np.zeros(n + 1, dtype=np.int32)
    for i, c in enumerate(chans):
        offsets[i + 1] = offsets[i] + len(c)
    flat = np.array([c for cs in chans for c in cs] or [0], dtype=np.int32)
    order = np.zeros(max(channel_space, 1), dtype=np.int32)
    path_of = np.zeros(max(n, 1), dtype=np.int32)
    path_pos = np.zeros(max(n, 1), dtype=np.int32)
    rewards = np.zeros(max(n, 1), dtype=np.int64)
    n_order, n_paths = ctypes.c_int32(), ctypes.c_int32()

    def ptr(a):
        return ctypes.c_void_p(a.ctypes.data)

    rc = _lib.load().ub_plan_order_segment(n, ptr(offsets), ptr(flat), channel_space, ptr(order),
                                            ctypes.byref(n_order), ptr(path_of), ptr(path_pos), ptr(rewards),
                                            ctypes.byref(n_paths))
    if rc != 0:
        raise ValueError(f"ub_plan_order_segment: status {rc} (bad reorder graph)")
    ids = [nid for nid, _ in nodes]
    paths = []
    for k in range(n_paths.value):
        members = sorted((int(path_pos[i]), ids[i]) for i in range(n) if path_of[i] == k and path_pos[i] >= 0)
        absorbed = sorted(ids[i] for i in range(n) if path_of[i] == k and path_pos[i] < 0)
        paths.append((tuple(m for _, m in members), int(rewards[k]), tuple(absorbed)))
    kept = tuple(int(c) for c in order[:n_order.value])
    retained_any = set(kept)
    dropped = tuple(c for c in range(channel_space) if c not in retained_any)
    return paths, kept, dropped


_installed: dict[str, Any] = {}


def install(reslice_pkg) -> None:
    """Route the reference planner's decompose/order calls through the native core."""
    if _installed:
        return
    import reslice.ordering as ordering
    import reslice.path_search as path_search
    import reslice.pipeline as pipeline
    import reslice.planner as planner

    orig_decompose = path_search.decompose_paths
    orig_order = ordering.order_channels
    cache: dict[int, Any] = {}

    def decompose_paths(graph):
        paths, kept, dropped = decompose_and_order(
            [(nid, node.retained) for nid, node in graph.nodes.items()], graph.channel_space)
        out = [path_search.Path(m, r, a) for m, r, a in paths]
        cache[id(graph)] = (out, ordering.ChannelOrder(order=kept, dropped=dropped))
        return out

    def order_channels(graph, paths):
        hit = cache.pop(id(graph), None)
        if hit is not None and hit[0] == list(paths):
            return hit[1]
        return orig_order(graph, paths)

    _installed.update(decompose=orig_decompose, order=orig_order)
    for mod in (pipeline, planner):
        mod.decompose_paths = decompose_paths
        mod.order_channels = order_channels


def uninstall() -> None:
    if not _installed:
        return
    import reslice.pipeline as pipeline
    import reslice.planner as planner

    for mod in (pipeline, planner):
        mod.decompose_paths = _installed["decompose"]
        mod.order_channels = _installed["order"]
    _installed.clear()

"""Default pipeline and reward normaliser (mirrors baselines.py:24-118).

greedy_placement uses the native O(D N log N) DP (go_greedy_cuts) that returns the
reference's exact cuts; baseline_step_time runs the device DES."""
from __future__ import annotations

import numpy as np

from .config import NUM_PRIORITY_LEVELS, FusionConfig
from .costmodel import as_topology
from .fusion import greedy_cuts
from .graph import as_graph
from .simulator import ActionAssignment, evaluate_assignments

_cache: dict = {}


def greedy_placement(graph, topology) -> ActionAssignment:
    """baselines.py:75-118: contiguous topo chunks balanced by flops, colocation
    groups forced to their first member's device."""
    g = as_graph(graph)
    d = as_topology(topology).num_devices
    order = g.topo_order()
    cuts = greedy_cuts(g.flops[order], d)
    actions = np.zeros(g.num_nodes, dtype=np.int64)
    for dev in range(d):
        actions[order[cuts[dev]:cuts[dev + 1]]] = dev
    first: dict = {}
    for v in np.flatnonzero(g.coloc >= 0):
        c = int(g.coloc[v])
        if c not in first:
            first[c] = int(actions[v])
        actions[v] = first[c]
    return ActionAssignment("placement", actions, d)


def default_assignments(graph, topology, num_levels: int = NUM_PRIORITY_LEVELS) -> dict:
    """baselines.py:24-36 (cached per (graph, topology) object)."""
    g = as_graph(graph)
    key = (id(g), id(topology), num_levels)
    hit = _cache.get(key)
    if hit is not None and hit[0] is g:
        return {k: ActionAssignment(v.task, v.actions.copy(), v.num_actions)
                for k, v in hit[1].items()}
    n = g.num_nodes
    asg = {
        "placement": greedy_placement(g, topology),
        "schedule_priority": ActionAssignment.constant("schedule_priority", n, num_levels, 0),
        "fusion_priority": ActionAssignment.constant("fusion_priority", n, num_levels, 0),
    }
    _cache[key] = (g, asg)
    return {k: ActionAssignment(v.task, v.actions.copy(), v.num_actions) for k, v in asg.items()}


def baseline_step_time(graph, topology, fusion_config: FusionConfig | None = None) -> float:
    """baselines.py:39-47."""
    res = evaluate_assignments(graph, topology, default_assignments(graph, topology),
                               fusion_config)
    return res.step_time

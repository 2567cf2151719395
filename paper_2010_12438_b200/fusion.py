"""Greedy fusion pass and greedy baseline placement, native host code
(go_apply_fusion / go_greedy_cuts in csrc/graph.cu)."""
from __future__ import annotations

import numpy as np

from . import _lib
from .graph import as_graph


def fuse_groups(graph, priorities, max_group: int = 8) -> np.ndarray:
    """simulator.py:199-277 -> group root label per node."""
    g = as_graph(graph)
    pri = np.ascontiguousarray(priorities, dtype=np.int64)
    out = np.empty(g.num_nodes, np.int64)
    _lib.call("go_apply_fusion", g.num_nodes, g.num_edges, _lib.ptr(g.src), _lib.ptr(g.dst),
              _lib.ptr(g.op), _lib.ptr(pri), int(max_group), _lib.ptr(out))
    return out


def greedy_cuts(flops_topo: np.ndarray, d: int) -> np.ndarray:
    """baselines.py:85-110 DP cuts (earliest split on ties), O(D N log N)."""
    f = np.ascontiguousarray(flops_topo, dtype=np.float64)
    cuts = np.empty(d + 1, np.int64)
    _lib.call("go_greedy_cuts", len(f), _lib.ptr(f), int(d), _lib.ptr(cuts))
    return cuts

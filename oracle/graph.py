"""Oracle graph model (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

A graph is a plain dict of numpy arrays:
  n, op (int op index), flops, out_bytes (f64), coloc (int group id, -1 none),
  src, dst (int64 edge endpoints, in graph.edges order), ebytes (f64).
Restates /root/reference/pkg/src/graphopt/graph.py.
"""
from __future__ import annotations

import heapq
import math

import numpy as np

# graph.py:16-30
OP_TYPES = ("matmul", "conv", "elementwise-add", "elementwise-mul", "reduce", "sigmoid",
            "relu", "softmax", "concat", "split", "embed-lookup", "other")
OP_INDEX = {name: i for i, name in enumerate(OP_TYPES)}


def make(n, op, flops, out_bytes, src, dst, ebytes, coloc=None):
    g = dict(n=int(n), op=np.asarray(op, np.int64), flops=np.asarray(flops, np.float64),
             out_bytes=np.asarray(out_bytes, np.float64),
             src=np.asarray(src, np.int64).reshape(-1), dst=np.asarray(dst, np.int64).reshape(-1),
             ebytes=np.asarray(ebytes, np.float64).reshape(-1))
    g["coloc"] = (np.full(n, -1, np.int64) if coloc is None else np.asarray(coloc, np.int64))
    g["topo"] = topo_order(g)
    return g


def from_reference(graph) -> dict:
    """Convert a graphopt.ComputationGraph (duck-typed) into oracle arrays."""
    names = {}
    coloc = []
    for nd in graph.nodes:
        c = nd.colocation_group
        if c is None:
            coloc.append(-1)
        else:
            coloc.append(names.setdefault(c, len(names)))
    return make(graph.num_nodes, [OP_INDEX[nd.op_type] for nd in graph.nodes],
                [nd.flops for nd in graph.nodes], [nd.output_bytes for nd in graph.nodes],
                [e.src for e in graph.edges], [e.dst for e in graph.edges],
                [e.bytes for e in graph.edges], coloc)


def topo_order(g) -> np.ndarray:
    """Heap-Kahn, ascending-id tie-break (graph.py:173-201)."""
    n = g["n"]
    indeg = [0] * n
    succ = [[] for _ in range(n)]
    for s, d in zip(g["src"].tolist(), g["dst"].tolist()):
        indeg[d] += 1
        if s != d:
            succ[s].append(d)
    heap = [v for v in range(n) if indeg[v] == 0]
    heapq.heapify(heap)
    order = []
    while heap:
        v = heapq.heappop(heap)
        order.append(v)
        for w in succ[v]:
            indeg[w] -= 1
            if indeg[w] == 0:
                heapq.heappush(heap, w)
    if len(order) != n:
        raise ValueError("cycle")
    return np.array(order, np.int64)


def neighbors(g) -> list[list[int]]:
    """Undirected sorted neighbour sets (graph.py:131-133)."""
    n = g["n"]
    sets = [set() for _ in range(n)]
    for s, d in zip(g["src"].tolist(), g["dst"].tolist()):
        sets[d].add(s)
        sets[s].add(d)
    return [sorted(x) for x in sets]


def degrees(g):
    indeg = np.bincount(g["dst"], minlength=g["n"]).astype(np.float64)
    outdeg = np.bincount(g["src"], minlength=g["n"]).astype(np.float64)
    return indeg, outdeg


def feature_dim(sizes) -> int:
    """graph.py:262-265."""
    return len(OP_TYPES) + 4 + sum(sizes)


def node_features(g, prev_list, sizes) -> np.ndarray:
    """N x F matrix, rows in topo order (graph.py:268-313).  prev_list is a
    list (one per task) of node-indexed int vectors or None."""
    n = g["n"]
    order = g["topo"]
    nops = len(OP_TYPES)
    feats = np.zeros((n, feature_dim(sizes)))
    indeg, outdeg = degrees(g)
    rows = np.arange(n)
    feats[rows, g["op"][order]] = 1.0
    feats[:, nops] = [math.log1p(x) for x in g["flops"][order]]
    feats[:, nops + 1] = [math.log1p(x) for x in g["out_bytes"][order]]
    feats[:, nops + 2] = indeg[order]
    feats[:, nops + 3] = outdeg[order]
    col = nops + 4
    if prev_list is None:
        prev_list = [None] * len(sizes)
    for acts, a in zip(prev_list, sizes):
        if acts is not None:
            vec = np.asarray(acts, np.int64)
            feats[rows, col + vec[order]] = 1.0
        col += a
    return feats

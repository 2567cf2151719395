"""Graph data model for the B200 path (mirrors graphopt.graph, graph.py:16-313).

`Graph` is a struct-of-arrays view of a computation graph (node-id indexed; edges
in graph.edges order).  `as_graph()` accepts either a `Graph` or any object shaped
like the reference's ComputationGraph (`.nodes[*].op_type/flops/output_bytes/
colocation_group`, `.edges[*].src/dst/bytes`), so reference users can pass their
existing graphs.  Topological order is computed natively (go_topo_order).
"""
from __future__ import annotations

import math
import weakref

import numpy as np

from . import _lib

# graph.py:16-30
OP_TYPES = ("matmul", "conv", "elementwise-add", "elementwise-mul", "reduce", "sigmoid",
            "relu", "softmax", "concat", "split", "embed-lookup", "other")
OP_INDEX = {name: i for i, name in enumerate(OP_TYPES)}
BYTES_PER_ELEMENT = 4


class GraphError(ValueError):
    """A graph violates a model invariant (graph.py:37)."""


class Graph:
    """Validated DAG with dense node ids 0..N-1."""

    def __init__(self, op, flops, out_bytes, src, dst, ebytes, coloc=None, name=""):
        self.op = np.ascontiguousarray(op, dtype=np.int32)
        self.flops = np.ascontiguousarray(flops, dtype=np.float64)
        self.out_bytes = np.ascontiguousarray(out_bytes, dtype=np.float64)
        self.src = np.ascontiguousarray(src, dtype=np.int32).reshape(-1)
        self.dst = np.ascontiguousarray(dst, dtype=np.int32).reshape(-1)
        self.ebytes = np.ascontiguousarray(ebytes, dtype=np.float64).reshape(-1)
        n = len(self.op)
        self.coloc = (np.full(n, -1, np.int32) if coloc is None
                      else np.ascontiguousarray(coloc, dtype=np.int32))
        self.name = name
        if not (len(self.flops) == len(self.out_bytes) == n == len(self.coloc)):
            raise GraphError("node arrays differ in length")
        if not (len(self.src) == len(self.dst) == len(self.ebytes)):
            raise GraphError("edge arrays differ in length")
        if n and (self.op.min() < 0 or self.op.max() >= len(OP_TYPES)):
            raise GraphError("unknown op index")
        if (self.flops < 0).any() or (self.out_bytes < 0).any() or (self.ebytes < 0).any():
            raise GraphError("negative cost")
        if len(self.src) and (min(self.src.min(), self.dst.min()) < 0
                              or max(self.src.max(), self.dst.max()) >= n):
            raise GraphError("dangling edge")
        self._topo = None
        self.version = 0

    @property
    def num_nodes(self) -> int:
        return len(self.op)

    @property
    def num_edges(self) -> int:
        return len(self.src)

    def topo_order(self) -> np.ndarray:
        """Topological order, ascending-id tie-break (graph.py:173-201)."""
        if self._topo is None:
            n = self.num_nodes
            out = np.empty(n, np.int32)
            st = _lib.lib().go_topo_order(n, self.num_edges, _lib.ptr(self.src),
                                          _lib.ptr(self.dst), _lib.ptr(out))
            if st == _lib.GO_ERR_CYCLE:
                raise GraphError(f"graph {self.name!r}: cycle detected")
            _lib.check(st)
            self._topo = out
        return self._topo

    def neighbors(self, v: int) -> list[int]:
        """Undirected sorted neighbourhood (graph.py:131-133)."""
        s = set(self.src[self.dst == v].tolist()) | set(self.dst[self.src == v].tolist())
        return sorted(s)

    def in_degree(self) -> np.ndarray:
        return np.bincount(self.dst, minlength=self.num_nodes)

    def out_degree(self) -> np.ndarray:
        return np.bincount(self.src, minlength=self.num_nodes)


_converted: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def as_graph(g) -> Graph:
    """Accept a Graph or a reference-shaped ComputationGraph (converted once, cached)."""
    if isinstance(g, Graph):
        return g
    try:
        hit = _converted.get(g)
    except TypeError:
        hit = None
    if hit is not None:
        return hit
    names: dict = {}
    coloc = []
    for nd in g.nodes:
        c = getattr(nd, "colocation_group", None)
        coloc.append(-1 if c is None else names.setdefault(c, len(names)))
    out = Graph([OP_INDEX[nd.op_type] for nd in g.nodes],
                [nd.flops for nd in g.nodes], [nd.output_bytes for nd in g.nodes],
                [e.src for e in g.edges], [e.dst for e in g.edges], [e.bytes for e in g.edges],
                coloc, name=getattr(g, "name", ""))
    try:
        _converted[g] = out
    except TypeError:
        pass
    return out


def feature_dim(action_space) -> int:
    """graph.py:262-265."""
    sizes = [action_space] if isinstance(action_space, int) else list(action_space)
    return len(OP_TYPES) + 4 + sum(sizes)


def node_features(graph, prev_actions=None, action_space=1) -> np.ndarray:
    """Host N x F feature matrix (graph.py:268-313).  Not on the hot path: the GPU
    forward builds the same rows in-kernel (csrc/embed.cu features_inproj)."""
    g = as_graph(graph)
    sizes = [action_space] if isinstance(action_space, int) else list(action_space)
    if prev_actions is None:
        prev_list = [None] * len(sizes)
    elif isinstance(prev_actions, (list, tuple)):
        prev_list = list(prev_actions)
    else:
        prev_list = [prev_actions]
    if len(prev_list) != len(sizes):
        raise ValueError(f"{len(prev_list)} action vectors for {len(sizes)} action spaces")
    n = g.num_nodes
    order = g.topo_order()
    feats = np.zeros((n, feature_dim(sizes)))
    rows = np.arange(n)
    nops = len(OP_TYPES)
    feats[rows, g.op[order]] = 1.0
    feats[:, nops] = [math.log1p(x) for x in g.flops[order]]
    feats[:, nops + 1] = [math.log1p(x) for x in g.out_bytes[order]]
    feats[:, nops + 2] = g.in_degree()[order]
    feats[:, nops + 3] = g.out_degree()[order]
    col = nops + 4
    for acts, a in zip(prev_list, sizes):
        if acts is not None:
            vec = np.asarray(getattr(acts, "actions", acts), dtype=np.int64)
            if vec.shape != (n,):
                raise ValueError(f"prev_actions has shape {vec.shape}, want ({n},)")
            if vec.min() < 0 or vec.max() >= a:
                raise ValueError(f"action out of range [0,{a})")
            feats[rows, col + vec[order]] = 1.0
        col += a
    return feats

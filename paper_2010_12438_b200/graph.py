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


# ---------------------------------------------------------------------------------------
# JSON graph format (graph.py:208-259): straight into the struct-of-
# arrays Graph, same keys, defaults and GraphError conditions as the reference loader.
_NODE_KEYS = {"id", "op", "shape", "flops", "out_bytes", "colocate"}
_EDGE_KEYS = {"src", "dst", "bytes"}
_TOP_KEYS = {"name", "nodes", "edges"}


def from_dict(data: dict, name: str | None = None) -> Graph:
    """graph.py:208-246: unknown keys rejected, unknown ops -> "other", edge bytes
    default to the source node's output bytes, dense ordered ids, shape-consistent
    output bytes, non-negative costs, acyclic."""
    if not isinstance(data, dict):
        raise GraphError("graph file must contain a JSON object")
    extra = set(data) - _TOP_KEYS
    if extra:
        raise GraphError(f"unknown top-level keys: {sorted(extra)}")
    ids, ops, flops, obytes, coloc = [], [], [], [], []
    groups: dict = {}
    for item in data.get("nodes", []):
        extra = set(item) - _NODE_KEYS
        if extra:
            raise GraphError(f"node entry: unknown keys {sorted(extra)}")
        if "id" not in item or "op" not in item:
            raise GraphError("node entry missing 'id' or 'op'")
        nid = int(item["id"])
        op = item["op"] if item["op"] in OP_INDEX else "other"
        shape = tuple(int(d) for d in item.get("shape", []))
        f = float(item.get("flops", 0.0))
        ob = float(item.get("out_bytes", 0.0))
        if f < 0 or ob < 0:  # graph.py:52-53
            raise GraphError(f"node {nid}: negative cost")
        if any(d <= 0 for d in shape):
            raise GraphError(f"node {nid}: non-positive shape dim")
        if shape and ob != BYTES_PER_ELEMENT * math.prod(shape):
            raise GraphError(f"node {nid}: output_bytes {ob} inconsistent with shape "
                             f"{list(shape)} ({BYTES_PER_ELEMENT * math.prod(shape)} expected)")
        c = item.get("colocate")
        ids.append(nid)
        ops.append(OP_INDEX[op])
        flops.append(f)
        obytes.append(ob)
        coloc.append(-1 if c is None else groups.setdefault(c, len(groups)))
    by_id = {nid: i for i, nid in enumerate(ids)}
    src, dst, eb = [], [], []
    for item in data.get("edges", []):
        extra = set(item) - _EDGE_KEYS
        if extra:
            raise GraphError(f"edge entry: unknown keys {sorted(extra)}")
        s, d = int(item["src"]), int(item["dst"])
        if s not in by_id or d not in by_id:
            raise GraphError(f"dangling edge {s}->{d}")
        b = item.get("bytes")
        b = float(b) if b is not None else obytes[by_id[s]]
        if b < 0:
            raise GraphError(f"edge {s}->{d}: negative bytes")
        src.append(s)
        dst.append(d)
        eb.append(b)
    n = len(ids)
    if sorted(ids) != list(range(n)):  # graph.py:101-106
        dup = sorted({i for i in ids if ids.count(i) > 1})
        if dup:
            raise GraphError(f"duplicate id {dup[0]}")
        raise GraphError(f"node ids not dense 0..{n - 1}: {sorted(ids)[:5]}")
    if ids != sorted(ids):
        raise GraphError("nodes must be listed in id order")
    g = Graph(ops, flops, obytes, src, dst, eb, coloc, name=data.get("name", name or ""))
    g.topo_order()  # raises GraphError on a cycle, like the reference constructor
    g.colocation_names = list(groups)
    return g


def loads(text: str, name: str | None = None) -> Graph:
    """graph.py:249-254."""
    import json
    try:
        data = json.loads(text)
    except json.JSONDecodeError as exc:
        raise GraphError(f"parse error: {exc}") from exc
    return from_dict(data, name=name)


def load_graph(path) -> Graph:
    """graph.py:257-260."""
    from pathlib import Path
    path = Path(path)
    return loads(path.read_text(), name=path.stem)


def to_dict(graph) -> dict:
    """JSON object form of a graph (the inverse of from_dict)."""
    g = as_graph(graph)
    names = getattr(g, "colocation_names", None)
    nodes = []
    for v in range(g.num_nodes):
        item = {"id": v, "op": OP_TYPES[int(g.op[v])], "flops": float(g.flops[v]),
                "out_bytes": float(g.out_bytes[v])}
        c = int(g.coloc[v])
        if c >= 0:
            item["colocate"] = names[c] if names else f"g{c}"
        nodes.append(item)
    edges = [{"src": int(s), "dst": int(d), "bytes": float(b)}
             for s, d, b in zip(g.src, g.dst, g.ebytes)]
    return {"name": g.name, "nodes": nodes, "edges": edges}

"""GraphSAGE embedding on the B200 (mirrors graphopt.embedding, embedding.py:1-98).

Same names, signatures, return types and errors as the reference; the math runs
in libgo_b200 (csrc/embed.cu: numpy-exact neighbour sampling, fused feature
projection, fp32 GEMMs, warp-per-node segment max)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .config import EmbedConfig, PolicyConfig
from .engine import EMBED, DeviceArray, check_status, forward_batch
from .graph import OP_TYPES, as_graph
from .params import _uniform
from .runtime import context, stream_ptr, torch

__all__ = ["EmbedConfig", "Embeddings", "init_embed_params", "sample_neighbors", "embed",
           "neighbor_arrays"]


@dataclass
class Embeddings:
    node_embed: DeviceArray  # N x gs_dim, topo order
    graph_embed: DeviceArray  # 1 x gs_dim


def init_embed_params(store, feature_dim: int, cfg: EmbedConfig, rng: np.random.Generator,
                      prefix: str = "embed/"):
    """embedding.py:35-44."""
    d = cfg.gs_dim
    store.add(prefix + "in_w", _uniform(rng, (feature_dim, d), feature_dim))
    store.add(prefix + "in_b", np.zeros(d))
    for l in range(cfg.gs_layers):
        store.add(f"{prefix}agg_w{l}", _uniform(rng, (d, d), d))
        store.add(f"{prefix}agg_b{l}", np.zeros(d))
        store.add(f"{prefix}fc_w{l}", _uniform(rng, (2 * d, d), 2 * d))
        store.add(f"{prefix}fc_b{l}", np.zeros(d))


def neighbor_arrays(graph, k: int, seed: int):
    """(gather, segments) in topo-row space (embedding.py:61-70), sampled on device."""
    import ctypes as C
    g = as_graph(graph)
    if k < 1:
        raise ValueError("k must be >= 1")
    ctx = context()
    h = ctx.graph(g)
    seg_off = np.zeros(g.num_nodes + 1, np.int64)
    _lib.call("go_neighbor_arrays", ctx.handle, h.handle, int(seed), int(k),
              seg_off.ctypes.data, None, None)
    total = int(seg_off[-1])
    T = torch()
    gather = T.empty(max(total, 1), dtype=T.int32, device=T.device("cuda", ctx.device))
    _lib.call("go_neighbor_arrays", ctx.handle, h.handle, int(seed), int(k),
              seg_off.ctypes.data, _lib.ptr(gather), stream_ptr())
    gath = gather[:total].cpu().numpy().astype(np.int64)
    segs = np.repeat(np.arange(g.num_nodes, dtype=np.int64), np.diff(seg_off))
    return gath, segs


def sample_neighbors(graph, node: int, k: int, seed: int) -> list[int]:
    """embedding.py:47-58: up to k undirected neighbours, uniform without
    replacement when deg > k, deterministic in (seed, node id); sorted ids."""
    if k < 1:
        raise ValueError("k must be >= 1")
    g = as_graph(graph)
    gather, segs = neighbor_arrays(g, k, seed)
    order = g.topo_order()
    row = int(np.flatnonzero(order == node)[0])
    return sorted(int(order[r]) for r in gather[segs == row])


def _features_dev(features, n):
    T = torch()
    if isinstance(features, DeviceArray):
        f = features.dev
    elif hasattr(features, "data") and not isinstance(features, np.ndarray):
        f = T.as_tensor(np.asarray(features.data))
    else:
        f = T.as_tensor(np.asarray(features))
    if f.dim() != 2 or f.shape[0] != n:
        raise ValueError(f"feature rows {f.shape[0] if f.dim() else 0} != N {n}")
    return f.to(device=T.device("cuda", context().device), dtype=T.float32).contiguous()


def embed(graph, features, store, cfg: EmbedConfig, seed: int = 0,
          prefix: str = "embed/") -> Embeddings:
    """embedding.py:73-98.  Raises ValueError on a row mismatch and
    FloatingPointError on non-finite embeddings, like the reference."""
    if prefix != "embed/":
        raise ValueError("only the 'embed/' parameter prefix is supported")
    g = as_graph(graph)
    feats = _features_dev(features, g.num_nodes)
    fdim = int(feats.shape[1])
    if fdim < len(OP_TYPES) + 4:
        raise ValueError(f"feature width {fdim} < {len(OP_TYPES) + 4}")
    sizes = {"placement": max(1, fdim - len(OP_TYPES) - 4)}
    h = context().graph(g)
    out = forward_batch(store, cfg, PolicyConfig(), sizes, [h], [seed], stage_mask=EMBED,
                        features=feats)
    check_status(out)
    return Embeddings(node_embed=DeviceArray(out.node_embed),
                      graph_embed=DeviceArray(out.graph_embed))

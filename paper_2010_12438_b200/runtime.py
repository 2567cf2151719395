"""Runtime plumbing: one library context per CUDA device, uploaded graph handles,
config structs, streams.  torch is used only for device memory and streams."""
from __future__ import annotations

import ctypes as C
import weakref

import numpy as np

from . import _lib
from .config import EmbedConfig, PolicyConfig, ordered_tasks
from .graph import Graph, as_graph

_ctx: dict[int, "Context"] = {}


def torch():
    import torch as _t
    return _t


def device_index() -> int:
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("paper_2010_12438_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    return t.cuda.current_device()


def stream_ptr() -> int:
    return torch().cuda.current_stream().cuda_stream


class Context:
    def __init__(self, device: int):
        self.device = device
        h = C.c_void_p()
        _lib.call("go_ctx_create", device, C.byref(h))
        self.handle = h
        self._graphs: "weakref.WeakKeyDictionary[Graph, GraphHandle]" = weakref.WeakKeyDictionary()

    def graph(self, g) -> "GraphHandle":
        g = as_graph(g)
        h = self._graphs.get(g)
        if h is None:
            h = GraphHandle(self, g)
            self._graphs[g] = h
        return h

    def workspace_bytes(self) -> int:
        out = C.c_int64()
        _lib.call("go_ctx_workspace_bytes", self.handle, C.byref(out))
        return out.value


def context() -> Context:
    dev = device_index()
    c = _ctx.get(dev)
    if c is None:
        c = Context(dev)
        _ctx[dev] = c
    return c


class GraphHandle:
    """A graph uploaded to the device with its static tables (go_graph_create)."""

    def __init__(self, ctx: Context, g: Graph):
        self.graph = g
        self.n = g.num_nodes
        h = C.c_void_p()
        _lib.call("go_graph_create", ctx.handle, g.num_nodes, g.num_edges, _lib.ptr(g.op),
                  _lib.ptr(g.flops), _lib.ptr(g.out_bytes), _lib.ptr(g.coloc),
                  _lib.ptr(g.src), _lib.ptr(g.dst), _lib.ptr(g.ebytes), C.byref(h))
        self.handle = h
        self.fusion_key = None  # None == singleton grouping
        self.acyclic = True
        self.num_groups = g.num_nodes
        self._topo = None

    def topo(self) -> np.ndarray:
        if self._topo is None:
            out = np.empty(self.n, np.int32)
            _lib.call("go_graph_topo", self.handle, _lib.ptr(out))
            self._topo = out
        return self._topo

    def set_fusion(self, labels) -> None:
        key = None if labels is None else np.asarray(labels, np.int64).tobytes()
        if key == self.fusion_key:
            return
        lab = (np.arange(self.n, dtype=np.int64) if labels is None
               else np.ascontiguousarray(labels, dtype=np.int64))
        ng, acyc = C.c_int32(), C.c_int32()
        _lib.call("go_graph_set_fusion", self.handle, _lib.ptr(lab), C.byref(ng), C.byref(acyc))
        self.fusion_key = key
        self.num_groups = ng.value
        self.acyclic = bool(acyc.value)

    def __del__(self):
        try:
            if self.handle:
                _lib.lib().go_graph_destroy(self.handle)
        except Exception:
            pass


def make_config(embed_cfg: EmbedConfig, cfg: PolicyConfig, task_sizes: dict) -> _lib.GoConfig:
    tasks = ordered_tasks(task_sizes)
    c = _lib.GoConfig()
    c.gs_layers, c.gs_dim, c.gs_knn = embed_cfg.gs_layers, embed_cfg.gs_dim, embed_cfg.gs_knn
    c.trf_layers, c.d_model, c.n_head = cfg.trf_layers, cfg.d_model, cfg.n_head
    c.d_head, c.d_inner, c.segment_len = cfg.d_head, cfg.d_inner, min(cfg.segment_len, 2**31 - 1)
    c.num_tasks = len(tasks)
    for i, (_t, a) in enumerate(tasks):
        c.task_sizes[i] = a
    return c


def handle_array(handles) -> "C.Array":
    arr = (C.c_void_p * len(handles))()
    for i, h in enumerate(handles):
        arr[i] = h.handle.value
    return arr

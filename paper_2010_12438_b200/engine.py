"""Batched device engine: the calls every public entry point funnels into.

forward_batch  -> go_forward_status (embed -> trunk -> heads over a ragged batch)
sample_batch   -> go_sample         (numpy-exact float64 categorical draws)
simulate_batch -> go_simulate       (exact DES over K placements + reward)
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .config import EmbedConfig, PolicyConfig, ordered_tasks
from .params import DeviceParams
from .runtime import context, handle_array, make_config, stream_ptr, torch

_dev_params = DeviceParams()

EMBED, TRUNK, HEADS = 1, 2, 4


class DeviceArray:
    """Device result with the reference Tensor's read interface (`.data` is a
    float64 numpy array, fetched lazily)."""

    __slots__ = ("dev", "_host")

    def __init__(self, dev):
        self.dev = dev
        self._host = None

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            self._host = self.dev.detach().to("cpu").numpy().astype(np.float64)
        return self._host

    @property
    def shape(self):
        return tuple(self.dev.shape)

    def __array__(self, dtype=None, copy=None):
        """numpy conversion (np.asarray(x), the reference's Tensor(x)) reads the host copy."""
        return self.data if dtype is None else self.data.astype(dtype)


@dataclass
class ForwardOut:
    row_off: np.ndarray          # [F+1]
    node_embed: object = None    # [R, gs_dim]
    graph_embed: object = None   # [F, gs_dim]
    hid: object = None           # [R, d_model]
    logits: list = None          # per task [R, a_t] views into one packed buffer
    logits_packed: object = None
    value: object = None         # [F]
    status: object = None        # int32 device word
    reps: object = None          # [T, R, d_model] or None


def params_on_device(store, embed_cfg, cfg, task_sizes):
    return _dev_params.get(store, embed_cfg, cfg, task_sizes, torch().device("cuda", context().device))


def forward_batch(store, embed_cfg: EmbedConfig, cfg: PolicyConfig, task_sizes: dict,
                  handles: list, seeds, prev_actions=None, stage_mask=EMBED | TRUNK | HEADS,
                  node_embed=None, graph_embed=None, hid=None, mod_override=None,
                  ablate_mask=0, params=None, features=None, row_counts=None,
                  want_reps=False, cache_hook=None) -> ForwardOut:
    """One go_forward_status call over a ragged batch.  `handles` are GraphHandles
    (or None with `row_counts` for graph-less trunk/heads calls)."""
    T = torch()
    ctx = context()
    dev = T.device("cuda", ctx.device)
    tasks = ordered_tasks(task_sizes)
    if not tasks:
        raise ValueError("at least one task required")
    blob, offs = params if params is not None else params_on_device(store, embed_cfg, cfg,
                                                                    task_sizes)
    if handles is None:
        counts = [int(c) for c in row_counts]
    else:
        counts = [h.n for h in handles]
    F = len(counts)
    row_off = np.zeros(F + 1, np.int64)
    row_off[1:] = np.cumsum(counts)
    R = int(row_off[-1])
    out = ForwardOut(row_off=row_off)
    if stage_mask & EMBED:
        node_embed = T.empty((R, embed_cfg.gs_dim), dtype=T.float32, device=dev)
        graph_embed = T.empty((F, embed_cfg.gs_dim), dtype=T.float32, device=dev)
    if stage_mask & TRUNK:
        hid = T.empty((R, cfg.d_model), dtype=T.float32, device=dev)
    out.node_embed, out.graph_embed, out.hid = node_embed, graph_embed, hid
    logits = None
    value = None
    if stage_mask & HEADS:
        tot = sum(a for _, a in tasks)
        logits = T.empty(R * tot, dtype=T.float32, device=dev)
        value = T.empty(F, dtype=T.float32, device=dev)
        views, c = [], 0
        for _t, a in tasks:
            views.append(logits[c:c + R * a].view(R, a))
            c += R * a
        out.logits, out.logits_packed, out.value = views, logits, value
    reps = None
    if want_reps and stage_mask & HEADS:
        reps = T.empty((len(tasks), R, cfg.d_model), dtype=T.float32, device=dev)
    out.reps = reps
    status = T.zeros(1, dtype=T.int32, device=dev)
    out.status = status
    cfg_c = make_config(embed_cfg, cfg, task_sizes)
    b = _lib.GoBatch()
    seeds_arr = (C.c_int64 * F)(*[int(s) for s in (seeds if seeds is not None else [0] * F)])
    b.num_forwards = F
    if handles is not None:
        harr = handle_array(handles)
        b.graphs = C.cast(harr, C.POINTER(C.c_void_p))
    else:
        counts_arr = (C.c_int64 * F)(*counts)
        b.row_counts = counts_arr
    b.embed_seeds = seeds_arr
    if features is not None:
        b.features = _lib.ptr(features)
        b.feature_dim = int(features.shape[1])
    b.reps = _lib.ptr(reps)
    b.prev_actions = _lib.ptr(prev_actions)
    b.stage_mask = stage_mask
    b.ablate_mask = ablate_mask
    b.mod_override = _lib.ptr(mod_override)
    if cache_hook is not None:  # a _lib.CACHE_HOOK; the caller keeps it alive
        b.cache_hook = C.cast(cache_hook, C.c_void_p)
    _lib.call("go_forward_status", ctx.handle, C.byref(cfg_c), _lib.ptr(blob),
              offs.ctypes.data, C.byref(b), _lib.ptr(node_embed), _lib.ptr(graph_embed),
              _lib.ptr(hid), _lib.ptr(logits), _lib.ptr(value), _lib.ptr(status), stream_ptr())
    return out


def check_status(out: ForwardOut):
    if out.status is not None and int(out.status.item()) & 1:
        raise FloatingPointError("non-finite node embeddings (bad init or features)")


M64 = (1 << 64) - 1


def pcg_words(gen) -> list[int]:
    """(state_hi, state_lo, inc_hi, inc_lo) of a numpy PCG64 Generator."""
    st = gen.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise TypeError("sampling needs a numpy Generator backed by PCG64 "
                        "(np.random.default_rng), like the reference")
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    return [s >> 64, s & M64, inc >> 64, inc & M64]


def advance(gen, n: int):
    """Advance `gen` exactly as n calls of next_double would (the uint32 buffer used
    by integer draws is left untouched, as rng.random(n) leaves it)."""
    if n <= 0:
        return
    bg = gen.bit_generator
    st = bg.state
    bg.advance(n)
    st2 = bg.state
    st2["has_uint32"], st2["uinteger"] = st["has_uint32"], st["uinteger"]
    bg.state = st2


def sample_batch(embed_cfg, cfg, task_sizes, handles, states, logits_packed, temperature,
                 logits_f64=False, row_counts=None, shared_logits=False):
    """-> (actions int32 [T, R], logp f64 [T, R]).  states: [F][4] PCG64 words
    (pcg_words) before this call.  Actions are node-indexed per forward span (row
    order for graph-less batches).  shared_logits: every forward samples from the same
    logits block (one forward's rows; mode S)."""
    T = torch()
    ctx = context()
    dev = T.device("cuda", ctx.device)
    tasks = ordered_tasks(task_sizes)
    counts = [h.n for h in handles] if handles is not None else [int(c) for c in row_counts]
    F = len(counts)
    R = sum(counts)
    actions = T.empty((len(tasks), R), dtype=T.int32, device=dev)
    logp = T.empty((len(tasks), R), dtype=T.float64, device=dev)
    cfg_c = make_config(embed_cfg, cfg, task_sizes)
    words = np.ascontiguousarray(np.asarray(states, dtype=np.uint64).reshape(F, 4))
    if handles is not None:
        harr = handle_array(handles)
        gptr, cptr = C.cast(harr, C.c_void_p), None
    else:
        carr = np.asarray(counts, np.int64)
        gptr, cptr = None, carr.ctypes.data
    _lib.call("go_sample", ctx.handle, C.byref(cfg_c), F, gptr, cptr, words.ctypes.data,
              _lib.ptr(logits_packed), (1 if logits_f64 else 0) | (2 if shared_logits else 0),
              float(temperature),
              _lib.ptr(actions), _lib.ptr(logp), stream_ptr())
    return actions, logp


@dataclass
class SimBatch:
    step_time: object
    valid: object
    violation: object
    busy: object
    peak: object
    reward: object


VIOLATIONS = {0: None, 1: "colocation", 2: "oom", 3: "cycle_after_fusion"}


def simulate_batch(handle, placement, priorities, topology, policy="priority",
                   baseline=0.0, prio_per_placement=True) -> SimBatch:
    """placement: int32 device tensor [K, n]; priorities int32 [K, n] or [n]."""
    T = torch()
    ctx = context()
    dev = T.device("cuda", ctx.device)
    if policy not in ("fifo", "priority"):
        raise ValueError(f"unknown policy {policy!r}")
    K = int(placement.shape[0])
    d = topology.num_devices
    out = SimBatch(step_time=T.empty(K, dtype=T.float64, device=dev),
                   valid=T.empty(K, dtype=T.uint8, device=dev),
                   violation=T.empty(K, dtype=T.int8, device=dev),
                   busy=T.empty((K, d), dtype=T.float64, device=dev),
                   peak=T.empty((K, d), dtype=T.float64, device=dev),
                   reward=T.empty(K, dtype=T.float64, device=dev))
    placement = placement.contiguous()
    priorities = priorities.contiguous()
    _lib.call("go_simulate", ctx.handle, handle.handle, K, _lib.ptr(placement),
              _lib.ptr(priorities), 1 if prio_per_placement else 0, d,
              _lib.ptr(topology.peak), _lib.ptr(topology.mem_bw), _lib.ptr(topology.cap),
              _lib.ptr(topology.link_bw), 0 if policy == "priority" else 1, float(baseline),
              _lib.ptr(out.step_time), _lib.ptr(out.valid), _lib.ptr(out.violation),
              _lib.ptr(out.busy), _lib.ptr(out.peak), _lib.ptr(out.reward), stream_ptr())
    return out


class GoTraceEvent(C.Structure):
    _fields_ = [("t_start", C.c_double), ("t_end", C.c_double), ("kind", C.c_int32),
                ("src_or_device", C.c_int32), ("dst", C.c_int32), ("group_id", C.c_int32)]


def simulate_trace(handle, placement, priorities, topology, policy="priority",
                   capacity: int = 0):
    """One placement through go_simulate_trace: (SimBatch of K=1, event records as a
    numpy structured array in start order)."""
    T = torch()
    ctx = context()
    dev = T.device("cuda", ctx.device)
    if policy not in ("fifo", "priority"):
        raise ValueError(f"unknown policy {policy!r}")
    d = topology.num_devices
    out = SimBatch(step_time=T.empty(1, dtype=T.float64, device=dev),
                   valid=T.empty(1, dtype=T.uint8, device=dev),
                   violation=T.empty(1, dtype=T.int8, device=dev),
                   busy=T.empty((1, d), dtype=T.float64, device=dev),
                   peak=T.empty((1, d), dtype=T.float64, device=dev), reward=None)
    rec = T.empty((max(1, capacity), C.sizeof(GoTraceEvent)), dtype=T.uint8, device=dev)
    count = T.zeros(1, dtype=T.int64, device=dev)
    _lib.call("go_simulate_trace", ctx.handle, handle.handle, _lib.ptr(placement.contiguous()),
              _lib.ptr(priorities.contiguous()), d, _lib.ptr(topology.peak),
              _lib.ptr(topology.mem_bw), _lib.ptr(topology.cap), _lib.ptr(topology.link_bw),
              0 if policy == "priority" else 1, _lib.ptr(out.step_time), _lib.ptr(out.valid),
              _lib.ptr(out.violation), _lib.ptr(out.busy), _lib.ptr(out.peak), _lib.ptr(rec),
              int(capacity), _lib.ptr(count), stream_ptr())
    n = int(count.item())
    if n > capacity:
        raise AssertionError(f"trace overflow: {n} events > capacity {capacity}")
    dt = np.dtype([("t_start", "<f8"), ("t_end", "<f8"), ("kind", "<i4"),
                   ("src_or_device", "<i4"), ("dst", "<i4"), ("group_id", "<i4")])
    events = rec[:n].cpu().numpy().reshape(-1).view(dt) if n else np.zeros(0, dt)
    return out, events

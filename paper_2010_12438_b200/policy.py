"""Decision network on the B200 (mirrors graphopt.policy, policy.py:1-330).

trunk_forward / task_heads / forward_policy / sample_actions / iterate_decisions
keep the reference signatures and return types; the computation is one
go_forward_status + go_sample per call (csrc/engine.cu, dense.cu, attention.cu,
sample.cu).  Batched twins used by training live in engine.py / training.py."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import TASK_ORDER, EmbedConfig, PolicyConfig, ordered_tasks
from .engine import (EMBED, HEADS, TRUNK, DeviceArray, advance, check_status, forward_batch,
                     pcg_words, sample_batch)
from .graph import as_graph
from .params import init_all_params
from .runtime import context, torch

__all__ = ["TASK_ORDER", "PolicyConfig", "HeadOutputs", "TaskActionBundle", "ordered_tasks",
           "modulation_gate", "trunk_forward", "task_heads", "sample_actions", "forward_policy",
           "iterate_decisions", "init_all_params"]


@dataclass
class HeadOutputs:
    logits: dict  # task -> N x a DeviceArray, rows in topo order
    action_reprs: dict
    value: DeviceArray  # 1 x 1


def _dev32(x, rows=None, cols=None):
    T = torch()
    if isinstance(x, DeviceArray):
        t = x.dev
    elif hasattr(x, "data") and not isinstance(x, np.ndarray) and not hasattr(x, "data_ptr"):
        t = T.as_tensor(np.asarray(x.data))
    else:
        t = T.as_tensor(np.asarray(x) if not hasattr(x, "data_ptr") else x)
    t = t.to(device=T.device("cuda", context().device), dtype=T.float32)
    if cols is not None:
        t = t.reshape(-1, cols)
    return t.contiguous()


def modulation_gate(x):
    """2 * sigmoid (policy.py:122-124); host helper for API completeness."""
    x = np.asarray(getattr(x, "data", x), dtype=np.float64)
    return 2.0 / (1.0 + np.exp(-x))


def trunk_forward(node_embed, graph_embed, store, cfg: PolicyConfig, prefix: str = "policy/",
                  modulation_override=None, cache_perturb=None):
    """policy.py:135-177 (layer-major block-banded attention on device).

    cache_perturb(segment_index, layer, array) -> array (policy.py:146-147, 170-172), the
    reference's diagnostics hook on the cached previous-segment states: the device
    trunk hands each layer's inputs to the hook (go_batch_t.cache_hook) and the
    segment's queries attend to the returned keys/values.  Calls arrive layer-major
    (every segment of layer 0, then layer 1, ...), not segment-major; a pure hook sees
    the same arrays (float32 values as float64) and gives the same result."""
    if prefix != "policy/":
        raise ValueError("only the 'policy/' parameter prefix is supported")
    ne = _dev32(node_embed)
    ge = _dev32(graph_embed).reshape(1, -1)
    n = int(ne.shape[0])
    gs = int(ne.shape[1])
    ecfg = EmbedConfig(gs_dim=gs)
    mod = None
    if modulation_override is not None:
        mod = _dev32(modulation_override).reshape(1, cfg.d_model)
    hook, errors = None, []
    if cache_perturb is not None:
        from . import _lib
        S = cfg.segment_len

        def _hook(_user, layer, xm_p, pfx_p, rows, dm):
            try:
                xm = np.ctypeslib.as_array(xm_p, shape=(rows, dm))
                pfx = np.ctypeslib.as_array(pfx_p, shape=(rows, dm))
                for s in range(1, (rows + S - 1) // S):
                    lo, hi = (s - 1) * S, s * S
                    arr = np.asarray(cache_perturb(s, int(layer), xm[lo:hi].astype(np.float64)),
                                     dtype=np.float64)
                    pfx[lo:hi] = arr.reshape(hi - lo, dm)
            except BaseException as exc:  # ctypes drops exceptions raised in callbacks
                errors.append(exc)

        hook = _lib.CACHE_HOOK(_hook)
    out = forward_batch(store, ecfg, cfg, {"placement": 1}, None, [0], stage_mask=TRUNK,
                        node_embed=ne, graph_embed=ge, mod_override=mod, row_counts=[n],
                        cache_hook=hook)
    if errors:
        raise errors[0]
    return DeviceArray(out.hid)


def task_heads(hiddens, store, cfg: PolicyConfig, tasks, prefix: str = "policy/",
               ablate_action_input=None) -> HeadOutputs:
    """policy.py:187-217 (full N x N attention per task on device)."""
    if not tasks:
        raise ValueError("at least one task required")
    if prefix != "policy/":
        raise ValueError("only the 'policy/' parameter prefix is supported")
    hid = _dev32(hiddens)
    n = int(hid.shape[0])
    sizes = dict(tasks)
    ordered = ordered_tasks(sizes)
    if [t for t, _ in ordered] != [t for t, _ in tasks]:
        raise ValueError("tasks must be in canonical order")
    ablate = 0
    for i, (t, _a) in enumerate(ordered):
        if ablate_action_input and t in ablate_action_input:
            ablate |= 1 << i
    out = forward_batch(store, EmbedConfig(), cfg, sizes, None, [0], stage_mask=HEADS, hid=hid,
                        ablate_mask=ablate, row_counts=[n], want_reps=True)
    logits = {t: DeviceArray(out.logits[i]) for i, (t, _a) in enumerate(ordered)}
    reps = {t: DeviceArray(out.reps[i]) for i, (t, _a) in enumerate(ordered)}
    return HeadOutputs(logits=logits, action_reprs=reps,
                       value=DeviceArray(out.value.reshape(1, 1)))


def sample_actions(logits, temperature: float, rng: np.random.Generator):
    """policy.py:220-237: per-row categorical draw in float64 on device, consuming
    exactly the uniforms rng.random((N, 1)) would; rng is advanced accordingly."""
    if temperature < 0:
        raise ValueError("temperature must be >= 0")
    T = torch()
    if isinstance(logits, DeviceArray):
        lg = logits.dev.to(T.float64)
    else:
        lg = T.as_tensor(np.asarray(getattr(logits, "data", logits), dtype=np.float64))
    lg = lg.to(T.device("cuda", context().device)).contiguous()
    n, a = int(lg.shape[0]), int(lg.shape[1])
    words = [pcg_words(rng)]
    acts, logp = sample_batch(EmbedConfig(), PolicyConfig(), {"placement": a}, None, words,
                              lg.reshape(-1), temperature, logits_f64=True, row_counts=[n])
    if temperature > 0:
        advance(rng, n)
    return acts[0].cpu().numpy().astype(np.int64), logp[0].cpu().numpy()


@dataclass
class TaskActionBundle:
    """policy.py:240-261."""

    tasks: list
    logits: dict
    actions: dict
    log_probs: dict
    value: float
    prev_actions: dict | None
    embed_seed: int
    temperature: float

    def joint_log_prob(self) -> float:
        return float(sum(np.asarray(lp).sum() for lp in self.log_probs.values()))

    def to_assignment(self, task: str, num_actions: int):
        from .simulator import ActionAssignment
        return ActionAssignment(task, self.actions[task], num_actions)


def forward_policy(graph, store, embed_cfg: EmbedConfig, cfg: PolicyConfig, task_sizes: dict,
                   prev_actions, embed_seed: int) -> HeadOutputs:
    """policy.py:264-276: features -> embed -> trunk -> heads, one device call."""
    g = as_graph(graph)
    tasks = ordered_tasks(task_sizes)
    h = context().graph(g)
    prev = _prev_dev(prev_actions, tasks, g.num_nodes)
    out = forward_batch(store, embed_cfg, cfg, task_sizes, [h], [embed_seed], prev_actions=prev,
                        want_reps=True)
    check_status(out)
    logits = {t: DeviceArray(out.logits[i]) for i, (t, _a) in enumerate(tasks)}
    reps = {t: DeviceArray(out.reps[i]) for i, (t, _a) in enumerate(tasks)}
    return HeadOutputs(logits=logits, action_reprs=reps, value=DeviceArray(out.value.reshape(1, 1)))


def _prev_dev(prev_actions, tasks, n):
    if prev_actions is None:
        return None
    T = torch()
    rows = []
    for t, a in tasks:
        v = np.asarray(getattr(prev_actions[t], "actions", prev_actions[t]), dtype=np.int64)
        if v.shape != (n,):
            raise ValueError(f"prev_actions has shape {v.shape}, want ({n},)")
        if v.min(initial=0) < 0 or v.max(initial=0) >= a:
            raise ValueError(f"action out of range [0,{a})")
        rows.append(v.astype(np.int32))
    return T.as_tensor(np.stack(rows)).to(T.device("cuda", context().device)).contiguous()


def iterate_decisions(graph, store, embed_cfg: EmbedConfig, cfg: PolicyConfig, task_sizes: dict,
                      iterations: int, seed: int, temperature: float = 1.0):
    """policy.py:279-319 -> (final bundle, trajectory)."""
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    from .training import run_decisions
    bundles = run_decisions(store, [as_graph(graph)], embed_cfg, cfg, task_sizes, iterations,
                            [seed], temperature, keep_trajectory=True)[0]
    return bundles[-1], bundles

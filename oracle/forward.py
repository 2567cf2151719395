"""Float64 numpy restatement of the reference forward path (TEST
INFRASTRUCTURE ONLY — see oracle/__init__.py).

No autodiff tape is kept ("ref-lean"): the trunk is
evaluated layer-major as the block-banded attention it is (each segment of
layer l reads only layer l-1 rows, policy.py:165-174) and the N x N task-head
attention is evaluated in row chunks, so 30k/80k-node graphs fit in RAM.
Parameters are a dict name -> float64 array with the reference names
(embedding.py:35-44, policy.py:44-94).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import graph as og

TASK_ORDER = ("placement", "schedule_priority", "fusion_priority")  # policy.py:18


@dataclass(frozen=True)
class EmbedCfg:  # embedding.py:17-21
    gs_layers: int = 4
    gs_dim: int = 128
    gs_knn: int = 5


@dataclass(frozen=True)
class PolicyCfg:  # policy.py:21-33
    trf_layers: int = 4
    d_model: int = 128
    n_head: int = 3
    d_head: int = 15
    d_inner: int = 512
    segment_len: int = 64
    iterations: int = 2


def ordered_tasks(task_sizes):  # policy.py:36-41
    return [(t, task_sizes[t]) for t in TASK_ORDER if t in task_sizes]


# ----------------------------------------------------------------------------------------
# primitives (tensor.py)

def sigmoid(x):  # tensor.py:141-145
    return 1.0 / (1.0 + np.exp(-x))


def relu(x):  # tensor.py:133-138
    return np.where(x > 0, x, 0.0)


def layer_norm(x, g, b, eps=1e-5):  # tensor.py:330-351
    mu = x.mean(axis=-1, keepdims=True)
    xc = x - mu
    var = (xc * xc).mean(axis=-1, keepdims=True)
    return g * (xc / np.sqrt(var + eps)) + b


def softmax(x):  # tensor.py:300-312
    s = x - x.max(axis=-1, keepdims=True)
    e = np.exp(s)
    return e / e.sum(axis=-1, keepdims=True)


# ----------------------------------------------------------------------------------------
# embedding (embedding.py)

def neighbor_arrays(g, k, seed):
    """(gather row, segment row) pairs in topo-row space (embedding.py:47-70).
    Sampling for deg > k uses numpy's own Generator.choice, the reference's
    dependency (restated in oracle/rng.py)."""
    order = g["topo"]
    pos = np.empty(g["n"], np.int64)
    pos[order] = np.arange(g["n"])
    nb = og.neighbors(g)
    gather, seg = [], []
    for row, v in enumerate(order.tolist()):
        lst = nb[v]
        if len(lst) > k:
            pick = np.random.default_rng([seed, v]).choice(len(lst), size=k, replace=False)
            lst = sorted(lst[i] for i in pick)
        for u in lst:
            gather.append(pos[u])
            seg.append(row)
    return np.array(gather, np.int64), np.array(seg, np.int64)


def segment_max(vals, seg, n):
    """tensor.py:229-263 forward: empty segments give zero rows."""
    out = np.zeros((n, vals.shape[1]))
    if len(seg) == 0:
        return out
    starts = np.flatnonzero(np.r_[True, seg[1:] != seg[:-1]])
    out[seg[starts]] = np.maximum.reduceat(vals, starts, axis=0)
    return out


def embed(g, feats, P, cfg: EmbedCfg, seed=0, prefix="embed/"):
    """embedding.py:73-98 -> (node_embed N x d, graph_embed 1 x d)."""
    n = g["n"]
    gather, seg = neighbor_arrays(g, cfg.gs_knn, seed)
    h = feats @ P[prefix + "in_w"] + P[prefix + "in_b"]
    for l in range(cfg.gs_layers):
        t = sigmoid(h @ P[f"{prefix}agg_w{l}"] + P[f"{prefix}agg_b{l}"])
        pooled = segment_max(t[gather], seg, n) if len(gather) else np.zeros((n, cfg.gs_dim))
        h = relu(np.concatenate([h, pooled], axis=1) @ P[f"{prefix}fc_w{l}"]
                 + P[f"{prefix}fc_b{l}"])
    if not np.isfinite(h).all():
        raise FloatingPointError("non-finite node embeddings (bad init or features)")
    return h, h.mean(axis=0, keepdims=True)


# ----------------------------------------------------------------------------------------
# policy (policy.py)

def mha(P, prefix, cfg: PolicyCfg, xq, xkv):
    """policy.py:97-109 for one query/key set (no segmentation)."""
    q = xq @ P[prefix + "q_w"] + P[prefix + "q_b"]
    k = xkv @ P[prefix + "k_w"] + P[prefix + "k_b"]
    v = xkv @ P[prefix + "v_w"] + P[prefix + "v_b"]
    heads = []
    for i in range(cfg.n_head):
        sl = slice(i * cfg.d_head, (i + 1) * cfg.d_head)
        s = (q[:, sl] @ k[:, sl].T) * (1.0 / math.sqrt(cfg.d_head))
        heads.append(softmax(s) @ v[:, sl])
    return np.concatenate(heads, axis=1) @ P[prefix + "o_w"] + P[prefix + "o_b"]


def block_post(P, prefix, x, attn):
    """Post-LN residual + FF half of transformer_block (policy.py:112-119)."""
    h = layer_norm(x + attn, P[prefix + "ln1_g"], P[prefix + "ln1_b"])
    ff = relu(h @ P[prefix + "ff_w1"] + P[prefix + "ff_b1"]) @ P[prefix + "ff_w2"] + P[prefix + "ff_b2"]
    return layer_norm(h + ff, P[prefix + "ln2_g"], P[prefix + "ln2_b"])


def modulate(graph_embed, P, cfg: PolicyCfg, prefix="policy/"):
    """policy.py:122-132: length-1 block on in_w(h_G), then 2*sigmoid."""
    g = graph_embed @ P[prefix + "in_w"] + P[prefix + "in_b"]
    out = block_post(P, prefix + "mod/", g, mha(P, prefix + "mod/attn_", cfg, g, g))
    return 2.0 * sigmoid(out)


def banded_attention(P, prefix, cfg: PolicyCfg, xm):
    """Layer-major restatement of the segment recurrence (policy.py:157-177):
    segment s's queries attend to [xm(seg s-1) || xm(seg s)], no mask."""
    n = xm.shape[0]
    S = cfg.segment_len
    q = xm @ P[prefix + "q_w"] + P[prefix + "q_b"]
    k = xm @ P[prefix + "k_w"] + P[prefix + "k_b"]
    v = xm @ P[prefix + "v_w"] + P[prefix + "v_b"]
    out = np.zeros((n, cfg.n_head * cfg.d_head))
    scale = 1.0 / math.sqrt(cfg.d_head)
    for lo in range(0, n, S):
        hi = min(n, lo + S)
        klo = max(0, lo - S)
        for i in range(cfg.n_head):
            sl = slice(i * cfg.d_head, (i + 1) * cfg.d_head)
            s = (q[lo:hi, sl] @ k[klo:hi, sl].T) * scale
            out[lo:hi, sl] = softmax(s) @ v[klo:hi, sl]
    return out @ P[prefix + "o_w"] + P[prefix + "o_b"]


def trunk_forward(node_embed, graph_embed, P, cfg: PolicyCfg, prefix="policy/", mod=None):
    """policy.py:135-177."""
    if mod is None:
        mod = modulate(graph_embed, P, cfg, prefix)
    x = node_embed @ P[prefix + "in_w"] + P[prefix + "in_b"]
    for l in range(cfg.trf_layers):
        xm = x * mod
        bp = f"{prefix}block{l}/"
        x = block_post(P, bp, xm, banded_attention(P, bp + "attn_", cfg, xm))
    return x


def full_attention_chunked(P, prefix, cfg: PolicyCfg, h, chunk=2048):
    """policy.py:210 multi_head_attention(h, h) over all N rows, evaluated in
    row chunks of queries (same math, bounded memory)."""
    n = h.shape[0]
    q = h @ P[prefix + "q_w"] + P[prefix + "q_b"]
    k = h @ P[prefix + "k_w"] + P[prefix + "k_b"]
    v = h @ P[prefix + "v_w"] + P[prefix + "v_b"]
    out = np.zeros((n, cfg.n_head * cfg.d_head))
    scale = 1.0 / math.sqrt(cfg.d_head)
    for i in range(cfg.n_head):
        sl = slice(i * cfg.d_head, (i + 1) * cfg.d_head)
        kt = k[:, sl].T.copy()
        vs = v[:, sl]
        for lo in range(0, n, chunk):
            s = (q[lo:lo + chunk, sl] @ kt) * scale
            out[lo:lo + chunk, sl] = softmax(s) @ vs
    return out @ P[prefix + "o_w"] + P[prefix + "o_b"]


def task_heads(hid, P, cfg: PolicyCfg, tasks, prefix="policy/", ablate=None, chunk=2048):
    """policy.py:187-217 -> (logits dict, reprs dict, value 1x1)."""
    n, d = hid.shape
    zeros = np.zeros((n, d))
    a_prev = zeros
    logits, reprs = {}, {}
    for task, a in tasks:
        p = f"{prefix}task/{task}/"
        a_in = zeros if (ablate and task in ablate) else a_prev
        h = layer_norm(np.concatenate([a_in, hid], axis=1) @ P[p + "cat_w"] + P[p + "cat_b"],
                       P[p + "ln_g"], P[p + "ln_b"])
        attn = full_attention_chunked(P, prefix + "task_attn/", cfg, h, chunk)
        rep = relu(attn @ P[p + "fc_w1"] + P[p + "fc_b1"]) @ P[p + "fc_w2"] + P[p + "fc_b2"]
        logits[task] = rep @ P[p + "out_w"] + P[p + "out_b"]
        reprs[task] = rep
        a_prev = rep
    value = a_prev.mean(axis=0, keepdims=True) @ P[prefix + "value_w"] + P[prefix + "value_b"]
    return logits, reprs, value


def task_heads_rows(hid, P, cfg: PolicyCfg, tasks, rows, prefix="policy/"):
    """policy.py:187-217 restricted to query rows `rows` (topo-row indices) for a
    single task: the head's keys/values still span all N rows (h for every row is
    one N x 256 x 128 product), only the queries and everything after the attention
    are evaluated for `rows`.  Returns (logits[len(rows), a], rep rows).  With more
    than one task the next task's keys need every row's rep, so use task_heads."""
    if len(tasks) != 1:
        raise ValueError("task_heads_rows evaluates a single task; use task_heads")
    task, _a = tasks[0]
    n, d = hid.shape
    p = f"{prefix}task/{task}/"
    pa = prefix + "task_attn/"
    h = layer_norm(np.concatenate([np.zeros((n, d)), hid], axis=1) @ P[p + "cat_w"] + P[p + "cat_b"],
                   P[p + "ln_g"], P[p + "ln_b"])
    rows = np.asarray(rows, np.int64)
    q = h[rows] @ P[pa + "q_w"] + P[pa + "q_b"]
    k = h @ P[pa + "k_w"] + P[pa + "k_b"]
    v = h @ P[pa + "v_w"] + P[pa + "v_b"]
    out = np.zeros((len(rows), cfg.n_head * cfg.d_head))
    scale = 1.0 / math.sqrt(cfg.d_head)
    for i in range(cfg.n_head):
        sl = slice(i * cfg.d_head, (i + 1) * cfg.d_head)
        out[:, sl] = softmax((q[:, sl] @ k[:, sl].T) * scale) @ v[:, sl]
    attn = out @ P[pa + "o_w"] + P[pa + "o_b"]
    rep = relu(attn @ P[p + "fc_w1"] + P[p + "fc_b1"]) @ P[p + "fc_w2"] + P[p + "fc_b2"]
    return rep @ P[p + "out_w"] + P[p + "out_b"], rep


def uniform_at(seed, index):
    """The reference's uniform number `index` of default_rng(seed).random() calls
    (policy.py:235 draws rng.random((N, 1)) per task and iteration, so row r of task t
    in iteration it is draw (it*T + t)*N + r).  PCG64.advance(k) jumps
    the stream by k 64-bit outputs, one per double."""
    gen = np.random.default_rng(seed)
    gen.bit_generator.advance(int(index))
    return float(gen.random())


def sample_row(logits_row, temperature, u):
    """sample_actions (policy.py:220-237) for one row given its uniform u."""
    class _U:
        def random(self, shape):
            return np.full(shape, u)
    a, lp = sample_actions(np.asarray(logits_row, np.float64)[None, :], temperature, _U())
    return int(a[0]), float(lp[0])


def sample_actions(logits, temperature, rng):
    """policy.py:220-237, verbatim numpy semantics."""
    if temperature < 0:
        raise ValueError("temperature must be >= 0")
    if temperature == 0.0:
        return np.argmax(logits, axis=1), np.zeros(len(logits))
    z = logits / temperature
    z = z - z.max(axis=1, keepdims=True)
    logp = z - np.log(np.exp(z).sum(axis=1, keepdims=True))
    cum = np.cumsum(np.exp(logp), axis=1)
    u = rng.random((len(logits), 1)) * cum[:, -1:]
    actions = (u > cum).sum(axis=1)
    return actions, logp[np.arange(len(logits)), actions]


def forward_policy(g, P, ecfg, pcfg, task_sizes, prev_actions, embed_seed):
    """policy.py:264-276."""
    tasks = ordered_tasks(task_sizes)
    prev = None if prev_actions is None else [prev_actions[t] for t, _ in tasks]
    feats = og.node_features(g, prev, [a for _, a in tasks])
    ne, ge = embed(g, feats, P, ecfg, seed=embed_seed)
    hid = trunk_forward(ne, ge, P, pcfg)
    return task_heads(hid, P, pcfg, tasks)


def iterate_decisions(g, P, ecfg, pcfg, task_sizes, iterations, seed, temperature=1.0):
    """policy.py:279-319; returns the list of per-iteration dicts."""
    if iterations < 1:
        raise ValueError("iterations must be >= 1")
    rng = np.random.default_rng(seed)
    tasks = ordered_tasks(task_sizes)
    order = g["topo"]
    prev = None
    traj = []
    for _ in range(iterations):
        logits, _reprs, value = forward_policy(g, P, ecfg, pcfg, task_sizes, prev, seed)
        acts, logps = {}, {}
        for task, _a in tasks:
            ra, rl = sample_actions(logits[task], temperature, rng)
            na = np.zeros(g["n"], np.int64)
            na[order] = ra
            acts[task] = na
            logps[task] = rl
        traj.append(dict(logits=logits, actions=acts, log_probs=logps,
                         value=float(value[0, 0]),
                         prev_actions=None if prev is None else {k: v.copy() for k, v in prev.items()},
                         embed_seed=seed, temperature=temperature))
        prev = acts
    return traj

"""Parameter initialisation restatement (TEST INFRASTRUCTURE ONLY — see
oracle/__init__.py).  Follows embedding.py:28-44, policy.py:44-94 and
policy.py:322-330: same names, shapes and numpy draw order, so the same seed
gives bit-identical float64 weights."""
from __future__ import annotations

import numpy as np

from .forward import EmbedCfg, PolicyCfg, ordered_tasks
from .graph import feature_dim


def _uniform(rng, shape, fan_in):
    s = 1.0 / np.sqrt(max(1, fan_in))
    return rng.uniform(-s, s, size=shape)


def init_all_params(ecfg: EmbedCfg, pcfg: PolicyCfg, task_sizes, seed):
    rng = np.random.default_rng(seed)
    P = {}
    tasks = ordered_tasks(task_sizes)
    fdim = feature_dim([a for _, a in tasks])
    d = ecfg.gs_dim
    P["embed/in_w"] = _uniform(rng, (fdim, d), fdim)
    P["embed/in_b"] = np.zeros(d)
    for l in range(ecfg.gs_layers):
        P[f"embed/agg_w{l}"] = _uniform(rng, (d, d), d)
        P[f"embed/agg_b{l}"] = np.zeros(d)
        P[f"embed/fc_w{l}"] = _uniform(rng, (2 * d, d), 2 * d)
        P[f"embed/fc_b{l}"] = np.zeros(d)
    dm, w, di = pcfg.d_model, pcfg.n_head * pcfg.d_head, pcfg.d_inner

    def attn(prefix):
        for name in ("q", "k", "v"):
            P[f"{prefix}{name}_w"] = _uniform(rng, (dm, w), dm)
            P[f"{prefix}{name}_b"] = np.zeros(w)
        P[f"{prefix}o_w"] = _uniform(rng, (w, dm), w)
        P[f"{prefix}o_b"] = np.zeros(dm)

    def block(prefix):
        attn(prefix + "attn_")
        P[prefix + "ln1_g"] = np.ones(dm)
        P[prefix + "ln1_b"] = np.zeros(dm)
        P[prefix + "ff_w1"] = _uniform(rng, (dm, di), dm)
        P[prefix + "ff_b1"] = np.zeros(di)
        P[prefix + "ff_w2"] = _uniform(rng, (di, dm), di)
        P[prefix + "ff_b2"] = np.zeros(dm)
        P[prefix + "ln2_g"] = np.ones(dm)
        P[prefix + "ln2_b"] = np.zeros(dm)

    P["policy/in_w"] = _uniform(rng, (d, dm), d)
    P["policy/in_b"] = np.zeros(dm)
    for l in range(pcfg.trf_layers):
        block(f"policy/block{l}/")
    block("policy/mod/")
    attn("policy/task_attn/")
    for task, a in tasks:
        p = f"policy/task/{task}/"
        P[p + "cat_w"] = _uniform(rng, (2 * dm, dm), 2 * dm)
        P[p + "cat_b"] = np.zeros(dm)
        P[p + "ln_g"] = np.ones(dm)
        P[p + "ln_b"] = np.zeros(dm)
        P[p + "fc_w1"] = _uniform(rng, (dm, di), dm)
        P[p + "fc_b1"] = np.zeros(di)
        P[p + "fc_w2"] = _uniform(rng, (di, dm), di)
        P[p + "fc_b2"] = np.zeros(dm)
        P[p + "out_w"] = np.zeros((dm, a))
        P[p + "out_b"] = np.zeros(a)
    P["policy/value_w"] = np.zeros((dm, 1))
    P["policy/value_b"] = np.zeros(1)
    return P


def randomize_zero_init(P, seed=1):
    """refill every all-zero tensor (biases, out/value
    heads) with Uniform(+-1/sqrt(shape[0])) from default_rng(seed), visiting
    names in sorted order, so logits are O(1) instead of identically 0."""
    rng = np.random.default_rng(seed)
    for name in sorted(P):
        a = P[name]
        if not np.any(a):
            P[name] = _uniform(rng, a.shape, a.shape[0])
    return P

#!/usr/bin/env python
"""Normwise logit/value error of each task-head attention variant vs the float64 oracle
(3,000 random hidden rows, default config).  Development aid."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np


def rel_err(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


from paper_2010_12438_b200 import EmbedConfig, PolicyConfig, init_all_params, randomize_zero_init
from paper_2010_12438_b200.policy import ordered_tasks, task_heads
from oracle import forward as of
sizes = {"placement": 8}
ecfg, pcfg = EmbedConfig(), PolicyConfig()
store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
P = {n: np.asarray(p.data) for n, p in store.items()}
rng = np.random.default_rng(1)
hid = rng.normal(size=(3000, 128))
tasks = ordered_tasks(sizes)
lg, _, val = of.task_heads(hid, P, of.PolicyCfg(), tasks)
for mode in ("tc", "tf32", "online", "simt"):
    os.environ["GO_ATTN"] = mode
    out = task_heads(hid, store, pcfg, tasks)
    print(mode, "logits rel err %.2e" % rel_err(out.logits["placement"].data, lg["placement"]), "value %.2e" % rel_err(out.value.data, val), flush=True)

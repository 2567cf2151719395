#!/usr/bin/env python
"""Head-attention cost when trained-magnitude weights push score bounds past the fp16
limit (VERDICT r1 "next" #5).  On the cfg4 graph's real trunk output, W_q and W_k are
scaled by s (scores grow by s^2, as training sharpens attention); for each s this prints
the fraction of (head, 384-query work item) pairs whose bound exceeds 14 (those items move
to the tf32 kernel, tc_attention16.cu) or 60 (whole launch to the online kernel), and the
task-head time per forward for the per-item fallback against forcing the tf32 kernel on
the whole launch (round 1's behaviour for any fallback).
    python scripts/attn_fallback.py > profiles/r2_attn_fallback.json"""
import json
import math
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def bounds(hid, P, task):
    p, pa = f"policy/task/{task}/", "policy/task_attn/"
    n, d = hid.shape
    x = np.concatenate([np.zeros((n, d)), hid], 1) @ P[p + "cat_w"] + P[p + "cat_b"]
    mu = x.mean(1, keepdims=True)
    var = ((x - mu) ** 2).mean(1, keepdims=True)
    h = P[p + "ln_g"] * (x - mu) / np.sqrt(var + 1e-5) + P[p + "ln_b"]
    q = h @ P[pa + "q_w"] + P[pa + "q_b"]
    k = h @ P[pa + "k_w"] + P[pa + "k_b"]
    sc = math.log2(math.e) / math.sqrt(15)
    return np.stack([np.linalg.norm(q[:, i * 15:(i + 1) * 15], axis=1)
                     * np.linalg.norm(k[:, i * 15:(i + 1) * 15], axis=1).max() * sc
                     for i in range(3)], 1)


def main():
    import torch

    from paper_2010_12438_b200 import EmbedConfig, PolicyConfig, init_all_params, randomize_zero_init
    from paper_2010_12438_b200.embedding import embed
    from paper_2010_12438_b200.graph import node_features
    from paper_2010_12438_b200.policy import task_heads, trunk_forward
    from synthetic.workloads import WorkloadSpec, gen_workload
    g = gen_workload(WorkloadSpec("attention-stack", 8000, 1, 64, seed=0), node_cap=10**6)
    sizes = {"placement": 8}
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
    emb = embed(g, node_features(g, None, [8]), store, ecfg, seed=1)
    hid_dev = trunk_forward(emb.node_embed, emb.graph_embed, store, pcfg)
    hid = hid_dev.data
    q0, k0 = store["policy/task_attn/q_w"].data.copy(), store["policy/task_attn/k_w"].data.copy()
    rows = []
    for s in (1.0, 1.5, 2.0, 2.5, 3.0):
        store["policy/task_attn/q_w"].data = q0 * s
        store["policy/task_attn/k_w"].data = k0 * s
        P = {n: np.asarray(p.data) for n, p in store.items()}
        b = bounds(hid, P, "placement")
        items = np.stack([(b[i:i + 384] > 14.0).any(0) for i in range(0, len(b), 384)])
        rec = {"scale": s, "bound_max": float(b.max()), "rows_over_14": float((b > 14).mean()),
               "items_tf32": float(items.mean()), "online": bool(b.max() > 60)}
        for mode in ("default", "tf32"):
            if mode == "tf32":
                os.environ["GO_ATTN"] = "tf32"
            for _ in range(2):
                task_heads(hid_dev, store, pcfg, [("placement", 8)])
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                task_heads(hid_dev, store, pcfg, [("placement", 8)])
            e1.record()
            torch.cuda.synchronize()
            rec[f"heads_ms_{mode}"] = e0.elapsed_time(e1) / 5
            os.environ.pop("GO_ATTN", None)
        rows.append(rec)
        print(rec, file=sys.stderr, flush=True)
    print(json.dumps({"what": "task_heads per cfg4 forward (80,001 rows, 1 task) with W_q, W_k x scale",
                      "rows": rows}, indent=1))


if __name__ == "__main__":
    main()

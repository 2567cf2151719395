"""Parity at the BASELINE configurations (VERDICT r1 "next" #1).

Helper module (not a test file): `tests/test_gpu_headline.py` asserts on what these
functions return and `scripts/parity_report.py` writes the same numbers to JSON
(profiles/r2_parity_headline.json).  Everything here compares the DEVICE path,
called through the product's public API, with the float64 CPU oracle (oracle/,
pinned to the unmodified reference by tests/golden) on the same inputs:

* stage by stage -- embeddings (embedding.py:73-98), trunk output (policy.py:135-177)
  and task-head logits (policy.py:187-217) -- both end to end (oracle chain from the
  oracle's own inputs) and isolated (oracle stage applied to the device's input of
  that stage, so one stage's error is not charged to the next);
* head logits on a seeded sample of query rows when N is too large for a float64
  N x N attention (oracle.forward.task_heads_rows; every key still enters);
* sampled actions and log-probs (policy.py:220-237, 279-319) row by row with the
  reference's own uniforms (draw (it*T + t)*N + r of default_rng(seed)); a row whose
  action differs is a FLIP and must be EXPLAINED: its uniform lies within
  4*max|d logit| of a CDF edge (softmax moves each cumulative probability by at most
  2*||d z||_inf to first order), i.e. the flip is the logit tolerance, not a sampler bug;
* DES results (simulator.py:280-441) bit-exact: step time, busy, peak memory, validity.

Errors are reported two ways: normwise max|d| / max|ref| (the 1e-4 bar of
BASELINE.json's north_star) and elementwise max |d| / (|ref| + 1e-3 * max|ref|).
"""
from __future__ import annotations

import numpy as np

from oracle import des as od
from oracle import forward as of
from oracle import graph as og

NORM_BAR = 1e-4


def errors(got, want, floor=1e-3):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    scale = max(float(np.abs(want).max(initial=0.0)), 1e-30)
    d = np.abs(got - want)
    return {"normwise": float(d.max(initial=0.0) / scale),
            "elementwise": float((d / (np.abs(want) + floor * scale)).max(initial=0.0)),
            "max_abs": float(d.max(initial=0.0)), "ref_max_abs": scale}


def oracle_graph(g):
    return og.make(g.num_nodes, g.op, g.flops, g.out_bytes, g.src, g.dst, g.ebytes,
                   getattr(g, "coloc", None))


def oracle_params(store):
    return {n: np.asarray(p.data, np.float64) for n, p in store.items()}


def sample_rows(n, count, seed=0):
    """Seeded query-row sample: always the first/last rows, the rest uniform."""
    if count >= n:
        return np.arange(n)
    rng = np.random.default_rng(seed)
    rest = rng.choice(np.arange(1, n - 1), size=count - 2, replace=False)
    return np.sort(np.r_[0, n - 1, rest])


def oracle_logits(ogr, P, sizes, prev, seed, rows=None, hid=None):
    """(logits of `rows` (all rows if None) for the last task, hid) through the oracle
    chain features -> embed -> trunk -> heads, or from a given `hid`."""
    tasks = of.ordered_tasks(sizes)
    if hid is None:
        prev_list = None if prev is None else [np.asarray(prev[t]) for t, _ in tasks]
        feats = og.node_features(ogr, prev_list, [a for _, a in tasks])
        ne, ge = of.embed(ogr, feats, P, of.EmbedCfg(), seed=seed)
        hid = of.trunk_forward(ne, ge, P, of.PolicyCfg())
    if rows is None:
        lg, _, _ = of.task_heads(hid, P, of.PolicyCfg(), tasks)
        return {t: lg[t] for t, _ in tasks}, hid
    lg, _ = of.task_heads_rows(hid, P, of.PolicyCfg(), tasks, rows)
    return {tasks[0][0]: lg}, hid


def check_actions(got_actions, got_logp, logits_ref, logits_dev, order, rows, seed, it, t_index,
                  num_tasks, temperature=1.0):
    """Row-by-row sampler check.  got_actions node-indexed, got_logp topo rows;
    logits_ref / logits_dev are [len(rows), a] (topo rows `rows`)."""
    n = len(order)
    flips, unexplained, lp_err = [], [], 0.0
    for j, r in enumerate(rows):
        u = of.uniform_at(seed, (it * num_tasks + t_index) * n + int(r))
        a_ref, lp_ref = of.sample_row(logits_ref[j], temperature, u)
        a_got = int(got_actions[order[r]])
        if a_got != a_ref:
            z = np.asarray(logits_ref[j], np.float64) / temperature
            p = np.exp(z - z.max())
            cum = np.cumsum(p / p.sum())
            gap = float(np.abs(cum[:-1] - u * cum[-1]).min(initial=np.inf))
            dz = float(np.abs(np.asarray(logits_dev[j], np.float64) - logits_ref[j]).max())
            flips.append(int(r))
            if not gap <= 4.0 * dz / temperature:
                unexplained.append({"row": int(r), "gap": gap, "max_dlogit": dz})
        else:
            lp_err = max(lp_err, abs(float(got_logp[r]) - lp_ref))
    return {"rows": int(len(rows)), "flips": len(flips), "flip_rate": len(flips) / max(1, len(rows)),
            "unexplained": unexplained, "logp_max_abs_err": lp_err}


def check_des(g, ogr, placements, topology_d, priorities=None):
    """Device simulate_many (the rollout path) vs the oracle DES, bit for bit."""
    from paper_2010_12438_b200.costmodel import uniform_topology
    from paper_2010_12438_b200.simulator import simulate_many, singleton_fused
    n = g.num_nodes
    pri = np.zeros(n, np.int64) if priorities is None else priorities
    placements = np.asarray(placements, np.int64).reshape(-1, n)
    res = simulate_many(singleton_fused(g), placements, pri, uniform_topology(topology_d))
    st = res.step_time.cpu().numpy()
    va = res.valid.cpu().numpy().astype(bool)
    busy = res.busy.cpu().numpy()
    peak = res.peak.cpu().numpy()
    fg = od.singleton(ogr)
    top = od.uniform_topology(topology_d)
    mism = []
    for k, pl in enumerate(placements):
        w = od.simulate(ogr, fg, pl, pri, top)
        ok = (st[k] == w["step_time"] and va[k] == w["valid"]
              and np.array_equal(busy[k], np.asarray(w["busy"]))
              and np.array_equal(peak[k], np.asarray(w["peak"])))
        if not ok:
            mism.append({"k": k, "got": float(st[k]), "want": float(w["step_time"])})
    return {"placements": int(len(placements)), "mismatches": mism,
            "step_times": [float(x) for x in st]}


def forward_and_decisions(g, sizes, seed, rows=None, iterations=2, isolate=True):
    """Stage errors + iterate_decisions actions for one graph.  rows=None: all rows
    (full float64 heads)."""
    from paper_2010_12438_b200 import EmbedConfig, PolicyConfig, init_all_params, randomize_zero_init
    from paper_2010_12438_b200.embedding import embed
    from paper_2010_12438_b200.graph import node_features
    from paper_2010_12438_b200.policy import (forward_policy, iterate_decisions, ordered_tasks,
                                              trunk_forward)
    ecfg, pcfg = EmbedConfig(), PolicyConfig(iterations=iterations)
    store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
    P = oracle_params(store)
    ogr = oracle_graph(g)
    tasks = ordered_tasks(sizes)
    task = tasks[-1][0]
    n = g.num_nodes
    order = np.asarray(g.topo_order())
    rep = {"nodes": n, "rows_checked": n if rows is None else int(len(rows))}
    sel = slice(None) if rows is None else rows

    # --- stages, iteration 1 (prev = None)
    feats = node_features(g, None, [a for _, a in tasks])
    emb = embed(g, feats, store, ecfg, seed=seed)
    ne_d, ge_d = emb.node_embed.data, emb.graph_embed.data
    hid_d = trunk_forward(emb.node_embed, emb.graph_embed, store, pcfg).data
    heads = forward_policy(g, store, ecfg, pcfg, sizes, None, seed)
    lg_d = heads.logits[task].data[sel]
    feats_o = og.node_features(ogr, None, [a for _, a in tasks])
    ne_o, ge_o = of.embed(ogr, feats_o, P, of.EmbedCfg(), seed=seed)
    hid_o = of.trunk_forward(ne_o, ge_o, P, of.PolicyCfg())
    lg_o, _ = oracle_logits(ogr, P, sizes, None, seed, rows, hid=hid_o)
    rep["embed"] = errors(ne_d, ne_o)
    rep["graph_embed"] = errors(ge_d, ge_o)
    rep["trunk_e2e"] = errors(hid_d, hid_o)
    rep["logits_e2e"] = errors(lg_d, lg_o[task])
    if isolate:
        hid_iso = of.trunk_forward(ne_d, ge_d, P, of.PolicyCfg())
        rep["trunk_isolated"] = errors(hid_d, hid_iso)
        lg_iso, _ = oracle_logits(ogr, P, sizes, None, seed, rows, hid=hid_d)
        rep["logits_isolated"] = errors(lg_d, lg_iso[task])
    if rows is None:
        rep["value_e2e"] = errors(heads.value.data, of.task_heads(hid_o, P, of.PolicyCfg(), tasks)[2])

    # --- iterate_decisions: every iteration's actions on the checked rows
    bundle, traj = iterate_decisions(g, store, ecfg, pcfg, sizes, iterations, seed)
    rep["iterations"] = []
    prev = None
    for it, b in enumerate(traj):
        lg_ref = lg_o if it == 0 else oracle_logits(ogr, P, sizes, prev, seed, rows)[0]
        it_rep = {"logits_e2e": errors(b.logits[task][sel], lg_ref[task])}
        for t_i, (t, _a) in enumerate(tasks):
            if t != task:
                continue
            it_rep["actions"] = check_actions(b.actions[t], b.log_probs[t], lg_ref[t],
                                              b.logits[t][sel], order,
                                              np.arange(n) if rows is None else rows, seed, it,
                                              t_i, len(tasks))
        rep["iterations"].append(it_rep)
        prev = b.actions  # the oracle's next iteration sees the DEVICE's actions
    rep["final_actions"] = {t: bundle.actions[t] for t, _ in tasks}
    return rep

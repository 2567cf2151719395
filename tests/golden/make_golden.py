"""Generate the golden fixtures in tests/golden/*.npz from the UNMODIFIED
reference package (/root/reference/pkg/src/graphopt, read-only).

Run once in the development container (the reference does not exist on the
GPU box; the fixtures travel instead):

    python tests/golden/make_golden.py

Parameters are never stored (1.2M float64 would bloat the fixtures): each
case records (config, task sizes, init seed) and the oracle/product rebuild
them with their restated init_all_params + randomize_zero_init; a per-tensor
checksum pins that restatement.
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(REF / "tests"))
ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from graphopt import tensor as T  # noqa: E402
from graphopt.baselines import default_assignments, greedy_placement  # noqa: E402
from graphopt.costmodel import DeviceSpec, DeviceTopology  # noqa: E402
from graphopt.embedding import EmbedConfig, _neighbor_arrays, embed, sample_neighbors  # noqa: E402
from graphopt.graph import OP_INDEX, node_features  # noqa: E402
from graphopt.policy import (PolicyConfig, init_all_params, iterate_decisions,  # noqa: E402
                             ordered_tasks, sample_actions, task_heads, trunk_forward)
from graphopt.simulator import (ActionAssignment, FusedGraph, FusionConfig,  # noqa: E402
                                apply_fusion, simulate, singleton_fused)
from graphopt.training import (PPOHyper, collect_rollouts, ppo_update,  # noqa: E402
                               task_action_sizes)
from graphopt.workloads import WorkloadSpec, gen_workload  # noqa: E402

import conftest as C  # noqa: E402  (reference test fixtures: random_graph, make_graph)

OUT = Path(__file__).resolve().parent


def graph_arrays(g, prefix, out):
    names = {}
    coloc = []
    for nd in g.nodes:
        c = nd.colocation_group
        coloc.append(-1 if c is None else names.setdefault(c, len(names)))
    out[prefix + "n"] = np.int64(g.num_nodes)
    out[prefix + "op"] = np.array([OP_INDEX[nd.op_type] for nd in g.nodes], np.int64)
    out[prefix + "flops"] = np.array([nd.flops for nd in g.nodes], np.float64)
    out[prefix + "out_bytes"] = np.array([nd.output_bytes for nd in g.nodes], np.float64)
    out[prefix + "coloc"] = np.array(coloc, np.int64)
    out[prefix + "src"] = np.array([e.src for e in g.edges], np.int64)
    out[prefix + "dst"] = np.array([e.dst for e in g.edges], np.int64)
    out[prefix + "ebytes"] = np.array([e.bytes for e in g.edges], np.float64)
    out[prefix + "topo"] = np.array(g.topo_order(), np.int64)


def randomize(store, seed=1):
    rng = np.random.default_rng(seed)
    for name in store.names():
        t = store[name]
        if not np.any(t.data):
            s = 1.0 / np.sqrt(max(1, t.data.shape[0]))
            t.data = rng.uniform(-s, s, size=t.data.shape)


def checksums(store):
    names = store.names()
    return (np.array(names), np.array([store[n].data.sum() for n in names]),
            np.array([(store[n].data ** 2).sum() for n in names]))


def topo_arrays(top, prefix, out):
    d = top.num_devices
    out[prefix + "top_peak"] = np.array([top.device(i).peak_flops for i in range(d)])
    out[prefix + "top_mem_bw"] = np.array([top.device(i).mem_bw for i in range(d)])
    out[prefix + "top_cap"] = np.array([top.device(i).mem_capacity for i in range(d)])
    lb = np.zeros((d, d))
    for i in range(d):
        for j in range(d):
            if i != j:
                lb[i, j] = top.link(i, j).bandwidth
    out[prefix + "top_link_bw"] = lb


# ------------------------------------------------------------------------------------------
def make_rng():
    out = {}
    rows = []
    for leaves in (6, 10, 30, 100, 7501):
        specs = [{"op": "relu", "out_bytes": 4} for _ in range(leaves + 1)]
        g = C.make_graph(specs, [(0, i) for i in range(1, leaves + 1)])
        for seed in (0, 1, 3, 9, 12345, 2**31 - 1):
            for k in (1, 3, 5):
                pick = sample_neighbors(g, 0, k, seed)
                rows.append([leaves, seed, k] + pick + [-1] * (5 - len(pick)))
    out["star_picks"] = np.array(rows, np.int64)
    us = []
    for seed in (0, 7, 2**31 - 1):
        r = np.random.default_rng(seed).random(3000)
        for idx in (0, 1, 2, 100, 1999, 2999):
            us.append([seed, idx, r[idx]])
    out["uniforms"] = np.array(us, np.float64)
    np.savez_compressed(OUT / "golden_rng.npz", **out)


FORWARD_CASES = [
    # name, graph builder, ecfg, pcfg, sizes, embed seed, decision seed
    ("tiny", lambda: C.random_graph(np.random.default_rng(0), 6, p_edge=0.4),
     EmbedConfig(1, 8, 4), PolicyConfig(2, 8, 2, 3, 16, 4, 2),
     {"placement": 3, "schedule_priority": 4, "fusion_priority": 4}, 0, 9),
    ("small", lambda: C.random_graph(np.random.default_rng(5), 13, p_edge=0.3),
     EmbedConfig(2, 8, 3), PolicyConfig(2, 8, 2, 3, 16, 4, 2), {"placement": 3}, 11, 4),
    ("default70", lambda: C.random_graph(np.random.default_rng(1), 70, p_edge=0.1),
     EmbedConfig(), PolicyConfig(), {"placement": 4, "schedule_priority": 8,
                                    "fusion_priority": 8}, 3, 21),
    ("cfg1", lambda: gen_workload(WorkloadSpec("attention-stack", 10, 1, 64, seed=0)),
     EmbedConfig(), PolicyConfig(), {"placement": 2}, 5, 17),
    ("dilated", lambda: gen_workload(WorkloadSpec("dilated-stack", 2, 50, 64, seed=3)),
     EmbedConfig(), PolicyConfig(), {"placement": 8}, 8, 33),
]


def make_forward():
    out = {}
    meta = []
    for name, build, ecfg, pcfg, sizes, eseed, dseed in FORWARD_CASES:
        g = build()
        p = name + "/"
        graph_arrays(g, p, out)
        store = init_all_params(ecfg, pcfg, sizes, seed=0)
        randomize(store)
        nm, s1, s2 = checksums(store)
        out[p + "param_names"], out[p + "param_sum"], out[p + "param_sq"] = nm, s1, s2
        tasks = ordered_tasks(sizes)
        feats = node_features(g, None, [a for _, a in tasks])
        gather, seg = _neighbor_arrays(g, ecfg.gs_knn, eseed)
        emb = embed(g, feats, store, ecfg, seed=eseed)
        hid = trunk_forward(emb.node_embed, emb.graph_embed, store, pcfg)
        heads = task_heads(hid, store, pcfg, tasks)
        out[p + "feats"] = feats
        out[p + "gather"], out[p + "seg"] = gather, seg
        out[p + "node_embed"] = emb.node_embed.data
        out[p + "graph_embed"] = emb.graph_embed.data
        out[p + "hid"] = hid.data
        for t, _a in tasks:
            out[p + f"logits/{t}"] = heads.logits[t].data
        out[p + "value"] = heads.value.data
        bundle, traj = iterate_decisions(g, store, ecfg, pcfg, sizes, pcfg.iterations, dseed)
        for it, b in enumerate(traj):
            for t, _a in tasks:
                out[p + f"it{it}/actions/{t}"] = b.actions[t]
                out[p + f"it{it}/logp/{t}"] = b.log_probs[t]
                out[p + f"it{it}/logits/{t}"] = b.logits[t]
            out[p + f"it{it}/value"] = np.float64(b.value)
        meta.append(dict(name=name, ecfg=ecfg.__dict__, pcfg=pcfg.__dict__, sizes=sizes,
                         embed_seed=eseed, decision_seed=dseed))
    out["meta"] = np.array(json.dumps(meta))
    np.savez_compressed(OUT / "golden_forward.npz", **out)


def rand_topology(rng, d, tight=False):
    devs = [DeviceSpec(i, float(rng.choice([1e9, 2e9, 1e12])), float(rng.choice([1e10, 1e11])),
                       float(rng.choice([1e3, 1e12]) if tight else 1e12)) for i in range(d)]
    top = DeviceTopology(devs, uniform_bandwidth=float(rng.choice([1e9, 1e10])))
    return top


def make_des():
    out = {}
    rng = np.random.default_rng(2024)
    cases = 0

    def record(g, fg_map, top, placement, pri, policy, tag):
        nonlocal cases
        p = f"c{cases}/"
        graph_arrays(g, p, out)
        topo_arrays(top, p, out)
        fg = FusedGraph(g, fg_map)
        res = simulate(fg, ActionAssignment("placement", placement, top.num_devices),
                       ActionAssignment("schedule_priority", pri, 8), top, policy=policy)
        out[p + "group_map"] = np.asarray(fg_map, np.int64)
        out[p + "placement"] = np.asarray(placement, np.int64)
        out[p + "priorities"] = np.asarray(pri, np.int64)
        out[p + "policy"] = np.array(policy)
        out[p + "tag"] = np.array(tag)
        out[p + "step_time"] = np.float64(res.step_time)
        out[p + "valid"] = np.bool_(res.valid)
        out[p + "violation"] = np.array(res.violation or "")
        out[p + "busy"] = np.array(res.per_device_busy, np.float64)
        out[p + "peak"] = np.array(res.peak_mem, np.float64)
        cases += 1

    # random small graphs, random placements / priorities, both policies
    for _ in range(120):
        n = int(rng.integers(1, 40))
        g = C.random_graph(rng, n, p_edge=float(rng.choice([0.05, 0.2, 0.5])))
        d = int(rng.integers(1, 5))
        top = rand_topology(rng, d, tight=bool(rng.random() < 0.3))
        placement = rng.integers(0, d, n)
        pri = rng.integers(0, 8, n) if rng.random() < 0.7 else np.zeros(n, np.int64)
        policy = "priority" if rng.random() < 0.7 else "fifo"
        record(g, np.arange(n), top, placement, pri, policy, "random")
    # colocation (hand-built) and fused groupings from the reference fusion pass
    for _ in range(30):
        n = int(rng.integers(2, 30))
        g = C.random_graph(rng, n, p_edge=0.3, fusible_only=True)
        pri_f = rng.integers(0, 8, n)
        fg = apply_fusion(g, ActionAssignment("fusion_priority", pri_f, 8), FusionConfig())
        top = rand_topology(rng, 3)
        record(g, fg.group_map, top, rng.integers(0, 3, n), rng.integers(0, 8, n),
               "priority", "fused")
    specs = [{"op": "relu", "flops": 1e9, "out_bytes": 8, "colocate": "g"},
             {"op": "relu", "flops": 1e9, "out_bytes": 8, "colocate": "g"},
             {"op": "relu", "flops": 1e9, "out_bytes": 8}]
    g = C.make_graph(specs, [(0, 2)])
    for pl in ([0, 1, 0], [1, 1, 0], [0, 0, 0]):
        record(g, np.arange(3), C.simple_topology(2), np.array(pl), np.zeros(3, np.int64),
               "priority", "coloc")
    g = C.make_graph([{"op": "relu", "out_bytes": 4}] * 3, [(0, 1), (1, 2), (0, 2)])
    record(g, np.array([0, 1, 0]), C.simple_topology(1), np.zeros(3, np.int64),
           np.zeros(3, np.int64), "priority", "cycle")
    # workload-scale graphs: greedy (default pipeline) and random 4/8-way placements
    for spec, d in ((WorkloadSpec("multi-branch-cnn", 200, 1, 64, seed=0), 4),
                    (WorkloadSpec("attention-stack", 100, 1, 64, seed=0), 8),
                    (WorkloadSpec("dilated-stack", 3, 60, 64, seed=1), 8)):
        g = gen_workload(spec, node_cap=10**6)
        from graphopt.costmodel import uniform_topology
        top = uniform_topology(d)
        base = default_assignments(g, top)
        record(g, np.arange(g.num_nodes), top, base["placement"].actions,
               np.zeros(g.num_nodes, np.int64), "priority", "greedy")
        out[f"c{cases - 1}/greedy"] = base["placement"].actions
        for _ in range(2):
            record(g, np.arange(g.num_nodes), top, rng.integers(0, d, g.num_nodes),
                   rng.integers(0, 8, g.num_nodes), "priority", "workload")
    out["count"] = np.int64(cases)
    np.savez_compressed(OUT / "golden_des.npz", **out)


def make_sample():
    out = {}
    rng = np.random.default_rng(99)
    k = 0
    for a in (1, 2, 3, 4, 7, 8, 9, 16):
        for temp in (1.0, 0.5, 0.0, 2.0):
            n = int(rng.integers(1, 300))
            logits = rng.normal(scale=float(rng.choice([0.1, 1.0, 5.0])), size=(n, a))
            if a > 1 and rng.random() < 0.3:
                logits[:, 1] = logits[:, 0]  # ties
            seed = int(rng.integers(2**31))
            r = np.random.default_rng(seed)
            skip = int(rng.integers(0, 3))
            if skip:
                r.random(skip)  # stream offset, as later (iteration, task) draws are
            acts, logp = sample_actions(logits, temp, r)
            p = f"s{k}/"
            out[p + "logits"], out[p + "temp"] = logits, np.float64(temp)
            out[p + "seed"], out[p + "offset"] = np.int64(seed), np.int64(skip)
            out[p + "actions"], out[p + "logp"] = np.asarray(acts, np.int64), logp
            k += 1
    out["count"] = np.int64(k)
    np.savez_compressed(OUT / "golden_sample.npz", **out)


def make_rollouts():
    out = {}
    g = gen_workload(WorkloadSpec("attention-stack", 10, 1, 64, seed=0))
    from graphopt.costmodel import uniform_topology
    top = uniform_topology(2)
    sizes = task_action_sizes(top, ["placement"], 8)
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = init_all_params(ecfg, pcfg, sizes, seed=0)
    randomize(store)
    base = default_assignments(g, top)
    from graphopt.baselines import baseline_step_time
    bl = baseline_step_time(g, top)
    hyper = PPOHyper(rollouts=6)
    batch = collect_rollouts(store, [g], top, sizes, [bl], 6, seed=0, hyper=hyper,
                             embed_cfg=ecfg, policy_cfg=pcfg, fusion_cfg=FusionConfig(),
                             base_assignments=[base])
    graph_arrays(g, "g/", out)
    out["baseline"] = np.float64(bl)
    for i, s in enumerate(batch.samples):
        p = f"r{i}/"
        out[p + "graph_index"] = np.int64(s.graph_index)
        out[p + "reward"] = np.float64(s.reward)
        out[p + "value"] = np.float64(s.value_estimate)
        out[p + "advantage"] = np.float64(s.advantage)
        out[p + "step_time"] = np.float64(s.step_time)
        out[p + "valid"] = np.bool_(s.valid)
        out[p + "actions"] = s.bundle.actions["placement"]
        out[p + "prev_actions"] = s.bundle.prev_actions["placement"]
        out[p + "logp"] = s.bundle.log_probs["placement"]
        out[p + "embed_seed"] = np.int64(s.bundle.embed_seed)
    out["count"] = np.int64(len(batch.samples))
    np.savez_compressed(OUT / "golden_rollouts.npz", **out)


def make_ppo(iterations=2, name="golden_ppo.npz"):
    out = {}
    ecfg = EmbedConfig(1, 8, 4)
    pcfg = PolicyConfig(1, 8, 2, 3, 16, 8, iterations)
    g = C.random_graph(np.random.default_rng(3), 12, p_edge=0.3)
    top = C.simple_topology(2)
    sizes = task_action_sizes(top, ["placement"], 8)
    store = init_all_params(ecfg, pcfg, sizes, seed=0)
    randomize(store)
    from graphopt.baselines import baseline_step_time
    bl = baseline_step_time(g, top)
    hyper = PPOHyper(lr=1e-2, rollouts=4, minibatches=2, epochs=2, entropy_coef=0.01)
    batch = collect_rollouts(store, [g], top, sizes, [bl], 4, seed=5, hyper=hyper,
                             embed_cfg=ecfg, policy_cfg=pcfg, fusion_cfg=FusionConfig())
    graph_arrays(g, "g/", out)
    before = {n: store[n].data.copy() for n in store.names()}
    stats = ppo_update(batch, store, [g], top, sizes, hyper, ecfg, pcfg, seed=7)
    for n in store.names():
        out["before/" + n] = before[n]
        out["after/" + n] = store[n].data
    for k, v in stats.items():
        out["stats/" + k] = np.float64(v)
    for i, s in enumerate(batch.samples):
        p = f"r{i}/"
        out[p + "reward"] = np.float64(s.reward)
        out[p + "advantage"] = np.float64(s.advantage)
        out[p + "actions"] = s.bundle.actions["placement"]
        if s.bundle.prev_actions is not None:
            out[p + "prev_actions"] = s.bundle.prev_actions["placement"]
        out[p + "logp"] = s.bundle.log_probs["placement"]
        out[p + "embed_seed"] = np.int64(s.bundle.embed_seed)
    np.savez_compressed(OUT / name, **out)


def make_ppo1():
    """ppo_update over single-iteration bundles (prev_actions None, training.py:156-158)."""
    make_ppo(iterations=1, name="golden_ppo1.npz")


WORKLOAD_SPECS = [
    ("attention-stack", 10, 1, 64, 0), ("multi-branch-cnn", 1857, 1, 64, 0),
    ("dilated-stack", 30, 250, 64, 0), ("dilated-stack", 10, 250, 64, 1),
    ("dilated-stack", 5, 100, 64, 2), ("dilated-stack", 2, 50, 64, 3),
    ("attention-stack", 8000, 1, 64, 0), ("grid-rnn", 3, 5, 16, 2),
    ("enc-dec-rnn", 2, 4, 32, 1), ("cell-stack-cnn", 6, 1, 32, 4),
]


def make_workloads():
    out = {}
    for i, (fam, L, S, w, seed) in enumerate(WORKLOAD_SPECS):
        g = gen_workload(WorkloadSpec(fam, L, S, w, seed=seed), node_cap=10**6)
        tmp = {}
        graph_arrays(g, "", tmp)
        p = f"w{i}/"
        out[p + "spec"] = np.array([fam, str(L), str(S), str(w), str(seed)])
        out[p + "n"], out[p + "e"] = np.int64(g.num_nodes), np.int64(g.num_edges)
        out[p + "op_sum"] = np.int64(tmp["op"].sum())
        out[p + "flops"] = np.float64(tmp["flops"].sum())
        out[p + "out_bytes"] = np.float64(tmp["out_bytes"].sum())
        out[p + "edge_sig"] = np.int64((tmp["src"] * 1000003 + tmp["dst"]).sum() % (2**61 - 1))
        out[p + "ebytes"] = np.float64(tmp["ebytes"].sum())
        out[p + "topo_sig"] = np.int64((tmp["topo"] * np.arange(g.num_nodes)).sum() % (2**61 - 1))
    out["count"] = np.int64(len(WORKLOAD_SPECS))
    np.savez_compressed(OUT / "golden_workloads.npz", **out)


def make_grads():
    """Per-sample PPO loss and its full parameter gradient from the reference tape
    (training.py:146-186 _sample_loss + tensor.py backward)."""
    import graphopt.training as tr
    out = {}
    cases = [
        ("small", EmbedConfig(1, 8, 4), PolicyConfig(1, 8, 2, 3, 16, 8, 2),
         lambda: C.random_graph(np.random.default_rng(3), 12, p_edge=0.3), 2, np.float64),
        ("joint", EmbedConfig(2, 8, 3), PolicyConfig(2, 8, 2, 3, 16, 4, 2),
         lambda: C.random_graph(np.random.default_rng(8), 15, p_edge=0.3), 3, np.float64),
        ("default", EmbedConfig(), PolicyConfig(),
         lambda: C.random_graph(np.random.default_rng(4), 100, p_edge=0.05), 4, np.float32),
    ]
    for name, ecfg, pcfg, build, d, dt in cases:
        g = build()
        top = C.simple_topology(d)
        tasks = ["placement"] if name != "joint" else ["placement", "schedule_priority",
                                                      "fusion_priority"]
        sizes = task_action_sizes(top, tasks, 8)
        store = init_all_params(ecfg, pcfg, sizes, seed=0)
        randomize(store)
        from graphopt.baselines import baseline_step_time
        bl = baseline_step_time(g, top)
        hyper = PPOHyper(lr=1e-2, rollouts=3, minibatches=1, epochs=1, entropy_coef=0.3,
                         temperature=0.8 if name == "joint" else 1.0)
        batch = collect_rollouts(store, [g], top, sizes, [bl], 3, seed=11, hyper=hyper,
                                 embed_cfg=ecfg, policy_cfg=pcfg, fusion_cfg=FusionConfig())
        p = name + "/"
        graph_arrays(g, p + "g/", out)
        out[p + "meta"] = np.array(json.dumps(dict(ecfg=ecfg.__dict__, pcfg=pcfg.__dict__,
                                                   sizes=sizes, d=d, hyper=hyper.__dict__)))
        for i, s in enumerate(batch.samples):
            q = p + f"s{i}/"
            for t in tasks:
                out[q + f"actions/{t}"] = s.bundle.actions[t]
                out[q + f"prev/{t}"] = s.bundle.prev_actions[t]
                out[q + f"logp/{t}"] = s.bundle.log_probs[t]
            out[q + "embed_seed"] = np.int64(s.bundle.embed_seed)
            out[q + "reward"] = np.float64(s.reward)
            out[q + "temperature"] = np.float64(s.bundle.temperature)
            adv = 0.7 - 0.9 * i
            out[q + "adv"] = np.float64(adv)
            store.zero_grads()
            stats = {"ratio_sum": 0.0, "clip_sum": 0.0, "node_count": 0, "entropy_sum": 0.0,
                     "entropy_count": 0, "value_loss_sum": 0.0, "value_count": 0}
            loss = tr._sample_loss(s, adv, g, store, sizes, hyper, ecfg, pcfg, stats)
            loss.backward()
            out[q + "loss"] = np.float64(loss.data)
            for k, v in stats.items():
                out[q + "stats/" + k] = np.float64(v)
            if name == "default" and i > 0:
                continue  # keep the fixture small: one full fp32 gradient at 1.2M params
            for n_ in store.names():
                gr = store[n_].grad
                out[q + "grad/" + n_] = (np.zeros_like(store[n_].data) if gr is None
                                         else gr).astype(dt)
    np.savez_compressed(OUT / "golden_grads.npz", **out)


def make_json():
    """JSON graph / topology loader cases (graph.py:208-260, costmodel.py:110-128):
    documents that parse (arrays of the reference's parse) and documents it rejects."""
    import json as _json
    from graphopt.costmodel import topology_from_dict
    from graphopt.graph import GraphError, from_dict
    docs = [
        {"name": "tiny", "nodes": [{"id": 0, "op": "matmul", "flops": 1e9, "out_bytes": 64},
                                   {"id": 1, "op": "relu", "shape": [4, 4], "out_bytes": 64},
                                   {"id": 2, "op": "mystery-op", "flops": 5, "colocate": "a"},
                                   {"id": 3, "op": "concat", "colocate": "a"}],
         "edges": [{"src": 0, "dst": 1}, {"src": 1, "dst": 2, "bytes": 7},
                   {"src": 0, "dst": 3}, {"src": 2, "dst": 3}, {"src": 0, "dst": 3}]},
        {"nodes": [{"id": i, "op": "conv", "flops": float(i)} for i in range(5)],
         "edges": [{"src": i, "dst": i + 1} for i in range(4)]},
        {"nodes": [], "edges": []},
        {"nodes": [{"id": 0, "op": "relu"}], "bogus": 1},
        {"nodes": [{"id": 0, "op": "relu", "extra": 2}]},
        {"nodes": [{"id": 1, "op": "relu"}]},
        {"nodes": [{"id": 0, "op": "relu"}, {"id": 0, "op": "relu"}]},
        {"nodes": [{"id": 1, "op": "relu"}, {"id": 0, "op": "relu"}]},
        {"nodes": [{"id": 0, "op": "relu"}], "edges": [{"src": 0, "dst": 4}]},
        {"nodes": [{"id": 0, "op": "relu"}, {"id": 1, "op": "relu"}],
         "edges": [{"src": 0, "dst": 1}, {"src": 1, "dst": 0}]},
        {"nodes": [{"id": 0, "op": "relu", "shape": [2], "out_bytes": 9}]},
        {"nodes": [{"id": 0, "op": "relu", "flops": -1}]},
        {"nodes": [{"op": "relu"}]},
    ]
    out = {}
    for i, doc in enumerate(docs):
        p = f"j{i}/"
        out[p + "doc"] = np.array(_json.dumps(doc))
        try:
            g = from_dict(doc, name="x")
            graph_arrays(g, p, out)
            out[p + "gname"] = np.array(g.name)
            out[p + "ok"] = np.bool_(True)
        except GraphError:
            out[p + "ok"] = np.bool_(False)
    out["json_count"] = np.int64(len(docs))
    tops = [{"devices": [{"id": 1, "peak_flops": 2e12, "mem_bw": 1e11, "mem_capacity": 8e9},
                         {"id": 0, "peak_flops": 1e12, "mem_bw": 2e11, "mem_capacity": 16e9}],
             "links": {"uniform_bandwidth": 5e9}},
            {"devices": [{"id": 0, "peak_flops": 1e12, "mem_bw": 1e11, "mem_capacity": 1e9},
                         {"id": 1, "peak_flops": 1e12, "mem_bw": 1e11, "mem_capacity": 1e9}],
             "links": [{"src": 0, "dst": 1, "bandwidth": 1e9}, {"src": 1, "dst": 0, "bandwidth": 3e9}]},
            {"devices": [{"id": 0, "peak_flops": 1e12, "mem_bw": 1e11, "mem_capacity": 1e9},
                         {"id": 1, "peak_flops": 1e12, "mem_bw": 1e11, "mem_capacity": 1e9}],
             "links": [{"src": 0, "dst": 1, "bandwidth": 1e9}]}]
    for i, doc in enumerate(tops):
        p = f"t{i}/"
        out[p + "doc"] = np.array(_json.dumps(doc))
        try:
            topo_arrays(topology_from_dict(doc), p, out)
            out[p + "ok"] = np.bool_(True)
        except ValueError:
            out[p + "ok"] = np.bool_(False)
    out["top_count"] = np.int64(len(tops))
    np.savez_compressed(OUT / "golden_json.npz", **out)


def make_rollouts_joint():
    """collect_rollouts with the joint task set (placement + schedule + fusion priorities)
    on a graph where fusion merges happen, so every rollout has its own fused grouping."""
    out = {}
    g = gen_workload(WorkloadSpec("multi-branch-cnn", 6, 1, 64, seed=1))
    from graphopt.costmodel import uniform_topology
    top = uniform_topology(3)
    tasks = ["placement", "schedule_priority", "fusion_priority"]
    sizes = task_action_sizes(top, tasks, 8)
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = init_all_params(ecfg, pcfg, sizes, seed=0)
    randomize(store)
    base = default_assignments(g, top)
    from graphopt.baselines import baseline_step_time
    bl = baseline_step_time(g, top)
    batch = collect_rollouts(store, [g], top, sizes, [bl], 8, seed=4, hyper=PPOHyper(rollouts=8),
                             embed_cfg=ecfg, policy_cfg=pcfg, fusion_cfg=FusionConfig(),
                             base_assignments=[base])
    graph_arrays(g, "g/", out)
    out["baseline"] = np.float64(bl)
    groups = set()
    for i, s in enumerate(batch.samples):
        p = f"r{i}/"
        out[p + "reward"] = np.float64(s.reward)
        out[p + "step_time"] = np.float64(s.step_time)
        out[p + "valid"] = np.bool_(s.valid)
        for t in tasks:
            out[p + "actions/" + t] = s.bundle.actions[t]
        fg = apply_fusion(g, ActionAssignment("fusion_priority", s.bundle.actions["fusion_priority"], 8),
                          FusionConfig())
        groups.add(tuple(fg.group_map))
    out["count"] = np.int64(len(batch.samples))
    out["distinct_groupings"] = np.int64(len(groups))
    np.savez_compressed(OUT / "golden_rollouts_joint.npz", **out)


def make_baselines():
    """Non-learned optimizers (baselines.py:50-237): fanout priorities, brute force over
    placement / schedule / fusion priorities, simulated annealing chains."""
    from graphopt.baselines import SAConfig, brute_force, fanout_priorities, simulated_annealing
    out = {}
    rng = np.random.default_rng(77)
    # fanout priorities
    graphs = [C.random_graph(rng, int(rng.integers(2, 40)), p_edge=float(p))
              for p in (0.05, 0.2, 0.5, 0.3, 0.1)]
    graphs.append(gen_workload(WorkloadSpec("multi-branch-cnn", 40, 1, 64, seed=3), node_cap=10**6))
    for i, g in enumerate(graphs):
        p = f"f{i}/"
        graph_arrays(g, p, out)
        out[p + "levels"] = fanout_priorities(g).actions
    out["fanout_count"] = np.int64(len(graphs))
    # brute force
    cases = [("placement", 6, 2), ("placement", 5, 3), ("placement", 7, 2),
             ("schedule_priority", 4, 8), ("placement", 8, 2), ("fusion_priority", 3, 8)]
    for i, (task, n, d) in enumerate(cases):
        p = f"b{i}/"
        g = C.random_graph(rng, n, p_edge=0.4, fusible_only=task == "fusion_priority")
        top = rand_topology(rng, d if task == "placement" else 2)
        best, t = brute_force(g, top, task)
        graph_arrays(g, p, out)
        topo_arrays(top, p, out)
        out[p + "task"] = np.array(task)
        out[p + "actions"] = best.actions
        out[p + "time"] = np.float64(t)
    out["brute_count"] = np.int64(len(cases))
    # simulated annealing
    sa_cases = [(["placement"], 25, 3, 0), (["placement", "schedule_priority"], 20, 2, 5),
                (["schedule_priority"], 15, 2, 9), (["fusion_priority", "placement"], 12, 2, 3)]
    for i, (tasks, n, d, seed) in enumerate(sa_cases):
        p = f"a{i}/"
        g = C.random_graph(rng, n, p_edge=0.3, fusible_only="fusion_priority" in tasks)
        top = rand_topology(rng, d)
        res, t = simulated_annealing(g, top, tasks, SAConfig(iterations=300, seed=seed,
                                                             cooling_rate=0.99))
        graph_arrays(g, p, out)
        topo_arrays(top, p, out)
        out[p + "tasks"] = np.array(tasks)
        out[p + "seed"] = np.int64(seed)
        out[p + "time"] = np.float64(t)
        for tk in tasks:
            out[p + "actions/" + tk] = res[tk].actions
    out["sa_count"] = np.int64(len(sa_cases))
    np.savez_compressed(OUT / "golden_baselines.npz", **out)


def make_train():
    """reference train() (training.py:251-317) for 3 steps on a 12-node graph, plus
    decode_step_time on the result and a save_state-free checkpoint round trip."""
    from graphopt.costmodel import uniform_topology
    from graphopt.training import decode_step_time, train
    out = {}
    ecfg = EmbedConfig(1, 8, 4)
    pcfg = PolicyConfig(1, 8, 2, 3, 16, 8, 2)
    g = C.random_graph(np.random.default_rng(3), 12, p_edge=0.3)
    top = uniform_topology(2)
    hyper = PPOHyper(lr=1e-2, rollouts=6, minibatches=2, epochs=2, entropy_coef=0.01)
    res = train([g], top, ["placement"], hyper, 3, 11, ecfg, pcfg, FusionConfig())
    graph_arrays(g, "g/", out)
    out["baselines"] = np.array(res.baselines, np.float64)
    out["best_step_times"] = np.array(res.best_step_times, np.float64)
    out["curve"] = np.array([c for _, c in res.curve], np.float64)
    out["has_best_actions"] = np.bool_(res.best_actions[0] is not None)
    if res.best_actions[0] is not None:
        out["best_actions"] = res.best_actions[0]["placement"]
    for i, st in enumerate(res.stats_history):
        for k, v in st.items():
            out[f"stats{i}/{k}"] = np.float64(v)
    for n in res.store.names():
        out["store/" + n] = res.store[n].data
        out["best/" + n] = res.best_store[n].data
    out["step_count"] = np.int64(res.store.step_count)
    out["decode"] = np.float64(decode_step_time(g, res.store, top, ["placement"], ecfg, pcfg,
                                                FusionConfig()))
    np.savez_compressed(OUT / "golden_train.npz", **out)


def make_fusion():
    """apply_fusion group maps (simulator.py:199-277) with the priorities and
    max_group that produced them: random DAGs (fusible-only and mixed ops, some
    priorities 0), the same DAGs with permuted (non-topological) node ids, and
    workload-family graphs.  The canonical FusedGraph.group_map is stored."""
    from graphopt.simulator import ActionAssignment as AA
    out = {}
    rng = np.random.default_rng(2024)
    cases = []
    for i in range(60):
        n = int(rng.integers(2, 41))
        g = C.random_graph(rng, n, p_edge=float(rng.choice([0.08, 0.2, 0.35])),
                           fusible_only=bool(i % 2 == 0))
        cases.append(("random", g))
        if i % 3 == 0:  # same structure, node ids permuted (edges no longer id-forward)
            perm = rng.permutation(n)
            specs = [None] * n
            for v, nd in enumerate(g.nodes):
                specs[perm[v]] = {"op": nd.op_type, "flops": nd.flops,
                                  "out_bytes": nd.output_bytes}
            edges = [(int(perm[e.src]), int(perm[e.dst]), e.bytes) for e in g.edges]
            cases.append(("permuted", C.make_graph(specs, edges)))
    for spec in [("attention-stack", 10, 1, 64, 0), ("dilated-stack", 2, 50, 64, 3),
                 ("multi-branch-cnn", 40, 1, 64, 0), ("grid-rnn", 3, 5, 16, 2),
                 ("enc-dec-rnn", 2, 4, 32, 1), ("cell-stack-cnn", 6, 1, 32, 4)]:
        cases.append(("workload", gen_workload(WorkloadSpec(*spec))))
    merged_any = 0
    for c, (tag, g) in enumerate(cases):
        n = g.num_nodes
        pri = rng.integers(0, 8, n)
        if c % 4 == 1:
            pri[rng.random(n) < 0.3] = 0
        mg = int(rng.choice([2, 3, 4, 8]))
        fg = apply_fusion(g, AA("fusion_priority", pri, 8), FusionConfig(max_group=mg))
        p = f"c{c}/"
        graph_arrays(g, p, out)
        out[p + "tag"] = np.array(tag)
        out[p + "pri"] = pri.astype(np.int64)
        out[p + "max_group"] = np.int64(mg)
        out[p + "group_map"] = fg.group_map.astype(np.int64)
        merged_any += int(len(fg.groups) < n)
    out["count"] = np.int64(len(cases))
    out["merged_cases"] = np.int64(merged_any)
    np.savez_compressed(OUT / "golden_fusion.npz", **out)


def make_trace():
    """simulate(record_trace=True) event logs (simulator.py:61-67, 360-373, 432-433):
    random graphs and placements (both policies, tight memory), fused groupings, a
    colocation violation, a cycle after fusion and a workload-scale graph."""
    out = {}
    rng = np.random.default_rng(77)
    cases = 0

    def record(g, fg_map, top, placement, pri, policy, tag):
        nonlocal cases
        p = f"c{cases}/"
        graph_arrays(g, p, out)
        topo_arrays(top, p, out)
        fg = FusedGraph(g, fg_map)
        res = simulate(fg, ActionAssignment("placement", placement, top.num_devices),
                       ActionAssignment("schedule_priority", pri, 8), top, policy=policy,
                       record_trace=True)
        out[p + "group_map"] = np.asarray(fg_map, np.int64)
        out[p + "placement"] = np.asarray(placement, np.int64)
        out[p + "priorities"] = np.asarray(pri, np.int64)
        out[p + "policy"] = np.array(policy)
        out[p + "tag"] = np.array(tag)
        out[p + "step_time"] = np.float64(res.step_time)
        tr = res.trace
        out[p + "t_start"] = np.array([e.time_start for e in tr], np.float64)
        out[p + "t_end"] = np.array([e.time_end for e in tr], np.float64)
        out[p + "device"] = np.array([e.device for e in tr], dtype="U16")
        out[p + "kind"] = np.array([e.kind for e in tr], dtype="U16")
        out[p + "group"] = np.array([e.group_id for e in tr], np.int64)
        cases += 1

    for _ in range(40):
        n = int(rng.integers(1, 40))
        g = C.random_graph(rng, n, p_edge=float(rng.choice([0.05, 0.2, 0.5])))
        d = int(rng.integers(1, 12))  # >= 10 devices: "10" sorts before "2"
        top = rand_topology(rng, d, tight=bool(rng.random() < 0.3))
        record(g, np.arange(n), top, rng.integers(0, d, n),
               rng.integers(0, 8, n) if rng.random() < 0.7 else np.zeros(n, np.int64),
               "priority" if rng.random() < 0.7 else "fifo", "random")
    for _ in range(10):
        n = int(rng.integers(2, 30))
        g = C.random_graph(rng, n, p_edge=0.3, fusible_only=True)
        fg = apply_fusion(g, ActionAssignment("fusion_priority", rng.integers(0, 8, n), 8),
                          FusionConfig())
        record(g, fg.group_map, rand_topology(rng, 3), rng.integers(0, 3, n),
               rng.integers(0, 8, n), "priority", "fused")
    specs = [{"op": "relu", "flops": 1e9, "out_bytes": 8, "colocate": "g"},
             {"op": "relu", "flops": 1e9, "out_bytes": 8, "colocate": "g"},
             {"op": "relu", "flops": 1e9, "out_bytes": 8}]
    record(C.make_graph(specs, [(0, 2)]), np.arange(3), C.simple_topology(2), np.array([0, 1, 0]),
           np.zeros(3, np.int64), "priority", "coloc")
    g = C.make_graph([{"op": "relu", "out_bytes": 4}] * 3, [(0, 1), (1, 2), (0, 2)])
    record(g, np.array([0, 1, 0]), C.simple_topology(1), np.zeros(3, np.int64),
           np.zeros(3, np.int64), "priority", "cycle")
    from graphopt.costmodel import uniform_topology
    g = gen_workload(WorkloadSpec("dilated-stack", 3, 60, 64, seed=1), node_cap=10**6)
    record(g, np.arange(g.num_nodes), uniform_topology(8), rng.integers(0, 8, g.num_nodes),
           rng.integers(0, 8, g.num_nodes), "priority", "workload")
    out["count"] = np.int64(cases)
    np.savez_compressed(OUT / "golden_trace.npz", **out)


def perturb_a(seg_index, layer, arr):  # the reference test's hook (test_policy.py:140-143)
    return arr + 0.5 if (seg_index == 1 and layer == 0) else arr


def perturb_b(seg_index, layer, arr):  # every segment and layer, position dependent
    return arr * (1.0 - 0.05 * layer) + 0.01 * seg_index


def make_perturb():
    """trunk_forward(cache_perturb=...) (policy.py:137, 170-172) from the reference on the
    reference tests' small configuration and on the default network (segment_len 64,
    150 rows), with the parameters' init seed and the node / graph embeddings stored."""
    from graphopt.tensor import Tensor
    out = {}
    rng = np.random.default_rng(99)
    cases = [("small", EmbedConfig(gs_layers=1, gs_dim=8, gs_knn=4),
              PolicyConfig(trf_layers=2, d_model=8, n_head=2, d_head=3, d_inner=16,
                           segment_len=4, iterations=2), 12),
             ("default", EmbedConfig(), PolicyConfig(), 150)]
    for name, ecfg, pcfg, n in cases:
        store = init_all_params(ecfg, pcfg, {"placement": 3}, seed=0)
        randomize(store)
        ne = rng.normal(size=(n, ecfg.gs_dim))
        ge = rng.normal(size=(1, ecfg.gs_dim)) * 0.1
        p = name + "/"
        out[p + "meta"] = np.array(json.dumps({"ecfg": ecfg.__dict__, "pcfg": pcfg.__dict__}))
        out[p + "node_embed"] = ne
        out[p + "graph_embed"] = ge
        out[p + "base"] = trunk_forward(Tensor(ne), Tensor(ge), store, pcfg).data
        for tag, fn in (("a", perturb_a), ("b", perturb_b)):
            out[p + tag] = trunk_forward(Tensor(ne), Tensor(ge), store, pcfg,
                                         cache_perturb=fn).data
    np.savez_compressed(OUT / "golden_perturb.npz", **out)


def make_sa_chains():
    """simulated_annealing (baselines.py:146-206) for 8 seeds per case, so the device's
    multi-chain annealing can be checked chain by chain: a 40-node multi-branch CNN on
    4 devices (placement), a random DAG annealing placement + schedule priorities with
    2 moves per step and a fixed initial temperature, and a fusion case."""
    from graphopt.baselines import SAConfig, simulated_annealing
    from graphopt.costmodel import uniform_topology
    out = {}
    rng = np.random.default_rng(31)
    cases = [("mbc", gen_workload(WorkloadSpec("multi-branch-cnn", 5, 1, 64, seed=0)),
              uniform_topology(4), ["placement"], dict(iterations=800, cooling_rate=0.995)),
             ("rand", C.random_graph(rng, 30, p_edge=0.25), rand_topology(rng, 3),
              ["schedule_priority", "placement"],
              dict(iterations=500, cooling_rate=0.99, moves_per_step=2,
                   initial_temperature=2e-4)),
             ("fuse", C.random_graph(rng, 14, p_edge=0.3, fusible_only=True),
              rand_topology(rng, 2), ["fusion_priority", "placement"],
              dict(iterations=150, cooling_rate=0.99))]
    for name, g, top, tasks, kw in cases:
        p = name + "/"
        graph_arrays(g, p, out)
        topo_arrays(top, p, out)
        out[p + "tasks"] = np.array(tasks)
        out[p + "sa"] = np.array(json.dumps(kw))
        for seed in range(8):
            res, t = simulated_annealing(g, top, tasks, SAConfig(seed=seed, **kw))
            out[p + f"s{seed}/time"] = np.float64(t)
            for tk in tasks:
                out[p + f"s{seed}/{tk}"] = res[tk].actions
    np.savez_compressed(OUT / "golden_sa_chains.npz", **out)


def make_cfg2():
    """The UNMODIFIED reference at BASELINE cfg2 (multi-branch-cnn, 13,000 nodes, 4
    devices, default networks; its tape holds ~15 GB for the heads): iterate_decisions
    with 2 iterations, then the DES.  Stored compactly -- per-row logit sums of both
    iterations, logits of 512 seeded rows, both iterations' actions, embedding row
    sums, the value and the step time -- so the oracle (and through it the device
    path, tests/test_gpu_headline.py) is pinned to the reference at a headline size,
    not only on the small fixtures."""
    from graphopt.costmodel import uniform_topology
    out = {}
    g = gen_workload(WorkloadSpec("multi-branch-cnn", 1857, 1, 64, seed=0), node_cap=10**6)
    top = uniform_topology(4)
    sizes = {"placement": 4}
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = init_all_params(ecfg, pcfg, sizes, seed=0)
    randomize(store)
    rows = np.sort(np.random.default_rng(5).choice(g.num_nodes, 512, replace=False))
    feats = node_features(g, None, [4])
    emb = embed(g, feats, store, ecfg, seed=77)
    out["node_embed_rowsum"] = emb.node_embed.data.sum(axis=1)
    out["graph_embed"] = emb.graph_embed.data
    bundle, traj = iterate_decisions(g, store, ecfg, pcfg, sizes, 2, 77)
    for it, b in enumerate(traj):
        lg = b.logits["placement"]
        out[f"it{it}/logit_rowsum"] = lg.sum(axis=1)
        out[f"it{it}/logits_rows"] = lg[rows]
        out[f"it{it}/actions"] = b.actions["placement"]
        out[f"it{it}/logp"] = b.log_probs["placement"]
        out[f"it{it}/value"] = np.float64(b.value)
    res = simulate(singleton_fused(g), ActionAssignment("placement", bundle.actions["placement"], 4),
                   ActionAssignment.constant("schedule_priority", g.num_nodes, 8), top)
    out["rows"] = rows
    out["step_time"] = np.float64(res.step_time)
    out["seed"] = np.int64(77)
    np.savez_compressed(OUT / "golden_cfg2.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["rng", "forward", "des", "sample", "rollouts", "ppo", "ppo1", "workloads", "grads",
                             "baselines", "rollouts_joint", "json", "train", "fusion", "trace", "perturb", "sa_chains", "cfg2"]
    for w in which:
        globals()["make_" + w]()
        print("wrote", w)

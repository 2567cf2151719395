"""Parity at the BASELINE configurations against the float64 oracle (SURVEY §8(c)
C3, rows A5-A11 and A15; VERDICT r1 "next" #1).  See tests/headline.py for what is
compared and how flips are explained.

cfg4  attention-stack L=8000 (80,001 nodes), 8 devices: embeddings and trunk output
      in full, head logits on 512 seeded query rows (all 80,001 keys), both
      iterations' actions on those rows, 8 DES placements bit-exact.
cfg2  multi-branch-cnn (13,000 nodes), 4 devices: the whole forward in float64
      (full 13k x 13k heads), every row's actions in both iterations, DES.
cfg3  dilated-stack (30,003 nodes incl. the 7,500-fan-in sink), 8 devices: forward
      on 512 rows, DES bit-exact; and the super-positioned batch (30,003 / 10,003 /
      2,003 / 403-node graphs, graph drawn per rollout) through collect_rollouts.

Bars: normwise relative 1e-4 for embeddings / trunk / logits (BASELINE north_star);
every action flip explained by the logit tolerance; DES bit-exact.
Set GO_PARITY_REPORT_DIR to also write the measured errors as JSON."""
import json
import os

import numpy as np
import pytest

import headline as H

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CFG = {
    "cfg2": (("multi-branch-cnn", 1857, 1, 64, 0), 4, None),
    "cfg3": (("dilated-stack", 30, 250, 64, 0), 8, 512),
    "cfg4": (("attention-stack", 8000, 1, 64, 0), 8, 512),
}


def _graph(spec):
    from synthetic.workloads import WorkloadSpec, gen_workload
    return gen_workload(WorkloadSpec(*spec), node_cap=10**6)


def _report(name, rep):
    d = os.environ.get("GO_PARITY_REPORT_DIR")
    if not d:
        return
    os.makedirs(d, exist_ok=True)
    clean = {k: v for k, v in rep.items() if k != "final_actions"}
    with open(os.path.join(d, f"parity_{name}.json"), "w") as f:
        json.dump(clean, f, indent=1, default=float)


def _assert_stages(rep):
    for k in ("embed", "graph_embed", "trunk_e2e", "trunk_isolated", "logits_e2e",
              "logits_isolated", "value_e2e"):
        if k in rep:
            assert rep[k]["normwise"] < H.NORM_BAR, (k, rep[k])
    for it, r in enumerate(rep["iterations"]):
        assert r["logits_e2e"]["normwise"] < H.NORM_BAR, (it, r["logits_e2e"])
        assert not r["actions"]["unexplained"], (it, r["actions"])
        assert r["actions"]["logp_max_abs_err"] < 1e-3, (it, r["actions"])


@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_forward_actions_des_at_baseline_config(name):
    spec, d, nrows = CFG[name]
    g = _graph(spec)
    n = g.num_nodes
    rows = None if nrows is None else H.sample_rows(n, nrows, seed=1)
    rep = H.forward_and_decisions(g, {"placement": d}, seed=20251019, rows=rows)
    # DES: the two iterations' device placements, the greedy default, random ones
    from paper_2010_12438_b200.baselines import greedy_placement
    rng = np.random.default_rng(7)
    pls = [rep["final_actions"]["placement"], greedy_placement(g, _top(d)).actions]
    pls += [rng.integers(0, d, n) for _ in range(6)]
    ogr = H.oracle_graph(g)
    rep["des"] = H.check_des(g, ogr, np.stack(pls), d)
    if name == "cfg3":  # same graph, priority policy with non-constant priorities
        pri = rng.integers(0, 8, n)
        rep["des_priorities"] = H.check_des(g, ogr, np.stack(pls[:3]), d, priorities=pri)
    _report(name, rep)
    _assert_stages(rep)
    assert not rep["des"]["mismatches"], rep["des"]
    if "des_priorities" in rep:
        assert not rep["des_priorities"]["mismatches"], rep["des_priorities"]


def _top(d):
    from paper_2010_12438_b200.costmodel import uniform_topology
    return uniform_topology(d)


def test_superpositioned_batch_cfg3_through_collect_rollouts():
    """graphs [dilated (30,250) s0, (10,250) s1, (5,100) s2,
    (2,50) s3], graph index drawn per rollout (training.py:122-126).  Each rollout's
    reward inputs (DES step time) are bit-exact against the oracle DES of its own
    actions, and its final-iteration logits on sampled rows match the oracle given
    the rollout's own previous actions and embed seed."""
    from paper_2010_12438_b200 import (EmbedConfig, FusionConfig, PolicyConfig, PPOHyper,
                                       init_all_params, randomize_zero_init)
    from paper_2010_12438_b200.baselines import baseline_step_time
    from paper_2010_12438_b200.training import collect_rollouts
    specs = [("dilated-stack", 30, 250, 64, 0), ("dilated-stack", 10, 250, 64, 1),
             ("dilated-stack", 5, 100, 64, 2), ("dilated-stack", 2, 50, 64, 3)]
    graphs = [_graph(s) for s in specs]
    assert [g.num_nodes for g in graphs] == [30003, 10003, 2003, 403]
    top = _top(8)
    sizes = {"placement": 8}
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
    bls = [baseline_step_time(g, top) for g in graphs]
    batch = collect_rollouts(store, graphs, top, sizes, bls, 12, seed=3, hyper=PPOHyper(),
                             embed_cfg=ecfg, policy_cfg=pcfg, fusion_cfg=FusionConfig())
    P = H.oracle_params(store)
    seen = set()
    rep = {"rollouts": []}
    for k, s in enumerate(batch.samples):
        g = graphs[s.graph_index]
        ogr = H.oracle_graph(g)
        w = H.od.simulate(ogr, H.od.singleton(ogr), s.bundle.actions["placement"],
                          np.zeros(g.num_nodes, np.int64), H.od.uniform_topology(8))
        r = {"graph": s.graph_index, "step_time": s.step_time, "want": w["step_time"]}
        assert s.step_time == w["step_time"] and s.valid == w["valid"], r
        want_reward = H.od.reward(w["step_time"], bls[s.graph_index], w["valid"])
        assert s.reward == want_reward, (s.reward, want_reward)
        if s.graph_index not in seen:  # logits once per distinct graph
            seen.add(s.graph_index)
            rows = H.sample_rows(g.num_nodes, 256, seed=k)
            lg, _ = H.oracle_logits(ogr, P, sizes, s.bundle.prev_actions, s.bundle.embed_seed,
                                    rows)
            e = H.errors(s.bundle.logits["placement"][rows], lg["placement"])
            r["logits"] = e
            assert e["normwise"] < H.NORM_BAR, (k, e)
        rep["rollouts"].append(r)
    assert len(seen) >= 3
    _report("cfg3_batch", rep)


def test_joint_tasks_at_13k_nodes():
    """cfg5's joint placement + scheduling + fusion heads (three chained task heads, each a
    full N x N attention; policy.py:187-217) on the 13,000-node cfg2 graph, both
    iterations, every row and task against the float64 oracle: logits 1e-4 normwise, every
    action flip explained; then the joint assignment through the fusion pass and the
    priority DES (evaluate_assignments, simulator.py:472-487) bit-exact against the
    oracle's apply_fusion + simulate."""
    from oracle import forward as of
    from paper_2010_12438_b200 import EmbedConfig, PolicyConfig, init_all_params, randomize_zero_init
    from paper_2010_12438_b200.costmodel import uniform_topology
    from paper_2010_12438_b200.policy import iterate_decisions
    from paper_2010_12438_b200.simulator import ActionAssignment, evaluate_assignments
    g = _graph(("multi-branch-cnn", 1857, 1, 64, 0))
    sizes = {"placement": 4, "schedule_priority": 8, "fusion_priority": 8}
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
    P = H.oracle_params(store)
    ogr = H.oracle_graph(g)
    seed = 4242
    bundle, traj = iterate_decisions(g, store, ecfg, pcfg, sizes, 2, seed)
    order = np.asarray(g.topo_order())
    tasks = of.ordered_tasks(sizes)
    rep = {"iterations": []}
    prev = None
    for it, b in enumerate(traj):
        lg_ref, _ = H.oracle_logits(ogr, P, sizes, prev, seed)
        r = {}
        for t_i, (t, _a) in enumerate(tasks):
            e = H.errors(b.logits[t], lg_ref[t])
            acts = H.check_actions(b.actions[t], b.log_probs[t], lg_ref[t], b.logits[t], order,
                                   np.arange(g.num_nodes), seed, it, t_i, len(tasks))
            r[t] = {"logits": e, "actions": acts}
            assert e["normwise"] < H.NORM_BAR, (it, t, e)
            assert not acts["unexplained"], (it, t, acts)
        rep["iterations"].append(r)
        prev = b.actions
    top = uniform_topology(4)
    asg = {t: ActionAssignment(t, bundle.actions[t], a) for t, a in sizes.items()}
    res = evaluate_assignments(g, top, asg)
    roots = H.od.apply_fusion(ogr, bundle.actions["fusion_priority"], max_group=8)
    fg = H.od.Fused(ogr, roots)
    want = H.od.simulate(ogr, fg, bundle.actions["placement"], bundle.actions["schedule_priority"],
                         H.od.uniform_topology(4))
    rep["des"] = {"got": res.step_time, "want": want["step_time"],
                  "groups": int(max(fg.group_map) + 1)}
    assert res.step_time == want["step_time"] and res.valid == want["valid"], rep["des"]
    assert res.per_device_busy == list(want["busy"]) and res.peak_mem == list(want["peak"])
    _report("cfg2_joint", rep)

"""GPU parity: the CUDA path (through the C-ABI) vs golden vectors from the
unmodified reference and the oracle.

Tolerances (SURVEY §8 / BASELINE north_star):
  * embeddings, hiddens, logits, value: normwise relative error
    max|gpu - ref| / max|ref| <= 1e-4 (fp32 kernels vs float64 reference);
  * neighbour samples, actions: bit-exact;
  * makespans / busy / peak memory / validity: bit-exact;
  * log-probs given identical float64 logits: <= 1e-12 relative (libm exp/log ulps).
"""
import numpy as np
import pytest

from conftest import forward_meta, golden, rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-4


def _g(z, p):
    from paper_2010_12438_b200.graph import Graph
    return Graph(z[p + "op"], z[p + "flops"], z[p + "out_bytes"], z[p + "src"], z[p + "dst"],
                 z[p + "ebytes"], z[p + "coloc"])


def _case(case):
    from paper_2010_12438_b200 import EmbedConfig, PolicyConfig, init_all_params, randomize_zero_init
    meta = {m["name"]: m for m in forward_meta()}[case]
    z = golden("forward")
    p = case + "/"
    ecfg = EmbedConfig(**meta["ecfg"])
    pcfg = PolicyConfig(**meta["pcfg"])
    store = randomize_zero_init(init_all_params(ecfg, pcfg, meta["sizes"], 0))
    return meta, z, p, _g(z, p), ecfg, pcfg, store


CASES = [m["name"] for m in forward_meta()]


@pytest.mark.parametrize("case", CASES)
def test_neighbor_arrays_exact(case):
    from paper_2010_12438_b200.embedding import neighbor_arrays
    meta, z, p, g, ecfg, pcfg, store = _case(case)
    gather, seg = neighbor_arrays(g, ecfg.gs_knn, meta["embed_seed"])
    assert np.array_equal(gather, z[p + "gather"])
    assert np.array_equal(seg, z[p + "seg"])


@pytest.mark.parametrize("case", CASES)
def test_embed_trunk_heads_parity(case):
    from paper_2010_12438_b200.embedding import embed
    from paper_2010_12438_b200.graph import node_features
    from paper_2010_12438_b200.policy import ordered_tasks, task_heads, trunk_forward
    meta, z, p, g, ecfg, pcfg, store = _case(case)
    tasks = ordered_tasks(meta["sizes"])
    feats = node_features(g, None, [a for _, a in tasks])
    assert np.array_equal(feats, z[p + "feats"])
    emb = embed(g, feats, store, ecfg, seed=meta["embed_seed"])
    assert rel_err(emb.node_embed.data, z[p + "node_embed"]) < TOL
    assert rel_err(emb.graph_embed.data, z[p + "graph_embed"]) < TOL
    hid = trunk_forward(z[p + "node_embed"], z[p + "graph_embed"], store, pcfg)
    assert rel_err(hid.data, z[p + "hid"]) < TOL
    heads = task_heads(z[p + "hid"], store, pcfg, tasks)
    for t, _a in tasks:
        assert rel_err(heads.logits[t].data, z[p + f"logits/{t}"]) < TOL, t
    assert rel_err(heads.value.data, z[p + "value"]) < TOL


@pytest.mark.parametrize("case", CASES)
def test_forward_policy_end_to_end(case):
    from paper_2010_12438_b200.policy import forward_policy, ordered_tasks
    meta, z, p, g, ecfg, pcfg, store = _case(case)
    heads = forward_policy(g, store, ecfg, pcfg, meta["sizes"], None, meta["embed_seed"])
    for t, _a in ordered_tasks(meta["sizes"]):
        assert rel_err(heads.logits[t].data, z[p + f"logits/{t}"]) < TOL, t


@pytest.mark.parametrize("case", CASES)
def test_iterate_decisions_parity(case):
    from paper_2010_12438_b200.policy import iterate_decisions, ordered_tasks
    meta, z, p, g, ecfg, pcfg, store = _case(case)
    bundle, traj = iterate_decisions(g, store, ecfg, pcfg, meta["sizes"], pcfg.iterations,
                                     meta["decision_seed"])
    assert len(traj) == pcfg.iterations
    for it, b in enumerate(traj):
        for t, _a in ordered_tasks(meta["sizes"]):
            assert np.array_equal(b.actions[t], z[p + f"it{it}/actions/{t}"]), (it, t)
            assert np.allclose(b.log_probs[t], z[p + f"it{it}/logp/{t}"], rtol=1e-4, atol=1e-5)
            assert rel_err(b.logits[t], z[p + f"it{it}/logits/{t}"]) < TOL
        assert abs(b.value - float(z[p + f"it{it}/value"])) <= TOL * max(1.0, abs(float(z[p + f"it{it}/value"])))
    assert bundle.prev_actions is not None or pcfg.iterations == 1


def test_sampler_bit_exact_given_logits_and_stream():
    from paper_2010_12438_b200.policy import sample_actions
    z = golden("sample")
    for k in range(int(z["count"])):
        p = f"s{k}/"
        r = np.random.default_rng(int(z[p + "seed"]))
        if int(z[p + "offset"]):
            r.random(int(z[p + "offset"]))
        a, lp = sample_actions(z[p + "logits"], float(z[p + "temp"]), r)
        assert np.array_equal(a, z[p + "actions"]), k
        assert np.allclose(lp, z[p + "logp"], rtol=1e-12, atol=1e-14), k
        # the generator advanced exactly like rng.random((N, 1)) would
        ref = np.random.default_rng(int(z[p + "seed"]))
        ref.random(int(z[p + "offset"]) + (len(a) if float(z[p + "temp"]) > 0 else 0))
        assert r.random() == ref.random()


def _topology(z, p):
    from paper_2010_12438_b200.costmodel import Topology
    return Topology(z[p + "top_peak"], z[p + "top_mem_bw"], z[p + "top_cap"], z[p + "top_link_bw"])


def test_des_bit_exact_all_golden_cases():
    from paper_2010_12438_b200.simulator import ActionAssignment, FusedGraph, simulate
    z = golden("des")
    for c in range(int(z["count"])):
        p = f"c{c}/"
        g = _g(z, p)
        top = _topology(z, p)
        d = top.num_devices
        fg = FusedGraph(g, z[p + "group_map"])
        res = simulate(fg, ActionAssignment("placement", z[p + "placement"], d),
                       ActionAssignment("schedule_priority", z[p + "priorities"], 8), top,
                       policy=str(z[p + "policy"]))
        assert res.step_time == float(z[p + "step_time"]), c
        assert res.valid == bool(z[p + "valid"]), c
        assert (res.violation or "") == str(z[p + "violation"]), c
        assert res.per_device_busy == list(z[p + "busy"]), c
        assert res.peak_mem == list(z[p + "peak"]), c


def test_des_batched_matches_oracle_random_placements():
    """Many placements of one workload graph in a single launch vs the oracle DES."""
    from oracle import des as od
    from oracle import graph as og
    from paper_2010_12438_b200.costmodel import uniform_topology
    from paper_2010_12438_b200.simulator import simulate_many, singleton_fused
    from synthetic.workloads import WorkloadSpec, gen_workload
    g = gen_workload(WorkloadSpec("attention-stack", 60, 1, 64, seed=0), node_cap=10**6)
    rng = np.random.default_rng(7)
    K, d = 48, 8
    pl = rng.integers(0, d, (K, g.num_nodes))
    pr = rng.integers(0, 8, (K, g.num_nodes))
    res = simulate_many(singleton_fused(g), pl, pr, uniform_topology(d), baseline=1e-3)
    st = res.step_time.cpu().numpy()
    rw = res.reward.cpu().numpy()
    og_g = og.make(g.num_nodes, g.op, g.flops, g.out_bytes, g.src, g.dst, g.ebytes)
    fg = od.singleton(og_g)
    top = od.uniform_topology(d)
    for k in range(0, K, 6):
        want = od.simulate(og_g, fg, pl[k], pr[k], top)
        assert st[k] == want["step_time"]
        assert rw[k] == od.reward(want["step_time"], 1e-3, want["valid"])


def test_collect_rollouts_parity_cfg1():
    from paper_2010_12438_b200 import EmbedConfig, PolicyConfig, PPOHyper, init_all_params, randomize_zero_init
    from paper_2010_12438_b200.baselines import baseline_step_time, default_assignments
    from paper_2010_12438_b200.config import FusionConfig
    from paper_2010_12438_b200.costmodel import uniform_topology
    from paper_2010_12438_b200.training import collect_rollouts
    z = golden("rollouts")
    g = _g(z, "g/")
    top = uniform_topology(2)
    sizes = {"placement": 2}
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
    bl = baseline_step_time(g, top)
    assert bl == float(z["baseline"])
    batch = collect_rollouts(store, [g], top, sizes, [bl], int(z["count"]), 0, PPOHyper(rollouts=6),
                             ecfg, pcfg, FusionConfig(), base_assignments=[default_assignments(g, top)])
    for i, s in enumerate(batch.samples):
        p = f"r{i}/"
        assert s.graph_index == int(z[p + "graph_index"])
        assert np.array_equal(s.bundle.actions["placement"], z[p + "actions"])
        assert np.array_equal(s.bundle.prev_actions["placement"], z[p + "prev_actions"])
        assert s.step_time == float(z[p + "step_time"])
        assert s.reward == float(z[p + "reward"])
        assert s.valid == bool(z[p + "valid"])
        assert abs(s.value_estimate - float(z[p + "value"])) < 1e-4 * max(1, abs(float(z[p + "value"])))


def test_nonfinite_embedding_raises():
    from paper_2010_12438_b200 import EmbedConfig, ParamStore
    from paper_2010_12438_b200.embedding import embed, init_embed_params
    from paper_2010_12438_b200.graph import Graph, node_features
    g = Graph([6, 6, 6], [0, 0, 0], [4, 4, 4], [0, 0], [1, 2], [4, 4])
    cfg = EmbedConfig(2, 8, 5)
    feats = node_features(g, None, 2)
    store = ParamStore()
    init_embed_params(store, feats.shape[1], cfg, np.random.default_rng(0))
    store[f"embed/fc_b{cfg.gs_layers - 1}"].data[:] = np.inf
    store.touch()
    with pytest.raises(FloatingPointError):
        embed(g, feats, store, cfg)
    with pytest.raises(ValueError):
        embed(g, np.zeros((1, feats.shape[1])), store, cfg)


def test_collect_rollouts_joint_tasks_match_reference():
    """Joint placement + schedule + fusion rollouts (SURVEY §8(f) F1 reward path): every
    rollout has its own fused grouping (native fusion pass, grouped DES launches); the
    sampled actions, step times and rewards are the reference's."""
    from paper_2010_12438_b200 import (EmbedConfig, FusionConfig, PolicyConfig, PPOHyper,
                                       init_all_params, randomize_zero_init, uniform_topology)
    from paper_2010_12438_b200.baselines import baseline_step_time, default_assignments
    from paper_2010_12438_b200.training import collect_rollouts
    z = golden("rollouts_joint")
    g = _g(z, "g/")
    top = uniform_topology(3)
    sizes = {"placement": 3, "schedule_priority": 8, "fusion_priority": 8}
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
    bl = baseline_step_time(g, top)
    assert bl == float(z["baseline"])
    n = int(z["count"])
    batch = collect_rollouts(store, [g], top, sizes, [bl], n, 4, PPOHyper(rollouts=n), ecfg, pcfg,
                             FusionConfig(), base_assignments=[default_assignments(g, top)])
    assert int(z["distinct_groupings"]) > 1
    for i, s in enumerate(batch.samples):
        p = f"r{i}/"
        for t in sizes:
            assert np.array_equal(s.bundle.actions[t], z[p + "actions/" + t]), (i, t)
        assert s.step_time == float(z[p + "step_time"]), i
        assert s.reward == float(z[p + "reward"]), i
        assert s.valid == bool(z[p + "valid"]), i


def test_simulate_record_trace_matches_reference():
    """simulate(record_trace=True): the device event log (go_simulate_trace), sorted
    like simulator.py:432-433, equals the reference's TraceEvent list exactly (starts,
    ends, device / link strings incl. >= 10 devices, kinds, groups), together with the
    untraced results (golden_trace.npz from make_golden.py make_trace)."""
    from paper_2010_12438_b200.simulator import ActionAssignment, FusedGraph, simulate
    z = golden("trace")
    total = 0
    for c in range(int(z["count"])):
        p = f"c{c}/"
        g = _g(z, p)
        top = _topology(z, p)
        d = top.num_devices
        fg = FusedGraph(g, z[p + "group_map"])
        pl = ActionAssignment("placement", z[p + "placement"], d)
        pr = ActionAssignment("schedule_priority", z[p + "priorities"], 8)
        res = simulate(fg, pl, pr, top, policy=str(z[p + "policy"]), record_trace=True)
        plain = simulate(fg, pl, pr, top, policy=str(z[p + "policy"]))
        assert res.step_time == float(z[p + "step_time"]) == plain.step_time, c
        assert res.per_device_busy == plain.per_device_busy and res.peak_mem == plain.peak_mem
        tr = res.trace
        assert [e.time_start for e in tr] == list(z[p + "t_start"]), c
        assert [e.time_end for e in tr] == list(z[p + "t_end"]), c
        assert [e.device for e in tr] == [str(x) for x in z[p + "device"]], c
        assert [e.kind for e in tr] == [str(x) for x in z[p + "kind"]], c
        assert [e.group_id for e in tr] == list(z[p + "group"]), c
        total += len(tr)
    assert total > 1000


def test_shared_logits_sampler_is_per_placement_sample_actions():
    """Mode S sampling (go_sample with shared logits): K placements
    drawn from ONE forward's logits, each with its own numpy stream, equal K separate
    sample_actions calls (policy.py:220-237) on those logits, bit for bit."""
    from paper_2010_12438_b200 import EmbedConfig, PolicyConfig, init_all_params, randomize_zero_init
    from paper_2010_12438_b200.engine import forward_batch, pcg_words, sample_batch
    from paper_2010_12438_b200.policy import sample_actions
    from paper_2010_12438_b200.runtime import context
    from synthetic.workloads import WorkloadSpec, gen_workload
    g = gen_workload(WorkloadSpec("attention-stack", 20, 1, 64, seed=0))
    sizes = {"placement": 8}
    ecfg, pcfg = EmbedConfig(), PolicyConfig(iterations=1)
    store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
    h = context().graph(g)
    out = forward_batch(store, ecfg, pcfg, sizes, [h], [11])
    seeds = [3, 1 << 40, 17, 99, 5]
    acts, logp = sample_batch(ecfg, pcfg, sizes, [h] * len(seeds),
                              [pcg_words(np.random.default_rng(s)) for s in seeds],
                              out.logits_packed, 1.0, shared_logits=True)
    lg = out.logits[0].double().cpu().numpy()
    order = np.asarray(g.topo_order())
    n = g.num_nodes
    for k, s in enumerate(seeds):
        a_ref, lp_ref = sample_actions(lg, 1.0, np.random.default_rng(s))
        node = np.zeros(n, np.int64)
        node[order] = a_ref
        assert np.array_equal(acts[0, k * n:(k + 1) * n].cpu().numpy(), node), k
        assert np.array_equal(logp[0, k * n:(k + 1) * n].cpu().numpy(), lp_ref), k

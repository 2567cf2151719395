"""Pin the CPU oracle against golden vectors produced by the unmodified
reference (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from conftest import forward_meta, golden, oracle_graph, rel_err
from oracle import des as od
from oracle import forward as of
from oracle import graph as og
from oracle import params as op
from oracle import rng as orng


def test_star_neighbor_picks_match_reference():
    z = golden("rng")
    for row in z["star_picks"]:
        leaves, seed, k = int(row[0]), int(row[1]), int(row[2])
        want = [int(x) for x in row[3:] if x >= 0]
        nbrs = list(range(1, leaves + 1))
        if leaves <= k:
            got = nbrs
        else:
            got = [nbrs[i] for i in orng.floyd_choice_set(seed, 0, leaves, k)]
        assert got == want, (leaves, seed, k)


def test_uniform_stream_matches_reference():
    z = golden("rng")
    for seed, idx, u in z["uniforms"]:
        assert orng.uniform_at(int(seed), int(idx)) == u


def test_seedsequence_matches_numpy():
    for e in (0, 1, 2**31 - 1, [5, 0], [2**31 - 1, 80000], [0, 2**32 + 3]):
        want = [int(x) for x in np.random.SeedSequence(e).generate_state(4, np.uint64)]
        assert orng.seedseq_generate_u64(e, 4) == want


@pytest.mark.parametrize("case", [m["name"] for m in forward_meta()])
def test_forward_oracle_matches_reference(case):
    meta = {m["name"]: m for m in forward_meta()}[case]
    z = golden("forward")
    p = case + "/"
    g = oracle_graph(z, p)
    assert np.array_equal(g["topo"], z[p + "topo"])
    ecfg = of.EmbedCfg(**meta["ecfg"])
    pcfg = of.PolicyCfg(**meta["pcfg"])
    sizes = meta["sizes"]
    P = op.randomize_zero_init(op.init_all_params(ecfg, pcfg, sizes, 0))
    names = [str(x) for x in z[p + "param_names"]]
    assert names == sorted(P)
    for n, s1, s2 in zip(names, z[p + "param_sum"], z[p + "param_sq"]):
        assert P[n].sum() == s1 and (P[n] ** 2).sum() == s2, n
    tasks = of.ordered_tasks(sizes)
    feats = og.node_features(g, None, [a for _, a in tasks])
    assert np.array_equal(feats, z[p + "feats"])
    gather, seg = of.neighbor_arrays(g, ecfg.gs_knn, meta["embed_seed"])
    assert np.array_equal(gather, z[p + "gather"]) and np.array_equal(seg, z[p + "seg"])
    ne, ge = of.embed(g, feats, P, ecfg, seed=meta["embed_seed"])
    assert rel_err(ne, z[p + "node_embed"]) < 1e-12
    assert rel_err(ge, z[p + "graph_embed"]) < 1e-12
    hid = of.trunk_forward(z[p + "node_embed"], z[p + "graph_embed"], P, pcfg)
    assert rel_err(hid, z[p + "hid"]) < 1e-12
    logits, _, value = of.task_heads(z[p + "hid"], P, pcfg, tasks, chunk=7)
    for t, _a in tasks:
        assert rel_err(logits[t], z[p + f"logits/{t}"]) < 1e-12
    assert rel_err(value, z[p + "value"]) < 1e-12
    traj = of.iterate_decisions(g, P, ecfg, pcfg, sizes, pcfg.iterations, meta["decision_seed"])
    for it, b in enumerate(traj):
        for t, _a in tasks:
            assert np.array_equal(b["actions"][t], z[p + f"it{it}/actions/{t}"])
            assert rel_err(b["log_probs"][t], z[p + f"it{it}/logp/{t}"]) < 1e-10


def _topology(z, p):
    return od.Topology(z[p + "top_peak"], z[p + "top_mem_bw"], z[p + "top_cap"], z[p + "top_link_bw"])


def test_des_oracle_bit_exact():
    z = golden("des")
    for c in range(int(z["count"])):
        p = f"c{c}/"
        g = oracle_graph(z, p)
        fg = od.Fused(g, z[p + "group_map"])
        res = od.simulate(g, fg, z[p + "placement"], z[p + "priorities"], _topology(z, p),
                          policy=str(z[p + "policy"]))
        assert res["step_time"] == z[p + "step_time"], c
        assert res["valid"] == bool(z[p + "valid"]), c
        assert (res["violation"] or "") == str(z[p + "violation"]), c
        assert res["busy"] == list(z[p + "busy"]), c
        assert res["peak"] == list(z[p + "peak"]), c
        if p + "greedy" in z:
            assert np.array_equal(od.greedy_placement(g, len(z[p + "peak"])), z[p + "greedy"])


def test_fusion_oracle_matches_reference_groups():
    """oracle.des.apply_fusion against the reference's apply_fusion group maps
    (golden_fusion.npz, with the priorities that produced them)."""
    z = golden("fusion")
    for c in range(int(z["count"])):
        p = f"c{c}/"
        g = oracle_graph(z, p)
        roots = od.apply_fusion(g, z[p + "pri"], max_group=int(z[p + "max_group"]))
        got = od.Fused(g, roots).group_map
        assert np.array_equal(np.asarray(got), z[p + "group_map"]), (c, str(z[p + "tag"]))


def test_sampler_oracle_bit_exact():
    z = golden("sample")
    for k in range(int(z["count"])):
        p = f"s{k}/"
        r = np.random.default_rng(int(z[p + "seed"]))
        if int(z[p + "offset"]):
            r.random(int(z[p + "offset"]))
        a, lp = of.sample_actions(z[p + "logits"], float(z[p + "temp"]), r)
        assert np.array_equal(a, z[p + "actions"])
        assert np.array_equal(lp, z[p + "logp"])


def test_rollout_oracle_matches_reference():
    z = golden("rollouts")
    g = oracle_graph(z, "g/")
    ecfg, pcfg = of.EmbedCfg(), of.PolicyCfg()
    sizes = {"placement": 2}
    P = op.randomize_zero_init(op.init_all_params(ecfg, pcfg, sizes, 0))
    top = od.uniform_topology(2)
    base = od.greedy_placement(g, 2)
    fg = od.singleton(g)
    bl = od.simulate(g, fg, base, np.zeros(g["n"]), top)["step_time"]
    assert bl == z["baseline"]
    rng = np.random.default_rng(0)
    for i in range(int(z["count"])):
        p = f"r{i}/"
        gi = int(rng.integers(1))
        seed = int(rng.integers(2**31))
        assert seed == int(z[p + "embed_seed"]) and gi == int(z[p + "graph_index"])
        traj = of.iterate_decisions(g, P, ecfg, pcfg, sizes, 2, seed)
        acts = traj[-1]["actions"]["placement"]
        assert np.array_equal(acts, z[p + "actions"])
        assert np.array_equal(traj[0]["actions"]["placement"], z[p + "prev_actions"])
        res = od.simulate(g, fg, acts, np.zeros(g["n"]), top)
        assert res["step_time"] == z[p + "step_time"]
        assert od.reward(res["step_time"], bl, res["valid"]) == z[p + "reward"]
        assert abs(traj[-1]["value"] - z[p + "value"]) < 1e-12


def test_row_subset_heads_and_per_row_sampler_match_full_oracle():
    """The helpers the headline parity tests use (tests/headline.py): task-head logits
    on a subset of query rows equal the full float64 heads on those rows, and the
    per-row sampler with the reference's uniform index reproduces iterate_decisions."""
    import headline as H
    z = golden("rollouts")
    g = oracle_graph(z, "g/")
    ecfg, pcfg = of.EmbedCfg(), of.PolicyCfg()
    sizes = {"placement": 2}
    P = op.randomize_zero_init(op.init_all_params(ecfg, pcfg, sizes, 0))
    feats = og.node_features(g, None, [2])
    ne, ge = of.embed(g, feats, P, ecfg, seed=11)
    hid = of.trunk_forward(ne, ge, P, pcfg)
    full, _, _ = of.task_heads(hid, P, pcfg, [("placement", 2)])
    rows = H.sample_rows(g["n"], 17, seed=2)
    sub, _ = of.task_heads_rows(hid, P, pcfg, [("placement", 2)], rows)
    assert np.allclose(sub, full["placement"][rows], rtol=1e-13, atol=1e-13)
    traj = of.iterate_decisions(g, P, ecfg, pcfg, sizes, 2, 11)
    n = g["n"]
    for it, step in enumerate(traj):
        rep = H.check_actions(step["actions"]["placement"], step["log_probs"]["placement"],
                              step["logits"]["placement"], step["logits"]["placement"],
                              g["topo"], np.arange(n), 11, it, 0, 1)
        assert rep["flips"] == 0 and rep["logp_max_abs_err"] == 0.0, rep


def test_oracle_matches_unmodified_reference_at_cfg2():
    """The float64 oracle (tape-free, layer-major trunk, row-chunked heads: 'ref-lean',
    SURVEY §8(d) D4) against the UNMODIFIED reference at BASELINE cfg2 (13,000 nodes,
    golden_cfg2.npz): both iterations' logits to 1e-9, every action identical, the DES
    step time bit-exact.  The device's headline parity tests check against this oracle."""
    from synthetic.workloads import WorkloadSpec, gen_workload
    z = golden("cfg2")
    g = gen_workload(WorkloadSpec("multi-branch-cnn", 1857, 1, 64, seed=0), node_cap=10**6)
    ogr = og.make(g.num_nodes, g.op, g.flops, g.out_bytes, g.src, g.dst, g.ebytes)
    ecfg, pcfg = of.EmbedCfg(), of.PolicyCfg()
    P = op.randomize_zero_init(op.init_all_params(ecfg, pcfg, {"placement": 4}, 0))
    seed = int(z["seed"])
    feats = og.node_features(ogr, None, [4])
    ne, ge = of.embed(ogr, feats, P, ecfg, seed=seed)
    assert np.allclose(ne.sum(axis=1), z["node_embed_rowsum"], rtol=1e-10, atol=1e-10)
    assert np.allclose(ge, z["graph_embed"], rtol=1e-11, atol=1e-12)
    traj = of.iterate_decisions(ogr, P, ecfg, pcfg, {"placement": 4}, 2, seed)
    rows = z["rows"]
    for it, step in enumerate(traj):
        lg = step["logits"]["placement"]
        assert np.allclose(lg[rows], z[f"it{it}/logits_rows"], rtol=1e-9, atol=1e-11), it
        assert np.allclose(lg.sum(axis=1), z[f"it{it}/logit_rowsum"], rtol=1e-9, atol=1e-10)
        assert np.array_equal(step["actions"]["placement"], z[f"it{it}/actions"]), it
        assert np.allclose(step["log_probs"]["placement"], z[f"it{it}/logp"], rtol=1e-9,
                           atol=1e-11)
        assert abs(step["value"] - float(z[f"it{it}/value"])) < 1e-9
    res = od.simulate(ogr, od.singleton(ogr), traj[-1]["actions"]["placement"],
                      np.zeros(ogr["n"]), od.uniform_topology(4))
    assert res["step_time"] == float(z["step_time"])

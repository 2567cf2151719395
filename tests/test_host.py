"""CPU tests of the product's host side: the C-ABI library loads and exports every
declared symbol, and the native host routines (topological order, greedy
placement DP, fusion pass, workload generator) match the reference via the golden
fixtures and the oracle.  No CUDA device needed."""
import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden, oracle_graph
from oracle import des as od
from paper_2010_12438_b200 import _lib
from paper_2010_12438_b200.fusion import fuse_groups, greedy_cuts
from paper_2010_12438_b200.graph import Graph, GraphError
from synthetic.workloads import WorkloadSpec, gen_workload


def test_header_symbols_exported():
    header = (ROOT / "include" / "go_b200.h").read_text()
    declared = set(re.findall(r"^(?:int|long long|const char\*)\s+(go_\w+)\(", header, re.M))
    assert declared == set(_lib.EXPORTS)
    L = _lib.lib()
    for name in declared:
        assert hasattr(L, name), name
    assert L.go_version() >= 1


def _product_graph(z, p):
    return Graph(z[p + "op"], z[p + "flops"], z[p + "out_bytes"], z[p + "src"], z[p + "dst"],
                 z[p + "ebytes"], z[p + "coloc"])


def test_topo_order_matches_reference():
    for name in ("des", "forward"):
        z = golden(name)
        prefixes = sorted({k.split("/")[0] for k in z if "/" in k and k.endswith("/topo")})
        for pre in prefixes:
            g = _product_graph(z, pre + "/")
            assert np.array_equal(g.topo_order(), z[pre + "/topo"]), pre


def test_topo_order_cycle():
    g = Graph([0, 0], [0, 0], [0, 0], [0, 1], [1, 0], [0, 0])
    with pytest.raises(GraphError):
        g.topo_order()


def test_greedy_cuts_match_reference_dp():
    z = golden("des")
    seen = 0
    for c in range(int(z["count"])):
        p = f"c{c}/"
        if p + "greedy" not in z:
            continue
        g = oracle_graph(z, p)
        d = len(z[p + "peak"])
        from paper_2010_12438_b200.baselines import greedy_placement  # noqa: F401
        order = g["topo"]
        cuts = greedy_cuts(g["flops"][order], d)
        acts = np.zeros(g["n"], np.int64)
        for dev in range(d):
            acts[order[cuts[dev]:cuts[dev + 1]]] = dev
        assert np.array_equal(acts, z[p + "greedy"])
        seen += 1
    assert seen == 3


@pytest.mark.parametrize("seed", range(12))
def test_greedy_cuts_random_vs_oracle(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 60))
    flops = rng.choice([0.0, 1.0, 2.5, 1e6], size=n) * rng.integers(0, 3, n)
    g = dict(n=n, topo=np.arange(n), flops=flops.astype(np.float64), coloc=np.full(n, -1))
    for d in (1, 2, 3, 8):
        want = od.greedy_placement(g, d)
        cuts = greedy_cuts(flops, d)
        acts = np.zeros(n, np.int64)
        for dev in range(d):
            acts[cuts[dev]:cuts[dev + 1]] = dev
        assert np.array_equal(acts, want), (seed, d)


def canonical_groups(labels):
    """Group labels renumbered by ascending min member id (simulator.py:98-109)."""
    labels = np.asarray(labels)
    first = {}
    return np.array([first.setdefault(int(x), len(first)) for x in labels], np.int64)


def _fusion_cases():
    z = golden("fusion")
    for c in range(int(z["count"])):
        p = f"c{c}/"
        yield c, z, p


def test_fusion_pass_matches_reference_group_maps():
    """go_apply_fusion (native) against the UNMODIFIED reference's apply_fusion group
    maps, with the priorities and max_group that produced them (tests/golden
    make_fusion: random DAGs, permuted ids, workload families)."""
    merged = 0
    for c, z, p in _fusion_cases():
        n = int(z[p + "n"])
        g = Graph(z[p + "op"], z[p + "flops"], z[p + "out_bytes"], z[p + "src"], z[p + "dst"],
                  z[p + "ebytes"])
        got = canonical_groups(fuse_groups(g, z[p + "pri"], int(z[p + "max_group"])))
        want = z[p + "group_map"]
        assert np.array_equal(got, want), (c, str(z[p + "tag"]))
        merged += int(want.max(initial=-1) + 1 < n)
    assert merged >= 40  # the fixture exercises real merges, not just singletons


@pytest.mark.parametrize("seed", range(20))
def test_fusion_pass_vs_oracle(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 40))
    fus = [2, 3, 4, 5, 6, 7]  # fusible op indices
    op = rng.choice(fus + [0, 1], size=n)
    src, dst = [], []
    for i in range(n):
        for j in range(i + 1, n):
            if rng.random() < 0.25:
                src.append(i)
                dst.append(j)
    g = dict(n=n, op=op, src=np.array(src, np.int64), dst=np.array(dst, np.int64))
    pri = rng.integers(0, 8, n)
    mg = int(rng.choice([2, 3, 8]))
    want = od.apply_fusion(g, pri, max_group=mg)
    got = fuse_groups(Graph(op, np.zeros(n), np.zeros(n), src, dst, np.zeros(len(src))), pri, mg)
    assert np.array_equal(got, want)


def test_workloads_match_reference():
    z = golden("workloads")
    for i in range(int(z["count"])):
        p = f"w{i}/"
        fam, L, S, w, seed = [str(x) for x in z[p + "spec"]]
        g = gen_workload(WorkloadSpec(fam, int(L), int(S), int(w), int(seed)), node_cap=10**6)
        assert g.num_nodes == int(z[p + "n"]) and g.num_edges == int(z[p + "e"])
        assert int(g.op.sum()) == int(z[p + "op_sum"])
        assert g.flops.sum() == z[p + "flops"] and g.out_bytes.sum() == z[p + "out_bytes"]
        assert g.ebytes.sum() == z[p + "ebytes"]
        sig = (g.src.astype(np.int64) * 1000003 + g.dst).sum() % (2**61 - 1)
        assert sig == int(z[p + "edge_sig"])
        topo = g.topo_order().astype(np.int64)
        assert (topo * np.arange(g.num_nodes)).sum() % (2**61 - 1) == int(z[p + "topo_sig"])


@pytest.mark.parametrize("seed", range(30))
def test_fusion_pass_vs_oracle_permuted_ids(seed):
    """Node ids in random (non-topological) order, multi-edges, long-range edges and
    up to 300 nodes: the windowed cycle check (group-graph topological order) must make
    exactly the reference's merge decisions."""
    rng = np.random.default_rng(900 + seed)
    n = int(rng.integers(2, 300))
    perm = rng.permutation(n)
    fus = [2, 3, 4, 5, 6, 7]
    op = rng.choice(fus + [0, 1], size=n, p=[0.14] * 6 + [0.08, 0.08])
    src, dst = [], []
    dens = float(rng.choice([0.01, 0.03, 0.08]))
    for i in range(n):
        for j in range(i + 1, min(n, i + 1 + int(rng.integers(1, 40)))):
            if rng.random() < dens * 8:
                src.append(perm[i])
                dst.append(perm[j])
                if rng.random() < 0.05:  # multi-edge
                    src.append(perm[i])
                    dst.append(perm[j])
        if i + 50 < n and rng.random() < 0.05:  # long-range edge
            j = int(rng.integers(i + 50, n))
            src.append(perm[i])
            dst.append(perm[j])
    g = dict(n=n, op=op, src=np.array(src, np.int64), dst=np.array(dst, np.int64))
    for k in range(3):
        pri = rng.integers(0, 8, n)
        mg = int(rng.choice([2, 4, 8]))
        want = od.apply_fusion(g, pri, max_group=mg)
        got = fuse_groups(Graph(op, np.zeros(n), np.zeros(n), src, dst, np.zeros(len(src))),
                          pri, mg)
        assert np.array_equal(got, want)


@pytest.mark.parametrize("spec", [("attention-stack", 30, 1, 64, 0), ("dilated-stack", 5, 60, 64, 2),
                                  ("multi-branch-cnn", 80, 1, 64, 1)])
def test_fusion_pass_vs_oracle_workloads(spec):
    g = gen_workload(WorkloadSpec(*spec), node_cap=10**6)
    og_ = dict(n=g.num_nodes, op=np.asarray(g.op), src=np.asarray(g.src), dst=np.asarray(g.dst))
    rng = np.random.default_rng(7)
    for k in range(4):
        pri = rng.integers(0, 8, g.num_nodes)
        want = od.apply_fusion(og_, pri, max_group=8)
        got = fuse_groups(g, pri, 8)
        assert np.array_equal(got, want)


def test_bench_reference_arm_json_contract():
    """`bench.py --impl reference` (the CPU oracle on the host cores) prints one JSON line
    with the contract's keys (run on the small cfg1 workload so the CPU suite stays fast)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference",
                          "--workload", "cfg1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1


def test_checkpoint_with_adam_state_roundtrip(tmp_path):
    """save_state / load_state keep parameters, Adam moments and the
    step count; the reference-format save() file still loads (values only), and the
    reference-semantics load() ignores the optimiser keys of a save_state() file."""
    from paper_2010_12438_b200 import EmbedConfig, PolicyConfig, init_all_params
    ecfg, pcfg = EmbedConfig(1, 8, 4), PolicyConfig(1, 8, 2, 3, 16, 8, 2)
    s = init_all_params(ecfg, pcfg, {"placement": 2}, 0)
    rng = np.random.default_rng(0)
    for n in s.names():
        s._m[n] = rng.standard_normal(s[n].data.shape)
        s._v[n] = rng.random(s[n].data.shape)
    s.step_count = 17
    s.save_state(tmp_path / "full.npz")
    s.save(tmp_path / "plain.npz")
    t = init_all_params(ecfg, pcfg, {"placement": 2}, 1)
    t.load_state(tmp_path / "full.npz")
    assert t.step_count == 17 and t.names() == s.names()
    for n in s.names():
        assert np.array_equal(t[n].data, s[n].data)
        assert np.array_equal(t._m[n], s._m[n]) and np.array_equal(t._v[n], s._v[n])
    u = init_all_params(ecfg, pcfg, {"placement": 2}, 1)
    u.load(tmp_path / "full.npz")
    assert u.names() == s.names() and u.step_count == 0
    assert all(np.array_equal(u[n].data, s[n].data) for n in s.names())
    w = init_all_params(ecfg, pcfg, {"placement": 2}, 1)
    w.load_state(tmp_path / "plain.npz")
    assert all(np.array_equal(w[n].data, s[n].data) for n in s.names())
    assert w.step_count == 0 and not any(w._m[n].any() for n in w.names())
    z = dict(np.load(tmp_path / "full.npz"))
    z["__adam_m__/embed/in_w"] = np.zeros(3)
    np.savez(tmp_path / "bad.npz", **z)
    with pytest.raises(ValueError):
        init_all_params(ecfg, pcfg, {"placement": 2}, 1).load_state(tmp_path / "bad.npz")

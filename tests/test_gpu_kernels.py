"""GPU kernel-level checks: the tcgen05/TMEM task-head attention against the
float64 oracle and against the SIMT fp32 kernel, ragged multi-forward batches,
and full-size (80k-node) agreement.  Tolerance: normwise relative 1e-4."""
import os

import numpy as np
import pytest

from conftest import rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _store(sizes, ecfg=None, pcfg=None):
    from paper_2010_12438_b200 import EmbedConfig, PolicyConfig, init_all_params, randomize_zero_init
    ecfg = ecfg or EmbedConfig()
    pcfg = pcfg or PolicyConfig()
    return ecfg, pcfg, randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))


def _oracle_P(store):
    return {n: np.asarray(p.data) for n, p in store.items()}


@pytest.mark.parametrize("n", [1, 63, 64, 65, 255, 256, 257, 1000])
def test_task_heads_tc_vs_oracle(n):
    from oracle import forward as of
    from paper_2010_12438_b200.policy import ordered_tasks, task_heads
    sizes = {"placement": 8, "schedule_priority": 8, "fusion_priority": 8}
    ecfg, pcfg, store = _store(sizes)
    rng = np.random.default_rng(n)
    hid = rng.normal(size=(n, pcfg.d_model))
    tasks = ordered_tasks(sizes)
    out = task_heads(hid, store, pcfg, tasks)
    lg, _, val = of.task_heads(hid, _oracle_P(store), of.PolicyCfg(), tasks)
    for t, _a in tasks:
        assert rel_err(out.logits[t].data, lg[t]) < 1e-4, t
    assert rel_err(out.value.data, val) < 1e-4


def _heads_with(mode, hid, store, pcfg, tasks):
    from paper_2010_12438_b200.policy import task_heads
    old = os.environ.get("GO_ATTN")
    os.environ["GO_ATTN"] = mode
    try:
        return task_heads(hid, store, pcfg, tasks)
    finally:
        if old is None:
            del os.environ["GO_ATTN"]
        else:
            os.environ["GO_ATTN"] = old


@pytest.mark.parametrize("mode", ["tc", "tf32", "online"])
def test_tc_vs_simt_full_size_80k(mode):
    """tc = fixed-offset tcgen05 kernel with fp16 operands (default), tf32 = the same
    kernel in kind::tf32 (taken when a score bound exceeds the fp16-exact range),
    online = online-softmax tcgen05 kernel (taken when a bound is too large for a fixed
    offset), simt = fp32 CUDA-core kernel."""
    from paper_2010_12438_b200.policy import ordered_tasks
    sizes = {"placement": 8}
    ecfg, pcfg, store = _store(sizes)
    rng = np.random.default_rng(0)
    hid = rng.normal(size=(80001, pcfg.d_model)).astype(np.float32)
    tasks = ordered_tasks(sizes)
    a = _heads_with(mode, hid, store, pcfg, tasks)
    b = _heads_with("simt", hid, store, pcfg, tasks)
    assert rel_err(a.logits["placement"].data, b.logits["placement"].data) < 1e-4
    assert rel_err(a.value.data, b.value.data) < 1e-4


def test_large_scores_take_online_kernel():
    """Weights scaled up so |q||k| exceeds the fixed-offset bound: the launch must
    fall back to the online-softmax kernel and still match the oracle.  Scores here
    are ~20x the default magnitude, so the single-pass tf32 Q.K^T error (2^-11 of
    |q||k|) is amplified by exp(); the tolerance is 2e-3 for this stress case (the
    default-magnitude cases above hold 1e-4)."""
    from oracle import forward as of
    from paper_2010_12438_b200.policy import ordered_tasks, task_heads
    sizes = {"placement": 4}
    ecfg, pcfg, store = _store(sizes)
    for nm in ("policy/task_attn/q_w", "policy/task_attn/k_w"):
        store[nm].data = store[nm].data * 6.0
    store.touch()
    rng = np.random.default_rng(3)
    hid = rng.normal(size=(700, pcfg.d_model))
    tasks = ordered_tasks(sizes)
    out = task_heads(hid, store, pcfg, tasks)
    lg, _, _ = of.task_heads(hid, _oracle_P(store), of.PolicyCfg(), tasks)
    assert rel_err(out.logits["placement"].data, lg["placement"]) < 2e-3


def test_medium_scores_take_tf32_kernel():
    """Weights scaled so the score bounds land between the fp16 limit (14) and the
    fixed-offset limit (60): the launch must flag over to the tf32 fixed-offset kernel
    and still match the oracle (tolerance scaled with the ~9x larger scores)."""
    from oracle import forward as of
    from paper_2010_12438_b200.policy import ordered_tasks, task_heads
    sizes = {"placement": 4}
    ecfg, pcfg, store = _store(sizes)
    for nm in ("policy/task_attn/q_w", "policy/task_attn/k_w"):
        store[nm].data = store[nm].data * 3.0
    store.touch()
    rng = np.random.default_rng(4)
    hid = rng.normal(size=(900, pcfg.d_model))
    tasks = ordered_tasks(sizes)
    out = task_heads(hid, store, pcfg, tasks)
    lg, _, _ = of.task_heads(hid, _oracle_P(store), of.PolicyCfg(), tasks)
    assert rel_err(out.logits["placement"].data, lg["placement"]) < 5e-4


def _head_bounds(hid, P, sizes):
    """Per (row, head) fixed-offset bound b = |q| max|k| log2(e)/sqrt(d) the repack
    kernels compute (tc_attention16.cu), in float64 from the oracle's h."""
    import math
    from oracle import forward as of
    t, _a = of.ordered_tasks(sizes)[0]
    p, pa = f"policy/task/{t}/", "policy/task_attn/"
    n, d = hid.shape
    h = of.layer_norm(np.concatenate([np.zeros((n, d)), hid], 1) @ P[p + "cat_w"] + P[p + "cat_b"],
                      P[p + "ln_g"], P[p + "ln_b"])
    q = h @ P[pa + "q_w"] + P[pa + "q_b"]
    k = h @ P[pa + "k_w"] + P[pa + "k_b"]
    s = math.log2(math.e) / math.sqrt(15)
    return np.stack([np.linalg.norm(q[:, i * 15:(i + 1) * 15], axis=1)
                     * np.linalg.norm(k[:, i * 15:(i + 1) * 15], axis=1).max() * s
                     for i in range(3)], axis=1)


def test_fp16_fallback_is_per_work_item():
    """W_q scaled so only a few rows' bounds pass the fp16 limit (14): only the 384-query
    work items holding such a row move to the tf32 kernel (the fp16 kernel marks them),
    the rest stay on the fp16 kernel, and the whole launch matches the oracle."""
    from oracle import forward as of
    from paper_2010_12438_b200.policy import ordered_tasks, task_heads
    sizes = {"placement": 4}
    ecfg, pcfg, store = _store(sizes)
    rng = np.random.default_rng(5)
    hid = rng.normal(size=(2300, pcfg.d_model))
    b = _head_bounds(hid, _oracle_P(store), sizes)
    store["policy/task_attn/q_w"].data = store["policy/task_attn/q_w"].data * (
        14.3 / np.quantile(b, 0.9985))
    b = _head_bounds(hid, _oracle_P(store), sizes)
    works = np.stack([(b[i * 384:(i + 1) * 384] > 14.0).any(axis=0)
                      for i in range((len(hid) + 383) // 384)])
    assert works.any() and not works.all() and b.max() < 60, works
    tasks = ordered_tasks(sizes)
    out = task_heads(hid, store, pcfg, tasks)
    lg, _, _ = of.task_heads(hid, _oracle_P(store), of.PolicyCfg(), tasks)
    assert rel_err(out.logits["placement"].data, lg["placement"]) < 1e-4


def test_ragged_batch_matches_single_forwards():
    """A super-positioned batch (cfg3 style: mixed graph sizes in one launch) gives
    each forward exactly what it gets alone."""
    from paper_2010_12438_b200.engine import forward_batch
    from paper_2010_12438_b200.runtime import context
    from synthetic.workloads import WorkloadSpec, gen_workload
    sizes = {"placement": 8}
    ecfg, pcfg, store = _store(sizes)
    graphs = [gen_workload(WorkloadSpec("dilated-stack", 2, 50, 64, seed=3)),
              gen_workload(WorkloadSpec("attention-stack", 10, 1, 64, seed=0)),
              gen_workload(WorkloadSpec("dilated-stack", 5, 100, 64, seed=2), node_cap=10**6)]
    ctx = context()
    hs = [ctx.graph(g) for g in graphs]
    seeds = [11, 12, 13]
    out = forward_batch(store, ecfg, pcfg, sizes, hs, seeds)
    lg = out.logits[0].cpu().numpy()
    for i, (h, s) in enumerate(zip(hs, seeds)):
        one = forward_batch(store, ecfg, pcfg, sizes, [h], [s])
        lo, hi = out.row_off[i], out.row_off[i + 1]
        assert rel_err(lg[lo:hi], one.logits[0].cpu().numpy()) < 1e-5
        assert abs(float(out.value[i]) - float(one.value[0])) < 1e-5


def _forward_with(mode, store, ecfg, pcfg, sizes, graphs, seeds):
    from paper_2010_12438_b200.engine import forward_batch
    from paper_2010_12438_b200.runtime import context
    old = os.environ.get("GO_GEMM")
    os.environ["GO_GEMM"] = mode
    try:
        ctx = context()
        out = forward_batch(store, ecfg, pcfg, sizes, [ctx.graph(g) for g in graphs], seeds)
        return (out.node_embed.cpu().numpy(), out.logits[0].cpu().numpy(), out.value.cpu().numpy())
    finally:
        if old is None:
            del os.environ["GO_GEMM"]
        else:
            os.environ["GO_GEMM"] = old


def test_tc_gemm_forward_matches_simt_and_oracle():
    """The tcgen05 3xTF32 dense layers (default 128-wide config) agree with the SIMT
    fp32 GEMMs and with the float64 oracle on a workload graph and a ragged batch."""
    from oracle import forward as of
    from oracle import graph as og
    from synthetic.workloads import WorkloadSpec, gen_workload
    sizes = {"placement": 8}
    ecfg, pcfg, store = _store(sizes)
    graphs = [gen_workload(WorkloadSpec("multi-branch-cnn", 300, 1, 64, seed=0), node_cap=10**6),
              gen_workload(WorkloadSpec("attention-stack", 10, 1, 64, seed=0))]
    seeds = [5, 6]
    # same trunk attention kernel in both modes (the default mma trunk runs fp16 operands)
    old_trunk = os.environ.get("GO_TRUNK")
    os.environ["GO_TRUNK"] = "simt"
    try:
        ne_t, lg_t, v_t = _forward_with("tc", store, ecfg, pcfg, sizes, graphs, seeds)
        ne_s, lg_s, v_s = _forward_with("simt", store, ecfg, pcfg, sizes, graphs, seeds)
    finally:
        if old_trunk is None:
            os.environ.pop("GO_TRUNK", None)
        else:
            os.environ["GO_TRUNK"] = old_trunk
    assert rel_err(ne_t, ne_s) < 1e-5
    assert rel_err(lg_t, lg_s) < 1e-5
    assert rel_err(v_t, v_s) < 1e-5
    g = graphs[0]
    ogr = og.make(g.num_nodes, g.op, g.flops, g.out_bytes, g.src, g.dst, g.ebytes)
    logits, _, value = of.forward_policy(ogr, _oracle_P(store), of.EmbedCfg(), of.PolicyCfg(),
                                         sizes, None, 5)
    assert rel_err(lg_t[:g.num_nodes], logits["placement"]) < 1e-4


def _forward_env(var, val, store, ecfg, pcfg, sizes, graphs, seeds):
    from paper_2010_12438_b200.engine import forward_batch
    from paper_2010_12438_b200.runtime import context
    old = os.environ.get(var)
    if val is None:
        os.environ.pop(var, None)
    else:
        os.environ[var] = val
    try:
        ctx = context()
        out = forward_batch(store, ecfg, pcfg, sizes, [ctx.graph(g) for g in graphs], seeds)
        return out.hid.cpu().numpy(), out.logits[0].cpu().numpy()
    finally:
        if old is None:
            os.environ.pop(var, None)
        else:
            os.environ[var] = old


@pytest.mark.parametrize("seg", [64, 32, 16, 48, 100])
def test_trunk_tc_matches_simt(seg):
    """The default trunk attention (split-fp16 mma.sync, trunk_mma.cu; the round-1 opt-in
    tcgen05 trunk behind GO_TRUNK=tc was removed, so "tc" selects the default) agrees with
    the fp32 SIMT banded kernel on a ragged batch whose forwards end mid-segment and
    mid-tile, for segment lengths below, at and above the 64-query tile."""
    from paper_2010_12438_b200 import EmbedConfig, PolicyConfig
    from synthetic.workloads import WorkloadSpec, gen_workload
    sizes = {"placement": 8}
    ecfg, pcfg, store = _store(sizes, EmbedConfig(), PolicyConfig(segment_len=seg))
    graphs = [gen_workload(WorkloadSpec("multi-branch-cnn", 60, 1, 64, seed=1), node_cap=10**6),
              gen_workload(WorkloadSpec("attention-stack", 10, 1, 64, seed=0)),
              gen_workload(WorkloadSpec("dilated-stack", 5, 40, 64, seed=2), node_cap=10**6)]
    seeds = [3, 4, 5]
    h_tc, lg_tc = _forward_env("GO_TRUNK", "tc", store, ecfg, pcfg, sizes, graphs, seeds)
    h_s, lg_s = _forward_env("GO_TRUNK", "simt", store, ecfg, pcfg, sizes, graphs, seeds)
    assert rel_err(h_tc, h_s) < 1e-4
    assert rel_err(lg_tc, lg_s) < 1e-4


@pytest.mark.parametrize("seg", [64, 32, 16, 48, 100, 200])
def test_trunk_mma_matches_simt(seg):
    """The default banded trunk attention on mma.sync (trunk_mma.cu: 64-query tiles,
    64-key chunks with an online max, fp16 operands) agrees with the fp32 SIMT kernel
    (GO_TRUNK=simt) on a ragged batch; segment lengths that are not multiples of the
    64-query tile and windows wider than one key chunk (200 -> 400 keys) included."""
    from paper_2010_12438_b200 import EmbedConfig, PolicyConfig
    from synthetic.workloads import WorkloadSpec, gen_workload
    sizes = {"placement": 8}
    ecfg, pcfg, store = _store(sizes, EmbedConfig(), PolicyConfig(segment_len=seg))
    graphs = [gen_workload(WorkloadSpec("multi-branch-cnn", 60, 1, 64, seed=1), node_cap=10**6),
              gen_workload(WorkloadSpec("attention-stack", 10, 1, 64, seed=0)),
              gen_workload(WorkloadSpec("dilated-stack", 5, 40, 64, seed=2), node_cap=10**6)]
    seeds = [3, 4, 5]
    h_m, lg_m = _forward_env("GO_TRUNK", None, store, ecfg, pcfg, sizes, graphs, seeds)
    h_s, lg_s = _forward_env("GO_TRUNK", "simt", store, ecfg, pcfg, sizes, graphs, seeds)
    assert rel_err(h_m, h_s) < 1e-4
    assert rel_err(lg_m, lg_s) < 1e-4


def test_trunk_mma_out_of_range_reruns_simt():
    """Q/K/V beyond the fp16 range flag the layer and the SIMT kernel re-runs it: the
    forward stays finite and equal to the SIMT-only forward up to the fp16 rounding of
    the other (in-range) layers; without the re-run layer 0 would be inf / NaN."""
    sizes = {"placement": 4}
    ecfg, pcfg, store = _store(sizes)
    # |q| ~ 1e5 > the fp16 range: softmax becomes a near-argmax, outputs stay moderate
    store["policy/block0/attn_q_w"].data = store["policy/block0/attn_q_w"].data * 3e5
    store.touch()
    from synthetic.workloads import WorkloadSpec, gen_workload
    graphs = [gen_workload(WorkloadSpec("attention-stack", 10, 1, 64, seed=0))]
    h_m, lg_m = _forward_env("GO_TRUNK", None, store, ecfg, pcfg, sizes, graphs, [7])
    h_s, lg_s = _forward_env("GO_TRUNK", "simt", store, ecfg, pcfg, sizes, graphs, [7])
    assert np.isfinite(h_s).all() and np.isfinite(h_m).all()
    assert rel_err(h_m, h_s) < 1e-4


def test_fp16_gemm_matches_tf32_and_reruns_out_of_range():
    """The fp16-operand GEMMs (default) agree with the tf32-operand GEMMs
    (GO_GEMM_F16=0); with embedding weights scaled so activations exceed the fp16
    range, the fp16 pass flags itself and the tf32 re-run produces the same result."""
    from synthetic.workloads import WorkloadSpec, gen_workload
    sizes = {"placement": 8}
    ecfg, pcfg, store = _store(sizes)
    graphs = [gen_workload(WorkloadSpec("multi-branch-cnn", 200, 1, 64, seed=4), node_cap=10**6)]
    seeds = [9]
    old_trunk = os.environ.get("GO_TRUNK")
    os.environ["GO_TRUNK"] = "simt"  # compare the GEMMs alone (the mma trunk is fp16)
    try:
        for scale in (1.0, 3e4):
            _fp16_gemm_case(store, ecfg, pcfg, sizes, graphs, seeds, scale)
    finally:
        if old_trunk is None:
            os.environ.pop("GO_TRUNK", None)
        else:
            os.environ["GO_TRUNK"] = old_trunk


def _fp16_gemm_case(store, ecfg, pcfg, sizes, graphs, seeds, scale):
    if scale != 1.0:
        store["embed/in_w"].data = store["embed/in_w"].data * scale
        store.touch()
    h16, lg16 = _forward_env("GO_GEMM_F16", None, store, ecfg, pcfg, sizes, graphs, seeds)
    h32, lg32 = _forward_env("GO_GEMM_F16", "0", store, ecfg, pcfg, sizes, graphs, seeds)
    assert np.isfinite(lg16).all()
    # at 3e4 the embedding is ~1e5 in magnitude and the trunk's LayerNorms amplify the
    # (equal-size, differently rounded) 3-pass errors of both paths; without the
    # re-run the fp16 pass would overflow to inf
    tol = 1e-5 if scale == 1.0 else 1e-4
    assert rel_err(h16, h32) < tol, scale
    assert rel_err(lg16, lg32) < tol, scale


def test_fused_ffn_matches_unfused_and_reruns_out_of_range():
    """The fused trunk feed-forward kernel (tc_ffn.cuh) issues the same 3-pass fp16 MMAs
    in the same order as the two unfused GEMMs, so the forward is bit-identical; with
    FF weights scaled so the 512-wide intermediate leaves the fp16 range, the fused pass
    flags itself and the unfused tf32 re-run produces the layer (finite, close to the
    unfused path)."""
    from synthetic.workloads import WorkloadSpec, gen_workload
    sizes = {"placement": 8}
    ecfg, pcfg, store = _store(sizes)
    graphs = [gen_workload(WorkloadSpec("multi-branch-cnn", 120, 1, 64, seed=5), node_cap=10**6),
              gen_workload(WorkloadSpec("attention-stack", 10, 1, 64, seed=0))]
    seeds = [21, 22]
    h_f, lg_f = _forward_env("GO_FFN", None, store, ecfg, pcfg, sizes, graphs, seeds)
    h_u, lg_u = _forward_env("GO_FFN", "0", store, ecfg, pcfg, sizes, graphs, seeds)
    assert np.array_equal(h_f, h_u)
    assert np.array_equal(lg_f, lg_u)
    store["policy/block1/ff_w1"].data = store["policy/block1/ff_w1"].data * 4e5
    store.touch()
    h_f, lg_f = _forward_env("GO_FFN", None, store, ecfg, pcfg, sizes, graphs, seeds)
    h_u, lg_u = _forward_env("GO_FFN", "0", store, ecfg, pcfg, sizes, graphs, seeds)
    assert np.isfinite(h_f).all() and np.isfinite(lg_f).all()
    assert rel_err(h_f, h_u) < 1e-4
    assert rel_err(lg_f, lg_u) < 1e-4


@pytest.mark.parametrize("diag", [1e12, 7.5e9])
def test_des_uniform_links_match_oracle(diag):
    """With one bandwidth on every link the DES takes its transfer times from a per-edge
    table built once per launch (des_etab_kernel); the diagonal (never used: a group's
    local consumers need no transfer) may differ without leaving that path.  Step times
    and busy times agree bit-for-bit with the oracle DES."""
    from oracle import des as od
    from oracle import graph as og
    from paper_2010_12438_b200.costmodel import Topology
    from paper_2010_12438_b200.simulator import ActionAssignment, simulate, singleton_fused
    from synthetic.workloads import WorkloadSpec, gen_workload
    d = 8
    rng = np.random.default_rng(7)
    g = gen_workload(WorkloadSpec("multi-branch-cnn", 30, 1, 64, seed=4), node_cap=10**6)
    ogr = og.make(g.num_nodes, g.op, g.flops, g.out_bytes, g.src, g.dst, g.ebytes)
    peak = rng.choice([1e11, 5e11, 1e12], d)
    bw = rng.choice([5e10, 1e11], d)
    cap = np.full(d, 1e12)
    lb = np.full((d, d), 3.3e9)
    np.fill_diagonal(lb, diag)
    top = Topology(peak, bw, cap, lb)
    otop = od.Topology(list(peak), list(bw), list(cap), [[float(x) for x in row] for row in lb])
    fg = singleton_fused(g)
    for policy in ("priority", "fifo"):
        pl = rng.integers(0, d, g.num_nodes)
        pr = rng.integers(0, 8, g.num_nodes)
        res = simulate(fg, ActionAssignment("placement", pl, d),
                       ActionAssignment("schedule_priority", pr, 8), top, policy=policy)
        want = od.simulate(ogr, od.singleton(ogr), pl, pr, otop, policy=policy)
        assert res.step_time == want["step_time"], policy
        assert res.per_device_busy == list(want["busy"]), policy


@pytest.mark.parametrize("d", [3, 6, 12, 16])
def test_des_device_bounds_match_oracle(d):
    """The DES kernel is instantiated for 4 / 8 / 16 devices with its per-placement state in
    shared memory; every bound agrees bit-for-bit with the oracle DES (random heterogeneous
    topologies, random placements and priorities, both policies)."""
    from oracle import des as od
    from oracle import graph as og
    from paper_2010_12438_b200.costmodel import Topology
    from paper_2010_12438_b200.simulator import ActionAssignment, simulate, singleton_fused
    from synthetic.workloads import WorkloadSpec, gen_workload
    rng = np.random.default_rng(100 + d)
    g = gen_workload(WorkloadSpec("multi-branch-cnn", 20, 1, 64, seed=d), node_cap=10**6)
    ogr = og.make(g.num_nodes, g.op, g.flops, g.out_bytes, g.src, g.dst, g.ebytes)
    peak = rng.choice([1e11, 5e11, 1e12], d)
    bw = rng.choice([5e10, 1e11], d)
    cap = np.full(d, 1e12)
    lb = rng.choice([1e9, 5e9, 1e10], (d, d))
    top = Topology(peak, bw, cap, lb)
    otop = od.Topology(list(peak), list(bw), list(cap), [[float(x) for x in row] for row in lb])
    fg = singleton_fused(g)
    for policy in ("priority", "fifo"):
        pl = rng.integers(0, d, g.num_nodes)
        pr = rng.integers(0, 8, g.num_nodes)
        res = simulate(fg, ActionAssignment("placement", pl, d),
                       ActionAssignment("schedule_priority", pr, 8), top, policy=policy)
        want = od.simulate(ogr, od.singleton(ogr), pl, pr, otop, policy=policy)
        assert res.step_time == want["step_time"], (d, policy)
        assert res.per_device_busy == list(want["busy"]), (d, policy)

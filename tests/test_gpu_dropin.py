"""Drop-in hazards at the Python boundary:

* the device parameter cache never serves stale weights: in-place edits the way the
  reference's own tests make them (tests/test_policy.py:212 `.data[:] = 0.01`),
  whole-array reassignment, and a new store that reuses a freed store's id();
* the float64-master Adam (go_adam64) is the reference's ParamStore.adam_step
  (tensor.py:428-441) bit for bit, given the same gradients.
"""
import gc

import numpy as np
import pytest

from conftest import rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _setup(seed=0):
    from paper_2010_12438_b200 import EmbedConfig, PolicyConfig, init_all_params, randomize_zero_init
    from synthetic.workloads import WorkloadSpec, gen_workload
    g = gen_workload(WorkloadSpec("attention-stack", 3, 1, 64, seed=0))
    sizes = {"placement": 4}
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, seed))
    return g, sizes, ecfg, pcfg, store


def _oracle_logits(g, store, sizes, seed):
    from oracle import forward as of
    from oracle import graph as og
    ogr = og.make(g.num_nodes, g.op, g.flops, g.out_bytes, g.src, g.dst, g.ebytes)
    P = {n: np.asarray(p.data) for n, p in store.items()}
    lg, _, _ = of.forward_policy(ogr, P, of.EmbedCfg(), of.PolicyCfg(), sizes, None, seed)
    return lg["placement"]


def test_in_place_edit_is_seen():
    from paper_2010_12438_b200.policy import forward_policy
    g, sizes, ecfg, pcfg, store = _setup()
    a = forward_policy(g, store, ecfg, pcfg, sizes, None, 3).logits["placement"].data
    # exactly what the reference's test_coupled_differs_from_single does between calls
    store["policy/task/placement/out_w"].data[:] = 0.01
    b = forward_policy(g, store, ecfg, pcfg, sizes, None, 3).logits["placement"].data
    assert not np.allclose(a, b)
    assert rel_err(b, _oracle_logits(g, store, sizes, 3)) < 1e-4
    # whole-array reassignment of another tensor
    store["policy/task/placement/out_b"].data = np.full(4, 0.5)
    c = forward_policy(g, store, ecfg, pcfg, sizes, None, 3).logits["placement"].data
    assert rel_err(c, _oracle_logits(g, store, sizes, 3)) < 1e-4


def test_new_store_reusing_an_id_is_not_served_stale_weights():
    from paper_2010_12438_b200.policy import forward_policy
    g, sizes, ecfg, pcfg, s0 = _setup(0)
    want0 = forward_policy(g, s0, ecfg, pcfg, sizes, None, 3).logits["placement"].data
    ids = {id(s0)}
    del s0
    gc.collect()
    for seed in (2, 3, 4):
        _g, _s, _e, _p, s = _setup(seed)
        got = forward_policy(g, s, ecfg, pcfg, sizes, None, 3).logits["placement"].data
        assert not np.allclose(got, want0)
        assert rel_err(got, _oracle_logits(g, s, sizes, 3)) < 1e-4
        ids.add(id(s))
        del s
        gc.collect()


def test_adam64_is_the_reference_adam_bit_for_bit():
    from paper_2010_12438_b200 import _lib
    from paper_2010_12438_b200.params import ParamStore
    from paper_2010_12438_b200.runtime import context, stream_ptr
    rng = np.random.default_rng(0)
    n = 100_003
    store = ParamStore()
    store.add("w", rng.normal(size=n))
    dev = torch.device("cuda", context().device)
    p64 = torch.as_tensor(store["w"].data.copy(), device=dev)
    p32 = p64.to(torch.float32)
    m = torch.zeros(n, dtype=torch.float64, device=dev)
    v = torch.zeros_like(m)
    for step in range(1, 6):
        g32 = rng.normal(size=n).astype(np.float32) * (10.0 ** -step)
        g32[::7] = 0.0  # coordinates without gradient still step (g = 0)
        store["w"].grad = g32.astype(np.float64)
        store.adam_step(lr=3e-4)
        gd = torch.as_tensor(g32, device=dev)
        _lib.call("go_adam64", context().handle, _lib.ptr(p64), _lib.ptr(p32), _lib.ptr(gd),
                  _lib.ptr(m), _lib.ptr(v), n, step, 3e-4, 0.9, 0.999, 1e-8, stream_ptr())
        got = p64.cpu().numpy()
        assert np.array_equal(got, store["w"].data), (step, np.abs(got - store["w"].data).max())
        assert np.array_equal(m.cpu().numpy(), store._m["w"])
        assert np.array_equal(v.cpu().numpy(), store._v["w"])
        assert np.array_equal(p32.cpu().numpy(), got.astype(np.float32))


def _perturb_a(seg_index, layer, arr):  # tests/golden/make_golden.py perturb_a
    return arr + 0.5 if (seg_index == 1 and layer == 0) else arr


def _perturb_b(seg_index, layer, arr):
    return arr * (1.0 - 0.05 * layer) + 0.01 * seg_index


@pytest.mark.parametrize("case", ["small", "default"])
def test_trunk_cache_perturb_matches_reference(case):
    """trunk_forward(cache_perturb=...) (policy.py:137, 170-172): the hook rewrites the
    previous segment's cached states; outputs match the reference's (golden_perturb)
    within 1e-4, and the reference test's own assertions hold
    (test_policy.py:134-149: segment 0 intact, segment 1 and downstream moved)."""
    import json

    from conftest import golden
    from paper_2010_12438_b200 import EmbedConfig, PolicyConfig, init_all_params, randomize_zero_init
    from paper_2010_12438_b200.policy import trunk_forward
    z = golden("perturb")
    p = case + "/"
    meta = json.loads(str(z[p + "meta"]))
    ecfg, pcfg = EmbedConfig(**meta["ecfg"]), PolicyConfig(**meta["pcfg"])
    store = randomize_zero_init(init_all_params(ecfg, pcfg, {"placement": 3}, 0))
    ne, ge = z[p + "node_embed"], z[p + "graph_embed"]
    base = trunk_forward(ne, ge, store, pcfg).data
    assert rel_err(base, z[p + "base"]) < 1e-4
    for tag, fn in (("a", _perturb_a), ("b", _perturb_b)):
        got = trunk_forward(ne, ge, store, pcfg, cache_perturb=fn).data
        assert rel_err(got, z[p + tag]) < 1e-4, (case, tag, rel_err(got, z[p + tag]))
    S = pcfg.segment_len
    bumped = trunk_forward(ne, ge, store, pcfg, cache_perturb=_perturb_a).data
    assert np.allclose(base[:S], bumped[:S], rtol=0, atol=1e-5)
    assert not np.allclose(base[S:2 * S], bumped[S:2 * S])
    assert not np.allclose(base[2 * S:], bumped[2 * S:])


def test_cache_perturb_errors_propagate():
    from paper_2010_12438_b200 import EmbedConfig, PolicyConfig, init_all_params, randomize_zero_init
    from paper_2010_12438_b200.policy import trunk_forward
    ecfg = EmbedConfig(gs_layers=1, gs_dim=8, gs_knn=4)
    pcfg = PolicyConfig(trf_layers=2, d_model=8, n_head=2, d_head=3, d_inner=16, segment_len=4)
    store = randomize_zero_init(init_all_params(ecfg, pcfg, {"placement": 3}, 0))

    def bad(seg, layer, arr):
        raise KeyError("boom")
    with pytest.raises(KeyError):
        trunk_forward(np.ones((12, 8)), np.zeros((1, 8)), store, pcfg, cache_perturb=bad)

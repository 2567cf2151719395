"""Non-learned optimizers (baselines.py:50-237) against golden vectors
from the unmodified reference (tests/golden/make_golden.py baselines): fanout priorities
on the host, brute force and simulated annealing on the device DES (bit-exact step
times, so the argmin and the annealing path are the reference's)."""
import numpy as np
import pytest

from conftest import golden


def _g(z, p):
    from paper_2010_12438_b200.graph import Graph
    return Graph(z[p + "op"], z[p + "flops"], z[p + "out_bytes"], z[p + "src"], z[p + "dst"],
                 z[p + "ebytes"], z[p + "coloc"])


def _topology(z, p):
    from paper_2010_12438_b200.costmodel import Topology
    return Topology(z[p + "top_peak"], z[p + "top_mem_bw"], z[p + "top_cap"], z[p + "top_link_bw"])


def test_fanout_priorities_match_reference():
    from paper_2010_12438_b200.baselines import fanout_priorities
    z = golden("baselines")
    for i in range(int(z["fanout_count"])):
        p = f"f{i}/"
        got = fanout_priorities(_g(z, p))
        assert got.task == "schedule_priority"
        assert np.array_equal(got.actions, z[p + "levels"]), i


def test_sa_config_validation():
    from paper_2010_12438_b200.baselines import SAConfig
    with pytest.raises(ValueError):
        SAConfig(iterations=0)
    with pytest.raises(ValueError):
        SAConfig(cooling_rate=1.0)
    with pytest.raises(ValueError):
        SAConfig(moves_per_step=0)


@pytest.mark.gpu
def test_brute_force_matches_reference():
    from paper_2010_12438_b200.baselines import brute_force
    z = golden("baselines")
    for i in range(int(z["brute_count"])):
        p = f"b{i}/"
        task = str(z[p + "task"])
        best, t = brute_force(_g(z, p), _topology(z, p), task)
        assert t == float(z[p + "time"]), (i, task)
        assert np.array_equal(best.actions, z[p + "actions"]), (i, task)


@pytest.mark.gpu
def test_brute_force_batches_and_limit():
    """Argmin and ties are independent of the device batch size; the search-space
    limit raises ValueError like the reference."""
    from paper_2010_12438_b200.baselines import brute_force
    z = golden("baselines")
    p = "b4/"
    g, top = _g(z, p), _topology(z, p)
    for batch in (1, 7, 64):
        best, t = brute_force(g, top, "placement", batch=batch)
        assert t == float(z[p + "time"])
        assert np.array_equal(best.actions, z[p + "actions"])
    with pytest.raises(ValueError):
        brute_force(g, top, "placement", limit=10)
    with pytest.raises(ValueError):
        brute_force(g, top, "bogus")


@pytest.mark.gpu
def test_simulated_annealing_matches_reference():
    from paper_2010_12438_b200.baselines import SAConfig, simulated_annealing
    z = golden("baselines")
    for i in range(int(z["sa_count"])):
        p = f"a{i}/"
        tasks = [str(t) for t in z[p + "tasks"]]
        res, t = simulated_annealing(_g(z, p), _topology(z, p), tasks,
                                     SAConfig(iterations=300, seed=int(z[p + "seed"]),
                                              cooling_rate=0.99))
        assert t == float(z[p + "time"]), (i, tasks)
        for tk in tasks:
            assert np.array_equal(res[tk].actions, z[p + "actions/" + tk]), (i, tk)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["mbc", "rand", "fuse"])
def test_anneal_chains_each_chain_is_the_reference_chain(case):
    """anneal_chains runs 8 chains at once (on the device for placement / priorities,
    device DES per candidate with host fusion passes for fusion priorities); chain k
    must end exactly where the reference's simulated_annealing with seed k ends
    (golden_sa_chains.npz): same best time, same best actions."""
    import json

    from paper_2010_12438_b200.baselines import SAConfig, anneal_chains
    z = golden("sa_chains")
    p = case + "/"
    tasks = [str(t) for t in z[p + "tasks"]]
    sa = SAConfig(**json.loads(str(z[p + "sa"])))
    out = anneal_chains(_g(z, p), _topology(z, p), tasks, sa, seeds=range(8))
    for seed, (res, t) in enumerate(out):
        assert t == float(z[p + f"s{seed}/time"]), (seed, t)
        for tk in tasks:
            assert np.array_equal(res[tk].actions, z[p + f"s{seed}/{tk}"]), (seed, tk)

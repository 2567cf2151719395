"""Test-only host driver: the reference's training loop (training.py:251-317) and greedy
decode (training.py:320-332) around the device step, so the golden `train` fixture
(tests/golden/make_golden.py make_train, produced by the unmodified reference) can be
checked on the GPU box, where the reference package is absent.

Not product code: in deployment the reference's own `train()` drives the device path
through the INTEGRATION.md shim.  Written against `training.train_step`; the numpy
stream is the reference's (one default_rng(seed); per step the rollout seed, then
the update seed).
"""
from __future__ import annotations

import math

import numpy as np


def run(graphs, topology, tasks, hyper, steps, seed, ecfg, pcfg, fcfg):
    from paper_2010_12438_b200.baselines import baseline_step_time, default_assignments
    from paper_2010_12438_b200.params import init_all_params
    from paper_2010_12438_b200.simulator import evaluate_assignments
    from paper_2010_12438_b200.training import task_action_sizes, train_step
    sizes = task_action_sizes(topology, tasks, fcfg.num_levels)
    store = init_all_params(ecfg, pcfg, sizes, seed)
    baselines = [baseline_step_time(g, topology, fcfg) for g in graphs]
    start = [evaluate_assignments(g, topology, default_assignments(g, topology, fcfg.num_levels),
                                  fcfg) for g in graphs]
    incumbent = [r.step_time if r.valid else math.inf for r in start]
    best_actions = [None] * len(graphs)
    curve, stats_history = [], []
    rng = np.random.default_rng(seed)
    for step in range(steps):
        rollout_seed = int(rng.integers(2**31))
        update_seed = int(rng.integers(2**31))  # drawn after the rollout seed, as there
        batch, stats = train_step(store, graphs, topology, sizes, baselines, hyper, ecfg, pcfg,
                                  fcfg, rollout_seed, update_seed, shard=(0, 1))
        # the reference reads the batch before its update; the batch holds the
        # pre-update results, so reading it afterwards is the same
        for s in batch.samples:
            if s.valid and s.step_time < incumbent[s.graph_index]:
                incumbent[s.graph_index] = s.step_time
                best_actions[s.graph_index] = {k: np.array(v) for k, v in s.bundle.actions.items()}
        stats_history.append(stats)
        fin = [t for t in incumbent if math.isfinite(t)]
        curve.append(float(np.mean(fin)) if fin else math.inf)
    return dict(store=store, baselines=baselines, best_step_times=incumbent,
                best_actions=best_actions, curve=curve, stats_history=stats_history)


def decode_step_time(graph, store, topology, tasks, ecfg, pcfg, fcfg):
    from paper_2010_12438_b200.policy import iterate_decisions
    from paper_2010_12438_b200.simulator import evaluate_assignments
    from paper_2010_12438_b200.training import bundle_assignments, task_action_sizes
    sizes = task_action_sizes(topology, tasks, fcfg.num_levels)
    bundle, _ = iterate_decisions(graph, store, ecfg, pcfg, sizes, pcfg.iterations, seed=0,
                                  temperature=0.0)
    res = evaluate_assignments(graph, topology,
                               bundle_assignments(graph, topology, bundle, sizes, fcfg), fcfg)
    return res.step_time if res.valid else math.inf

#!/usr/bin/env python
"""One PPO step (collect_rollouts + ppo_update, reference defaults: 800 rollouts, 20 epochs
x 40 minibatches) on the cfg1 graph (attention-stack L=10, 101 nodes, 2 devices): the
reference's cfg1 "one PPO step of the reference CPU policy", on the device.
    python scripts/bench_ppo.py [epochs]          # prints one JSON line"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    big = len(sys.argv) > 2 and sys.argv[2] == "cfg4"
    import torch

    from paper_2010_12438_b200 import (EmbedConfig, FusionConfig, PolicyConfig, PPOHyper,
                                       init_all_params, randomize_zero_init, uniform_topology)
    from paper_2010_12438_b200.baselines import baseline_step_time, default_assignments
    from paper_2010_12438_b200.training import collect_rollouts, ppo_update
    from synthetic.workloads import WorkloadSpec, gen_workload
    if big:  # cfg4 graph: per-sample cost of the device backward at 80,001 nodes
        g = gen_workload(WorkloadSpec("attention-stack", 8000, 1, 64, seed=0), node_cap=10**6)
        top = uniform_topology(8)
        sizes = {"placement": 8}
    else:
        g = gen_workload(WorkloadSpec("attention-stack", 10, 1, 64, seed=0))
        top = uniform_topology(2)
        sizes = {"placement": 2}
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
    hyper = PPOHyper(epochs=epochs) if not big else PPOHyper(epochs=epochs, rollouts=4, minibatches=2)
    bl = baseline_step_time(g, top)
    base = [default_assignments(g, top)]
    # warm-up (context, graph upload, kernels)
    nw = 2 if big else 40
    b = collect_rollouts(store, [g], top, sizes, [bl], nw, 1, hyper, ecfg, pcfg, FusionConfig(),
                         base_assignments=base)
    ppo_update(b, store, [g], top, sizes, PPOHyper(epochs=1, minibatches=1, rollouts=nw), ecfg,
               pcfg, seed=0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    batch = collect_rollouts(store, [g], top, sizes, [bl], hyper.rollouts, 7, hyper, ecfg, pcfg,
                             FusionConfig(), base_assignments=base)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    stats = ppo_update(batch, store, [g], top, sizes, hyper, ecfg, pcfg, seed=3)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(json.dumps({"metric": "PPO step (collect + update), " + ("cfg4 graph" if big else "cfg1"), "rollouts": hyper.rollouts,
                      "epochs": hyper.epochs, "minibatches": hyper.minibatches,
                      "collect_s": t1 - t0, "update_s": t2 - t1,
                      "minibatch_updates_per_s": hyper.epochs * hyper.minibatches / (t2 - t1),
                      "stats": {k: float(v) for k, v in stats.items()},
                      "reference_note": "SURVEY.md §8 A18: the reference CPU policy takes 43.8 s "
                                        "per epoch (800 samples, 101 nodes)"}))


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""BASELINE cfg5 training on one B200: the cfg4 graph (attention-stack L=8000, 80,001
nodes, 8 devices) with the joint placement + scheduling + fusion heads (a = 8, 8, 8) and
the reference's default PPOHyper (800 rollouts, 40 minibatches of 20 samples, 20 epochs;
training.py:47-67, 196-233).

Measures one collect_rollouts of the 800 rollouts and `epochs` epochs of ppo_update
(default 1: 40 minibatch forward+backward+Adam steps over 20 x 80,001-node samples each),
the device memory high-water mark, and extrapolates the full 20-epoch PPO step on 1 GPU
and with the owner-computes split over 8 GPUs.
    python scripts/bench_ppo_cfg5.py [epochs] [rollouts]   # one JSON line"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    rollouts = int(sys.argv[2]) if len(sys.argv) > 2 else 800
    import torch

    from paper_2010_12438_b200 import (EmbedConfig, FusionConfig, PolicyConfig, PPOHyper,
                                       init_all_params, randomize_zero_init, uniform_topology)
    from paper_2010_12438_b200.baselines import baseline_step_time, default_assignments
    from paper_2010_12438_b200.training import collect_rollouts, ppo_update
    from synthetic.workloads import WorkloadSpec, gen_workload
    g = gen_workload(WorkloadSpec("attention-stack", 8000, 1, 64, seed=0), node_cap=10**6)
    top = uniform_topology(8)
    sizes = {"placement": 8, "schedule_priority": 8, "fusion_priority": 8}
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
    hyper = PPOHyper(rollouts=rollouts, epochs=epochs)  # minibatches = 40 (default)
    bl = baseline_step_time(g, top)
    base = [default_assignments(g, top)]
    free0, total = torch.cuda.mem_get_info()
    # warm-up: a small collection and a 2-sample update (graph upload, kernels, workspaces)
    b = collect_rollouts(store.clone(), [g], top, sizes, [bl], 2, 1, hyper, ecfg, pcfg,
                         FusionConfig(), base_assignments=base)
    ppo_update(b, store.clone(), [g], top, sizes, PPOHyper(epochs=1, minibatches=1, rollouts=2),
               ecfg, pcfg, seed=0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    batch = collect_rollouts(store, [g], top, sizes, [bl], hyper.rollouts, 7, hyper, ecfg, pcfg,
                             FusionConfig(), base_assignments=base)
    _ = batch.samples  # per-rollout results read back
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    stats = ppo_update(batch, store, [g], top, sizes, hyper, ecfg, pcfg, seed=3)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    free1, _ = torch.cuda.mem_get_info()
    per_epoch = (t2 - t1) / epochs
    mb = hyper.epochs * hyper.minibatches
    samples = hyper.rollouts // hyper.minibatches
    full_1 = (t1 - t0) + 20 * per_epoch
    print(json.dumps({
        "metric": "cfg5 PPO step (collect + update), 80,001 nodes, 3 tasks, default PPOHyper",
        "rollouts": hyper.rollouts, "minibatches": hyper.minibatches, "epochs_measured": epochs,
        "samples_per_minibatch": samples, "collect_s": t1 - t0, "update_s": t2 - t1,
        "seconds_per_epoch": per_epoch,
        "minibatch_steps_per_s": mb / (t2 - t1),
        "sample_fwd_bwd_per_s": mb * samples / (t2 - t1),
        "full_ppo_step_s_1gpu_extrapolated": full_1,
        "full_ppo_step_s_8gpu_extrapolated": (t1 - t0) / 8 + 20 * per_epoch / 8,
        "device_memory_used_gb": (free0 - free1) / 1e9, "device_memory_total_gb": total / 1e9,
        "stats": {k: float(v) for k, v in stats.items()}}))


if __name__ == "__main__":
    main()

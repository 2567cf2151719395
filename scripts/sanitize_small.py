#!/usr/bin/env python
"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel family of the device path on small graphs --
neighbour sampling, embedding GEMMs + segment max, modulation, the mma.sync trunk, the
tcgen05 GEMMs and fused FFN, the fp16 head attention with its per-work-item tf32 fallback
and the online kernel, the sampler, the DES (plain, traced, annealing), and the PPO
forward + backward + Adam.
    compute-sanitizer --tool memcheck python scripts/sanitize_small.py"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2010_12438_b200 import (EmbedConfig, FusionConfig, PolicyConfig, PPOHyper,
                                       init_all_params, randomize_zero_init, uniform_topology)
    from paper_2010_12438_b200.baselines import (SAConfig, anneal_chains, baseline_step_time,
                                                 default_assignments)
    from paper_2010_12438_b200.policy import task_heads
    from paper_2010_12438_b200.simulator import ActionAssignment, simulate, singleton_fused
    from paper_2010_12438_b200.training import collect_rollouts, ppo_update
    from synthetic.workloads import WorkloadSpec, gen_workload
    g = gen_workload(WorkloadSpec("attention-stack", 12, 1, 64, seed=0))  # 121 nodes
    top = uniform_topology(4)
    sizes = {"placement": 4, "schedule_priority": 8, "fusion_priority": 8}
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
    bl = baseline_step_time(g, top)
    base = [default_assignments(g, top)]
    hyper = PPOHyper(rollouts=4, minibatches=2, epochs=1)
    batch = collect_rollouts(store, [g], top, sizes, [bl], 4, 3, hyper, ecfg, pcfg,
                             FusionConfig(), base_assignments=base)
    ppo_update(batch, store, [g], top, sizes, hyper, ecfg, pcfg, seed=1)
    # head attention: fp16 kernel, per-work-item tf32 fallback, online kernel
    rng = np.random.default_rng(0)
    hid = rng.normal(size=(900, pcfg.d_model))
    for scale in (1.0, 3.0, 8.0):
        s2 = store.clone()
        s2["policy/task_attn/q_w"].data = s2["policy/task_attn/q_w"].data * scale
        task_heads(hid, s2, pcfg, [("placement", 4)])
    # DES: traced single placement and device annealing chains
    pl = ActionAssignment("placement", rng.integers(0, 4, g.num_nodes), 4)
    pr = ActionAssignment("schedule_priority", rng.integers(0, 8, g.num_nodes), 8)
    simulate(singleton_fused(g), pl, pr, top, record_trace=True)
    anneal_chains(g, top, ["placement"], SAConfig(iterations=20), seeds=range(4))
    torch.cuda.synchronize()
    print("sanitize workload done")


if __name__ == "__main__":
    main()

"""Worker for tests/test_gpu_multirank.py: one rank of a sharded device training step
(training.train_step) on cuda:0.  Env: RANK, WORLD_SIZE, MASTER_ADDR, MASTER_PORT,
GO_MR_OUT (npz path written by rank 0)."""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    import torch
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(0)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2010_12438_b200 import (EmbedConfig, FusionConfig, PolicyConfig, PPOHyper,
                                       init_all_params, randomize_zero_init, uniform_topology)
    from paper_2010_12438_b200.baselines import baseline_step_time
    from paper_2010_12438_b200.training import train_step
    from synthetic.workloads import WorkloadSpec, gen_workload
    graphs = [gen_workload(WorkloadSpec("attention-stack", 10, 1, 64, seed=0)),
              gen_workload(WorkloadSpec("dilated-stack", 2, 50, 64, seed=3))]
    top = uniform_topology(2)
    sizes = {"placement": 2}
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
    hyper = PPOHyper(rollouts=10, minibatches=3, epochs=2, lr=3e-4)
    bls = [baseline_step_time(g, top) for g in graphs]
    batch, stats = train_step(store, graphs, top, sizes, bls, hyper, ecfg, pcfg, FusionConfig(),
                              rollout_seed=5, update_seed=9,
                              shard=(rank, world) if world > 1 else None)
    if world > 1:
        rw = batch.global_rewards.cpu().numpy()
        st = batch.global_step_times.cpu().numpy()
        lo, hi = batch.shard
        assert hi - lo < hyper.rollouts  # really sharded
    else:
        rw = batch.rewards.cpu().numpy()
        st = batch.step_times.cpu().numpy()
    if rank == 0:
        out = {"rewards": rw, "step_times": st, "step_count": store.step_count}
        out.update({f"stat/{k}": v for k, v in stats.items()})
        out.update({f"p/{n}": p.data for n, p in store.items()})
        np.savez(os.environ["GO_MR_OUT"], **out)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

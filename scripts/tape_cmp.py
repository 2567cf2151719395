"""Loss / gradient of one cfg4 PPO sample under the tape modes (GO_TRAIN_ATTN, GO_TRAIN_GEMM)."""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))


def main():
    import torch
    from paper_2010_12438_b200 import (EmbedConfig, FusionConfig, PolicyConfig, PPOHyper,
                                       init_all_params, randomize_zero_init, uniform_topology)
    from paper_2010_12438_b200.baselines import baseline_step_time
    from paper_2010_12438_b200.params import pack
    from paper_2010_12438_b200.policy import ordered_tasks
    from paper_2010_12438_b200.training import _device_samples, collect_rollouts, ppo_grad
    from synthetic.workloads import WorkloadSpec, gen_workload
    L = int(sys.argv[1]) if len(sys.argv) > 1 else 8000
    g = gen_workload(WorkloadSpec("attention-stack", L, 1, 64, seed=0), node_cap=10**6)
    top = uniform_topology(8)
    sizes = {"placement": 8}
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
    batch = collect_rollouts(store, [g], top, sizes, [baseline_step_time(g, top)], 1, 3,
                             PPOHyper(rollouts=1), ecfg, pcfg, FusionConfig())
    res = {}
    for mode in ["simt/simt", "simt/tc", "tc/simt", "tc/tc"]:
        at, gm = mode.split("/")
        for k in ("GO_TRAIN_ATTN", "GO_TRAIN_GEMM"):
            os.environ.pop(k, None)
        if at == "simt":
            os.environ["GO_TRAIN_ATTN"] = "simt"
        if gm == "simt":
            os.environ["GO_TRAIN_GEMM"] = "simt"
        blob_h, offs = pack(store, ecfg, pcfg, sizes)
        blob = torch.as_tensor(blob_h, device="cuda")
        samples = _device_samples(batch, [g], ordered_tasks(sizes))
        grads = torch.zeros_like(blob)
        adv = np.array([s.advantage for s in batch.samples])
        loss, _ = ppo_grad((blob, offs), ecfg, pcfg, sizes, samples, adv, PPOHyper(), grads)
        res[mode] = (loss, grads.cpu().numpy().astype(np.float64))
    if len(sys.argv) > 2:  # dump the sample + losses for a float64 oracle check on the CPU
        b = batch.samples[0].bundle
        np.savez(sys.argv[2], L=L, actions=b.actions["placement"],
                 prev=b.prev_actions["placement"], logp=b.log_probs["placement"],
                 embed_seed=b.embed_seed, temperature=b.temperature,
                 reward=batch.samples[0].reward, advantage=batch.samples[0].advantage,
                 **{"loss_" + m.replace("/", "_"): v[0] for m, v in res.items()})
    l0, g0 = res["simt/simt"]
    for m, (l, gr) in res.items():
        print(m, "loss", repr(l), "dloss", (l - l0) / abs(l0),
              "grad rel", np.linalg.norm(gr - g0) / np.linalg.norm(g0))


if __name__ == "__main__":
    main()

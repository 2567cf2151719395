"""One cfg4-size PPO minibatch (1 sample), for kernel launch lists (development aid)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from paper_2010_12438_b200 import (EmbedConfig, FusionConfig, PolicyConfig, PPOHyper,  # noqa: E402
                                   init_all_params, randomize_zero_init, uniform_topology)
from paper_2010_12438_b200.baselines import baseline_step_time, default_assignments  # noqa: E402
from paper_2010_12438_b200.training import collect_rollouts, ppo_update  # noqa: E402
from synthetic.workloads import WorkloadSpec, gen_workload  # noqa: E402

g = gen_workload(WorkloadSpec("attention-stack", 8000, 1, 64, seed=0), node_cap=10**6)
top = uniform_topology(8)
sizes = {"placement": 8}
ecfg, pcfg = EmbedConfig(), PolicyConfig()
store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
bl = baseline_step_time(g, top)
hyper = PPOHyper(epochs=1, minibatches=1, rollouts=1)
b = collect_rollouts(store, [g], top, sizes, [bl], 1, 1, hyper, ecfg, pcfg, FusionConfig(),
                     base_assignments=[default_assignments(g, top)])
ppo_update(b, store, [g], top, sizes, hyper, ecfg, pcfg, seed=0)
torch.cuda.synchronize()
print("ok")

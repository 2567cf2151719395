"""Time the UNMODIFIED reference (graphopt, pip-installed into baseline/_ref from
/root/reference, git-ignored, travels to the GPU box with the snapshot) on the host
cores, next to the float64 oracle port bench.py's reference arm uses, so the port's
speed relative to the reference is measured rather than assumed (
BASELINE.md §2).

  cfg1  attention-stack L=10 (101 nodes), 2 devices: collect_rollouts of K rollouts
        (training.py:114-143; base_assignments precomputed, a reference-API argument)
  cfg2  multi-branch-cnn (13,000 nodes), 4 devices: collect_rollouts of 1 rollout
        (the reference keeps ~88 N^2 bytes of tape for the heads: 14.8 GB at 13k)

each at all BLAS threads and at 1 thread, and the port on the same work.
Usage: python scripts/ref_cpu_timing.py [cfg1 cfg2] > profiles/r2_cpu_reference.json
"""
import json
import os
import platform
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path[:0] = [str(ROOT), str(ROOT / "baseline" / "_ref")]


def host():
    model = ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
        mem = [l for l in open("/proc/meminfo") if l.startswith("MemTotal")][0].split()[1]
        mem_gb = int(mem) / 1e6
    except OSError:
        mem_gb = None
    return {"cpu_model": model, "logical_cpus": os.cpu_count(), "ram_gb": mem_gb,
            "python": platform.python_version(), "numpy": np.__version__}


def reference_collect(spec, d, count, seed=0):
    from graphopt.baselines import baseline_step_time, default_assignments
    from graphopt.costmodel import uniform_topology
    from graphopt.embedding import EmbedConfig
    from graphopt.policy import PolicyConfig, init_all_params
    from graphopt.simulator import FusionConfig
    from graphopt.training import PPOHyper, collect_rollouts, task_action_sizes
    from graphopt.workloads import WorkloadSpec, gen_workload
    g = gen_workload(WorkloadSpec(*spec[:4], seed=spec[4]), node_cap=10**6)
    top = uniform_topology(d)
    sizes = task_action_sizes(top, ["placement"], 8)
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = init_all_params(ecfg, pcfg, sizes, seed=0)
    rng = np.random.default_rng(1)  # the benchmark weights
    for name in store.names():
        t = store[name]
        if not np.any(t.data):
            s = 1.0 / np.sqrt(max(1, t.data.shape[0]))
            t.data = rng.uniform(-s, s, size=t.data.shape)
    base = [default_assignments(g, top)]
    bl = [baseline_step_time(g, top)]
    t0 = time.perf_counter()
    batch = collect_rollouts(store, [g], top, sizes, bl, count, seed, PPOHyper(rollouts=count),
                             ecfg, pcfg, FusionConfig(), base_assignments=base)
    dt = time.perf_counter() - t0
    return dt, g.num_nodes, [s.step_time for s in batch.samples]


def port_rollouts(spec, d, count, seed=0):
    """The oracle port on the same rollouts: iterate_decisions (2 forwards, full heads)
    + DES per rollout, outer stream as training.py:122-126."""
    from oracle import des as od
    from oracle import forward as of
    from oracle import graph as og
    from oracle import params as op
    from synthetic.workloads import WorkloadSpec, gen_workload
    g = gen_workload(WorkloadSpec(*spec[:4], seed=spec[4]), node_cap=10**6)
    ogr = og.make(g.num_nodes, g.op, g.flops, g.out_bytes, g.src, g.dst, g.ebytes)
    sizes = {"placement": d}
    P = op.randomize_zero_init(op.init_all_params(of.EmbedCfg(), of.PolicyCfg(), sizes, 0))
    top = od.uniform_topology(d)
    fg = od.singleton(ogr)
    rng = np.random.default_rng(seed)
    t0 = time.perf_counter()
    steps = []
    for _ in range(count):
        rng.integers(1)
        s = int(rng.integers(2**31))
        traj = of.iterate_decisions(ogr, P, of.EmbedCfg(), of.PolicyCfg(), sizes, 2, s)
        res = od.simulate(ogr, fg, traj[-1]["actions"]["placement"], np.zeros(ogr["n"]), top)
        steps.append(res["step_time"])
    return time.perf_counter() - t0, steps


def main(names):
    from threadpoolctl import threadpool_info, threadpool_limits
    out = {"host": host(), "blas": [{k: i.get(k) for k in ("internal_api", "num_threads",
                                                            "version")}
                                    for i in threadpool_info()]}
    cases = {"cfg1": (("attention-stack", 10, 1, 64, 0), 2, 64),
             "cfg2": (("multi-branch-cnn", 1857, 1, 64, 0), 4, 1)}
    for name in names:
        spec, d, count = cases[name]
        rec = {"rollouts": count}
        for label, limit in (("all_threads", None), ("one_thread", 1)):
            with threadpool_limits(limits=limit):
                dt, n, st_ref = reference_collect(spec, d, count)
                dp, st_port = port_rollouts(spec, d, count)
            rec[label] = {"reference_s": dt, "reference_placements_per_s": count / dt,
                          "port_s": dp, "port_placements_per_s": count / dp,
                          "port_speedup_over_reference": dt / dp,
                          "same_step_times": bool(st_ref == st_port)}
            print(name, label, rec[label], file=sys.stderr, flush=True)
        rec["nodes"] = n
        out[name] = rec
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg1", "cfg2"])

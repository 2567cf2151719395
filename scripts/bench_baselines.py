#!/usr/bin/env python
"""Throughput of the device brute-force search next to the CPU oracle
DES (the reference algorithm restated, one simulate() per combination, as the
reference's brute_force does) on a bounded sample of the same combinations.

    python scripts/bench_baselines.py [n_nodes] [devices]     # prints one JSON line"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
    d = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    import torch

    from paper_2010_12438_b200.baselines import brute_force
    from paper_2010_12438_b200.costmodel import uniform_topology
    from synthetic.workloads import WorkloadSpec, gen_workload
    g = gen_workload(WorkloadSpec("attention-stack", 1, 1, 64, seed=0), node_cap=10**6)
    if g.num_nodes != n:  # a random DAG of exactly n nodes otherwise
        from paper_2010_12438_b200.graph import Graph
        rng = np.random.default_rng(0)
        src, dst = [], []
        for v in range(1, n):
            for u in rng.choice(v, size=min(v, 2), replace=False):
                src.append(int(u))
                dst.append(v)
        g = Graph(np.full(n, 1), rng.uniform(1e8, 1e10, n), rng.uniform(1e5, 1e7, n),
                  src, dst, rng.uniform(1e5, 1e7, len(src)))
    top = uniform_topology(d)
    total = d ** n
    brute_force(g, top, "placement", limit=total)  # warm-up (graph upload, context)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    best, t = brute_force(g, top, "placement", limit=total)
    torch.cuda.synchronize()
    gpu_s = time.perf_counter() - t0
    # CPU: the oracle DES on a bounded sample of the same combinations
    from oracle import des as od
    from oracle import graph as og
    ogr = og.make(g.num_nodes, g.op, g.flops, g.out_bytes, g.src, g.dst, g.ebytes)
    fg = od.singleton(ogr)
    otop = od.uniform_topology(d)
    sample = min(total, 2000)
    t0 = time.perf_counter()
    for i in range(sample):
        pl = np.array([(i // d ** (n - 1 - j)) % d for j in range(n)], np.int64)
        od.simulate(ogr, fg, pl, np.zeros(n, np.int64), otop)
    cpu_s = (time.perf_counter() - t0) * total / sample
    print(json.dumps({"metric": "brute-force placements scored/s", "nodes": n, "devices": d,
                      "combinations": total, "gpu_seconds": gpu_s,
                      "gpu_value": total / gpu_s, "cpu_oracle_value": total / cpu_s,
                      "cpu_sample": f"{sample} combinations, scaled", "best_time": t,
                      "best_actions": best.actions.tolist()}))


if __name__ == "__main__":
    main()

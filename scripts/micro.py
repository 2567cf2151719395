#!/usr/bin/env python
"""Micro-benchmarks on one GPU (development aid, not the headline bench):
  des      : batched DES throughput on the cfg4 graph (random placements)
  forward  : one wave of cfg4 forwards, per-kernel-class CUDA-event times
  attn     : forward with the fp16 / tf32 head-attention kernels (GO_ATTN)
Usage: python scripts/micro.py des|forward|poly [K]"""
import ctypes as C
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def cfg4():
    from synthetic.workloads import WorkloadSpec, gen_workload
    return gen_workload(WorkloadSpec("attention-stack", 8000, 1, 64, seed=0), node_cap=10**6)


def des(K):
    from paper_2010_12438_b200.costmodel import uniform_topology
    from paper_2010_12438_b200.simulator import simulate_many, singleton_fused
    g = cfg4()
    rng = np.random.default_rng(0)
    pl = torch.as_tensor(rng.integers(0, 8, (K, g.num_nodes)), dtype=torch.int32, device="cuda")
    pr = torch.zeros(g.num_nodes, dtype=torch.int32, device="cuda")
    fg = singleton_fused(g)
    top = uniform_topology(8)
    simulate_many(fg, pl[:32], pr, top)
    simulate_many(fg, pl, pr, top)  # workspace sized for K
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = simulate_many(fg, pl, pr, top)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"DES K={K}: {dt*1e3:.1f} ms  ({K/dt:.1f} placements/s)  "
          f"step[0]={float(r.step_time[0]):.6g}", flush=True)


def forward(F, modes=("tc", "simt"), env=None):
    from paper_2010_12438_b200 import EmbedConfig, PolicyConfig, init_all_params, randomize_zero_init
    from paper_2010_12438_b200 import _lib
    from paper_2010_12438_b200.engine import forward_batch
    from paper_2010_12438_b200.runtime import context
    g = cfg4()
    sizes = {"placement": 8}
    ecfg, pcfg = EmbedConfig(), PolicyConfig()
    store = randomize_zero_init(init_all_params(ecfg, pcfg, sizes, 0))
    ctx = context()
    hs = [ctx.graph(g)] * F
    names = ["heads_attn", "trunk_attn", "segmax", "gemm", "des", "sample", "neighbor", "other"]
    runs = [(m, None) for m in modes] if env is None else [(modes[0], e) for e in env]
    for mode, ev in runs:
        os.environ["GO_GEMM"] = mode
        if ev:
            os.environ[ev[0]] = ev[1]
        forward_batch(store, ecfg, pcfg, sizes, hs, list(range(F)))
        torch.cuda.synchronize()
        _lib.call("go_ctx_set_timing", ctx.handle, 1)
        t0 = time.perf_counter()
        out = forward_batch(store, ecfg, pcfg, sizes, hs, list(range(F)))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        parts = []
        for i, nm in enumerate(names):
            cnt, ms, work = C.c_int64(), C.c_double(), C.c_double()
            _lib.call("go_ctx_kernel_stats", ctx.handle, i, C.byref(cnt), C.byref(ms), C.byref(work))
            if cnt.value:
                rate = work.value / (ms.value / 1e3)
                parts.append(f"{nm}={ms.value:.1f}ms({rate/1e12:.1f}T/s)")
        _lib.call("go_ctx_set_timing", ctx.handle, 0)
        print(f"forward GEMM={mode} {ev or ''} F={F}: {dt*1e3:.1f} ms total ({dt*1e3/F:.2f} ms/forward) "
              + " ".join(parts), flush=True)
        lg = out.logits[0].float()
        print("  logits checksum", float(lg.sum()), float(lg.abs().max()), flush=True)
        if os.environ.get("GO_SAVE_LOGITS"):
            torch.save(out.logits[0].float().cpu(), os.environ["GO_SAVE_LOGITS"])


if __name__ == "__main__":
    what = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    if what == "des":
        des(n or 512)
    elif what == "attn":
        forward(n or 8, env=[("GO_ATTN", "f16"), ("GO_ATTN", "tf32"), ("GO_ATTN", "f16")])
    elif what == "tc":
        forward(n or 8, modes=("tc",))
    else:
        forward(n or 8)

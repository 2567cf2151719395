"""Sharded rollouts composed with the owner-computes PPO update, with the REAL device
compute (VERDICT r1 "next" #3): two ranks (processes) on cuda:0 over
gloo run training.train_step -- each decides and scores its own global rollouts, the
per-rollout results are all-gathered, advantages are normalised over all rollouts,
each minibatch member's forward+backward runs on the rank that collected it and the
gradients are all-reduced -- against the same step in one process.

Rollout results must be bit-identical to the single-process run (the rollouts are
independent and seeded per global rollout id).  Parameters after the update agree to
the summation-order tolerance of the gradient all-reduce: |d| <= 1e-5 on >= 99.9% of
coordinates (Adam's first steps are ~lr*sign(g), so a near-zero gradient summed in a
different order can move a coordinate by up to 2*lr)."""
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = Path(__file__).resolve().parent


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(world, out):
    port = _port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1",
                   MASTER_PORT=str(port), GO_MR_OUT=str(out))
        procs.append(subprocess.Popen([sys.executable, str(HERE / "mr_worker.py")], env=env))
    for p in procs:
        assert p.wait(timeout=600) == 0
    return dict(np.load(out))


def test_sharded_collect_and_ppo_match_single_process(tmp_path):
    one = _run(1, tmp_path / "w1.npz")
    two = _run(2, tmp_path / "w2.npz")
    assert np.array_equal(one["rewards"], two["rewards"])
    assert np.array_equal(one["step_times"], two["step_times"])
    assert int(one["step_count"]) == int(two["step_count"]) == 6
    for k in ("mean_ratio", "clip_fraction", "entropy", "value_loss"):
        a, b = float(one["stat/" + k]), float(two["stat/" + k])
        assert abs(a - b) <= 1e-5 * max(1.0, abs(a)), (k, a, b)
    d = np.concatenate([np.abs(one[k] - two[k]).reshape(-1) for k in one if k.startswith("p/")])
    assert (d <= 1e-5).mean() >= 0.999, (d.max(), (d <= 1e-5).mean())

"""World-size-2 gloo test (CPU) of the multi-rank scoring logic: every rank draws the
same outer rollout stream (training.py:122-126), scores only its contiguous shard, and
the per-rollout results are all-gathered back into global rollout order."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, count, seed, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2010_12438_b200.training import gather_results, outer_draws, shard_bounds
        gi, seeds = outer_draws(seed, count, 3)
        lo, hi = shard_bounds(count, rank, world)
        # stand-in for the device scoring: a deterministic function of the rollout
        reward = -np.sqrt((seeds[lo:hi] % 1000) / 1000.0 + 1.0)
        step = seeds[lo:hi].astype(np.float64) * 1e-6
        packed = torch.tensor(np.stack([reward, step, gi[lo:hi].astype(np.float64)]))
        full = gather_results(packed, count, world)
        out[rank] = full.numpy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("count", [7, 64])
def test_sharded_scoring_gather_world2(count):
    world, seed = 2, 123
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), count, seed, out), nprocs=world, join=True)
    from paper_2010_12438_b200.training import outer_draws, shard_bounds
    gi, seeds = outer_draws(seed, count, 3)
    want = np.stack([-np.sqrt((seeds % 1000) / 1000.0 + 1.0), seeds * 1e-6, gi.astype(np.float64)])
    for r in range(world):
        assert np.array_equal(out[r], want)
    covered = np.concatenate([np.arange(*shard_bounds(count, r, world)) for r in range(world)])
    assert np.array_equal(covered, np.arange(count))


def test_outer_draws_match_reference_stream():
    """Same numpy calls in the same order as training.py:122-126."""
    from paper_2010_12438_b200.training import outer_draws
    gi, seeds = outer_draws(0, 6, 1)
    rng = np.random.default_rng(0)
    for k in range(6):
        assert gi[k] == int(rng.integers(1))
        assert seeds[k] == int(rng.integers(2**31))


def _ppo_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2010_12438_b200.training import allreduce_sum, rank_share
        chunk = np.array([7, 3, 11, 0, 5])
        mine = rank_share(chunk, rank, world)
        # per-sample "gradient" = sample id * ones; loss = sample id; divided by |chunk|
        g = torch.zeros(4, dtype=torch.float32)
        loss = 0.0
        for k in mine:
            g += float(k) / len(chunk)
            loss += float(k) / len(chunk)
        loss = allreduce_sum(g, loss)
        out[rank] = (sorted(int(k) for k in mine), g.numpy().tolist(), loss)
    finally:
        dist.destroy_process_group()


def test_ppo_minibatch_split_and_allreduce_world2():
    """Owner-computes split of a minibatch over 2 ranks + all-reduce(sum) of the
    partial gradients equals the single-rank minibatch mean on every rank."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_ppo_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    owned = sorted(out[0][0] + out[1][0])
    assert owned == [0, 3, 5, 7, 11]
    want = sum([7, 3, 11, 0, 5]) / 5
    for r in range(world):
        assert np.allclose(out[r][1], [want] * 4)
        assert abs(out[r][2] - want) < 1e-12

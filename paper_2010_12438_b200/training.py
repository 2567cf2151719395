"""Rollout collection (and the PPO update) on the B200 (mirrors training.py:1-384).

collect_rollouts keeps the reference signature and per-sample fields; underneath,
all K rollouts are decided in waves of batched forwards (iteration-major: every
rollout's iteration-1 forward, sample, then iteration-2 ...) and all placements
of a graph are scored by ONE batched DES launch with the reward fused in.
Results stay on the device until a field is read.
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

from .baselines import default_assignments
from .config import INVALID_REWARD, EmbedConfig, FusionConfig, PolicyConfig, PPOHyper, ordered_tasks
from .engine import (DeviceArray, advance, check_status, forward_batch, params_on_device,
                     pcg_words, sample_batch)
from .graph import as_graph
from .policy import TaskActionBundle
from .runtime import context, torch
from .simulator import ActionAssignment, FusedGraph, apply_fusion, simulate_many

__all__ = ["Reward", "reward", "PPOHyper", "RolloutSample", "RolloutBatch", "task_action_sizes",
           "bundle_assignments", "collect_rollouts", "run_decisions", "INVALID_REWARD",
           "ppo_update", "TrainResult", "train", "decode_step_time", "pretrain_finetune_zeroshot"]


@dataclass(frozen=True)
class Reward:
    value: float
    source: str  # "measured" | "invalid"


def reward(step_time: float, baseline_time: float, valid: bool) -> Reward:
    """training.py:37-44 (the batched path computes the same value in des.cu)."""
    if baseline_time <= 0:
        raise ValueError("baseline_time must be positive")
    if not valid:
        return Reward(INVALID_REWARD, "invalid")
    return Reward(-math.sqrt(step_time / baseline_time), "measured")


def task_action_sizes(topology, tasks, num_levels: int) -> dict:
    """training.py:93-98."""
    from .costmodel import as_topology
    d = as_topology(topology).num_devices
    return {t: (d if t == "placement" else num_levels) for t in tasks}


def bundle_assignments(graph, topology, bundle, task_sizes, fusion_cfg, base=None) -> dict:
    """training.py:101-111."""
    asg = dict(base) if base else default_assignments(graph, topology, fusion_cfg.num_levels)
    for task, a in task_sizes.items():
        asg[task] = ActionAssignment(task, bundle.actions[task], a)
    return asg


# ---------------------------------------------------------------------------------------
# decisions

def _wave_rows() -> int:
    return int(os.environ.get("GO_WAVE_ROWS", str(1 << 21)))


def _waves(sizes, max_rows):
    waves, cur, rows = [], [], 0
    for i, n in enumerate(sizes):
        if cur and rows + n > max_rows:
            waves.append(cur)
            cur, rows = [], 0
        cur.append(i)
        rows += n
    if cur:
        waves.append(cur)
    return waves


class DecisionWave:
    """Device results of one wave of rollouts (all tensors on device).
    actions/prev: int32 [T, R] node-indexed per rollout span; logp f64 [T, R]."""

    def __init__(self, idx, handles, row_off):
        self.idx = idx
        self.handles = handles
        self.row_off = row_off
        self.iters = []  # per iteration dict(actions, logp, value, logits)


def decide(store, graphs, embed_cfg, cfg, task_sizes, iterations, seeds, temperature,
           keep_logits=True, keep_trajectory=False, params=None):
    """Batched iterate_decisions over rollouts (graphs[k], seeds[k]).  Returns a list
    of DecisionWave covering all rollouts in order."""
    ctx = context()
    handles = [ctx.graph(g) for g in graphs]
    tasks = ordered_tasks(task_sizes)
    params = params or params_on_device(store, embed_cfg, cfg, task_sizes)
    out_waves = []
    statuses = []
    for idx in _waves([h.n for h in handles], _wave_rows()):
        hs = [handles[i] for i in idx]
        sd = [int(seeds[i]) for i in idx]
        rngs = [np.random.default_rng(s) for s in sd]
        row_off = np.zeros(len(idx) + 1, np.int64)
        row_off[1:] = np.cumsum([h.n for h in hs])
        wave = DecisionWave(idx, hs, row_off)
        prev = None
        for it in range(iterations):
            out = forward_batch(store, embed_cfg, cfg, task_sizes, hs, sd, prev_actions=prev,
                                params=params)
            statuses.append(out.status)
            acts, logp = sample_batch(embed_cfg, cfg, task_sizes, hs, [pcg_words(r) for r in rngs],
                                      out.logits_packed, temperature)
            if temperature > 0:
                for r, h in zip(rngs, hs):
                    advance(r, len(tasks) * h.n)
            rec = dict(actions=acts, logp=logp, value=out.value, prev=prev,
                       logits=out.logits if keep_logits else None)
            if keep_trajectory or it == iterations - 1:
                wave.iters.append(rec)
            prev = acts
        out_waves.append(wave)
    for s in statuses:
        if int(s.item()) & 1:
            raise FloatingPointError("non-finite node embeddings (bad init or features)")
    return out_waves


def _bundle(wave, rec, j, tasks, seed, temperature, order):
    lo, hi = int(wave.row_off[j]), int(wave.row_off[j + 1])
    acts = rec["actions"][:, lo:hi].cpu().numpy().astype(np.int64)
    logp = rec["logp"][:, lo:hi].cpu().numpy()
    prev = None
    if rec["prev"] is not None:
        pv = rec["prev"][:, lo:hi].cpu().numpy().astype(np.int64)
        prev = {t: pv[i].copy() for i, (t, _a) in enumerate(tasks)}
    logits = {}
    if rec["logits"] is not None:
        for i, (t, _a) in enumerate(tasks):
            logits[t] = rec["logits"][i][lo:hi].cpu().numpy().astype(np.float64)
    return TaskActionBundle(
        tasks=[t for t, _ in tasks], logits=logits,
        actions={t: acts[i] for i, (t, _a) in enumerate(tasks)},
        log_probs={t: logp[i] for i, (t, _a) in enumerate(tasks)},
        value=float(rec["value"][j].item()), prev_actions=prev, embed_seed=int(seed),
        temperature=temperature)


def run_decisions(store, graphs, embed_cfg, cfg, task_sizes, iterations, seeds, temperature=1.0,
                  keep_trajectory=False):
    """Host bundles per rollout: list (per rollout) of per-iteration bundles."""
    tasks = ordered_tasks(task_sizes)
    waves = decide(store, graphs, embed_cfg, cfg, task_sizes, iterations, seeds, temperature,
                   keep_logits=True, keep_trajectory=keep_trajectory)
    out = [None] * len(graphs)
    for w in waves:
        for j, k in enumerate(w.idx):
            out[k] = [_bundle(w, rec, j, tasks, seeds[k], temperature, None) for rec in w.iters]
    return out


# ---------------------------------------------------------------------------------------
# rollouts

@dataclass
class RolloutSample:
    graph_index: int
    bundle: object
    reward: float
    value_estimate: float
    advantage: float
    step_time: float
    valid: bool


class LazyBundle:
    """TaskActionBundle view over device results; arrays are fetched on access."""

    def __init__(self, batch, k):
        self._b, self._k = batch, k
        self._cache = None

    def _get(self):
        if self._cache is None:
            b = self._b
            w, j = b._loc[self._k]
            self._cache = _bundle(b._waves[w], b._waves[w].iters[-1], j, b._tasks, b.seeds[self._k],
                                  b.temperature, None)
        return self._cache

    def __getattr__(self, name):
        if name.startswith("_"):
            raise AttributeError(name)
        return getattr(self._get(), name)


class RolloutBatch:
    """training.py:79-90 with device-resident per-rollout results."""

    def __init__(self, samples=None):
        self._samples = samples
        self.rewards = None

    @property
    def samples(self) -> list:
        if self._samples is None:
            self._materialize()
        return self._samples

    def _materialize(self):
        r = self.rewards.cpu().numpy()
        st = self.step_times.cpu().numpy()
        va = self.valid.cpu().numpy().astype(bool)
        vals = self.values.cpu().numpy().astype(np.float64)
        self._samples = [RolloutSample(graph_index=int(self.graph_index[k]),
                                       bundle=LazyBundle(self, k), reward=float(r[k]),
                                       value_estimate=float(vals[k]),
                                       advantage=float(r[k] - vals[k]), step_time=float(st[k]),
                                       valid=bool(va[k]))
                         for k in range(len(r))]

    @property
    def mean_reward(self) -> float:
        return float(np.mean([s.reward for s in self.samples]))

    def any_valid(self) -> bool:
        return any(s.valid for s in self.samples)


def outer_draws(seed: int, count: int, num_graphs: int):
    """training.py:122-126: per rollout, graph index then sample seed, from one
    numpy stream (host; identical on every rank)."""
    rng = np.random.default_rng(seed)
    gi = np.empty(count, np.int64)
    seeds = np.empty(count, np.int64)
    for k in range(count):
        gi[k] = int(rng.integers(num_graphs))
        seeds[k] = int(rng.integers(2**31))
    return gi, seeds


def shard_bounds(count: int, rank: int, world: int):
    """Contiguous shard of global rollout ids owned by `rank`."""
    return rank * count // world, (rank + 1) * count // world


def gather_results(packed, count: int, world: int):
    """All-gather per-rollout result columns ([C, local] tensors) from every rank into
    [C, count] in global rollout order -- the one collective of the scoring path
    (NCCL on GPUs, gloo in the CPU tests)."""
    import torch.distributed as dist
    T = torch()
    sizes = [shard_bounds(count, q, world)[1] - shard_bounds(count, q, world)[0]
             for q in range(world)]
    mx = max(sizes)
    pad = T.zeros((packed.shape[0], mx), dtype=packed.dtype, device=packed.device)
    pad[:, :packed.shape[1]] = packed
    bufs = [T.empty_like(pad) for _ in sizes]
    dist.all_gather(bufs, pad)
    return T.cat([b[:, :s] for b, s in zip(bufs, sizes)], dim=1)


def collect_rollouts(store, graphs, topology, task_sizes, baselines, count, seed, hyper,
                     embed_cfg, policy_cfg, fusion_cfg, base_assignments=None,
                     keep_logits: bool = True, shard=None) -> RolloutBatch:
    """training.py:114-143: `count` independent decision bundles, graphs drawn
    uniformly by the same outer numpy stream; all scored on device.

    shard=(rank, world) scores only global rollouts [rank*count/world,
    (rank+1)*count/world) (rollouts are independent, no
    communication while scoring); when torch.distributed is initialised the
    per-rollout results are then all-gathered (NCCL) into batch.global_*."""
    T = torch()
    dev = T.device("cuda", context().device)
    graphs = [as_graph(g) for g in graphs]
    gi_all, seeds_all = outer_draws(seed, count, len(graphs))
    lo, hi = shard_bounds(count, *(shard or (0, 1)))
    gi, seeds = gi_all[lo:hi], seeds_all[lo:hi]
    count = hi - lo
    tasks = ordered_tasks(task_sizes)
    waves = decide(store, [graphs[i] for i in gi], embed_cfg, policy_cfg, task_sizes,
                   policy_cfg.iterations, seeds, hyper.temperature, keep_logits=keep_logits)
    batch = RolloutBatch()
    batch._waves, batch._tasks, batch.seeds, batch.temperature = waves, tasks, seeds, hyper.temperature
    batch.graph_index = gi
    batch._loc = [None] * count
    for w_i, w in enumerate(waves):
        for j, k in enumerate(w.idx):
            batch._loc[k] = (w_i, j)
    tnames = [t for t, _ in tasks]
    rewards = T.empty(count, dtype=T.float64, device=dev)
    steps = T.empty(count, dtype=T.float64, device=dev)
    valid = T.empty(count, dtype=T.uint8, device=dev)
    values = T.empty(count, dtype=T.float32, device=dev)
    for w in waves:
        rec = w.iters[-1]
        ix = T.as_tensor(np.asarray(w.idx, np.int64), device=dev)
        values[ix] = rec["value"]
    for g_i, g in enumerate(graphs):
        ks = np.flatnonzero(gi == g_i)
        if len(ks) == 0:
            continue
        base = (base_assignments[g_i] if base_assignments
                else default_assignments(g, topology, fusion_cfg.num_levels))
        n = g.num_nodes

        def task_rows(task):
            t = tnames.index(task)
            rows = []
            for k in ks:
                w_i, j = batch._loc[k]
                w = waves[w_i]
                lo = int(w.row_off[j])
                rows.append(w.iters[-1]["actions"][t, lo:lo + n])
            return T.stack(rows)

        pl = (task_rows("placement") if "placement" in task_sizes
              else T.as_tensor(base["placement"].actions, device=dev).to(T.int32).expand(len(ks), n))
        pr = (task_rows("schedule_priority") if "schedule_priority" in task_sizes
              else T.as_tensor(base["schedule_priority"].actions, device=dev).to(T.int32))
        ix = T.as_tensor(ks, device=dev)
        if "fusion_priority" in task_sizes:
            # the native fusion pass per rollout (threads: the ctypes call releases the
            # GIL), then ONE batched DES launch per distinct grouping -- on graphs where
            # no merge succeeds (attention-stack) that is a single launch
            from concurrent.futures import ThreadPoolExecutor

            from .fusion import fuse_groups
            fus = task_rows("fusion_priority").cpu().numpy()
            a_f = task_sizes["fusion_priority"]
            for r in range(len(ks)):  # the reference's validation (simulator.py:199-210)
                ActionAssignment("fusion_priority", fus[r], a_f)
            with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as ex:
                maps = list(ex.map(lambda r: fuse_groups(g, fus[r], fusion_cfg.max_group),
                                   range(len(ks))))
            by_map: dict = {}
            for r, m in enumerate(maps):
                by_map.setdefault(m.tobytes(), []).append(r)
            for rs in by_map.values():
                fg = FusedGraph(g, maps[rs[0]])
                sel = T.as_tensor(rs, device=dev)
                res = simulate_many(fg, pl[sel].contiguous(), pr[sel] if pr.dim() == 2 else pr,
                                    topology, baseline=baselines[g_i])
                rewards[ix[sel]] = res.reward
                steps[ix[sel]] = res.step_time
                valid[ix[sel]] = res.valid
        else:
            fg = apply_fusion(g, base["fusion_priority"], fusion_cfg)
            res = simulate_many(fg, pl.contiguous(), pr, topology, baseline=baselines[g_i])
            rewards[ix] = res.reward
            steps[ix] = res.step_time
            valid[ix] = res.valid
    batch.rewards, batch.step_times, batch.valid, batch.values = rewards, steps, valid, values
    batch.shard = (lo, hi)
    if shard is not None and shard[1] > 1:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            full = gather_results(T.stack([rewards, steps, valid.to(T.float64),
                                           values.to(T.float64)]), len(gi_all), shard[1])
            batch.global_rewards, batch.global_step_times = full[0], full[1]
            batch.global_valid, batch.global_values = full[2] > 0.5, full[3]
    return batch


# ---------------------------------------------------------------------------------------
# PPO update on device


@dataclass
class _DevSample:
    handle: object
    prev: object       # int32 [T, n] node-indexed previous-iteration actions, or None
                       # (iterations == 1: the re-forward sees zero action features)
    actions: object    # int32 [T, n] node-indexed
    logp: object       # float64 [T, n] topo-row indexed
    seed: int
    temperature: float
    reward: float


def _device_samples(batch, graphs, tasks):
    """Upload (once) what each sample's re-forward and loss need."""
    T_ = torch()
    ctx = context()
    dev = T_.device("cuda", ctx.device)
    out = []
    for s in batch.samples:
        g = as_graph(graphs[s.graph_index])
        b = s.bundle
        n = g.num_nodes
        # training.py:156-158: the loss re-forwards with the bundle's prev_actions,
        # which is None when the policy ran a single iteration
        prev = (None if b.prev_actions is None else
                np.stack([np.asarray(b.prev_actions[t], np.int32) for t, _ in tasks]))
        acts = np.stack([np.asarray(b.actions[t], np.int32) for t, _ in tasks])
        logp = np.stack([np.asarray(b.log_probs[t], np.float64) for t, _ in tasks])
        if (prev is not None and prev.shape != (len(tasks), n)) or acts.shape != (len(tasks), n):
            raise ValueError("bundle arrays do not match the graph")
        out.append(_DevSample(ctx.graph(g),
                              None if prev is None else T_.as_tensor(prev, device=dev),
                              T_.as_tensor(acts, device=dev), T_.as_tensor(logp, device=dev),
                              int(b.embed_seed), float(b.temperature), float(s.reward)))
    return out


def ppo_grad(params, embed_cfg, policy_cfg, task_sizes, samples, advantages, hyper, grads,
             denominator=None):
    """One minibatch (or this rank's part of one): loss + gradient accumulated into
    `grads` (go_ppo_grad), both divided by `denominator` (default: len(samples)).
    Returns (loss, host stats array [14 * F])."""
    import ctypes as C

    from . import _lib
    from .runtime import handle_array, make_config, stream_ptr
    T_ = torch()
    tasks = ordered_tasks(task_sizes)
    F = len(samples)
    blob, offs = params
    has_prev = [s.prev is not None for s in samples]
    if any(has_prev) and not all(has_prev):
        raise ValueError("a minibatch mixes single- and multi-iteration bundles")
    prev = T_.cat([s.prev for s in samples], dim=1).contiguous() if all(has_prev) else None
    acts = T_.cat([s.actions for s in samples], dim=1).contiguous()
    logp = T_.cat([s.logp for s in samples], dim=1).contiguous()
    fparams = np.zeros((F, 4), np.float64)
    for i, s in enumerate(samples):
        fparams[i] = (advantages[i], s.temperature, s.reward, 0.0)
    harr = handle_array([s.handle for s in samples])
    seeds = (C.c_int64 * F)(*[s.seed for s in samples])
    b = _lib.GoBatch()
    b.num_forwards = F
    b.graphs = C.cast(harr, C.POINTER(C.c_void_p))
    b.embed_seeds = seeds
    b.prev_actions = _lib.ptr(prev)
    b.stage_mask = 7
    cfg_c = make_config(embed_cfg, policy_cfg, task_sizes)
    stats = np.zeros(14 * F, np.float64)
    _lib.call("go_ppo_grad", context().handle, C.byref(cfg_c), _lib.ptr(blob), offs.ctypes.data,
              C.byref(b), _lib.ptr(acts), _lib.ptr(logp), fparams.ctypes.data,
              float(hyper.clip_epsilon), float(hyper.entropy_coef), float(hyper.value_coef),
              int(denominator or F), _lib.ptr(grads), stats.ctypes.data, stream_ptr())
    Tn = len(tasks)
    per = stats[:12 * F].reshape(F, 3, 4)
    verr = stats[12 * F:13 * F]
    loss = 0.0
    for i, s in enumerate(samples):
        n = s.handle.n
        pol = sum(per[i, t, 0] / n for t in range(Tn)) / Tn
        ent = sum(per[i, t, 1] / n for t in range(Tn)) / Tn
        loss += -(pol + hyper.entropy_coef * ent) + hyper.value_coef * verr[i]
    return loss / float(denominator or F), stats


def rank_share(chunk, rank: int, world: int):
    """Samples of a minibatch this rank evaluates (owner-computes)."""
    return chunk[rank::world]


def _dist_rank_world():
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_rank(), dist.get_world_size()
    except Exception:
        pass
    return 0, 1


def allreduce_sum(grads, loss: float) -> float:
    """NCCL all-reduce(sum) of the gradient blob and the scalar loss; every rank then
    runs the identical fused Adam step, so parameters stay replicated."""
    import torch.distributed as dist
    T_ = torch()
    lt = T_.tensor([loss], dtype=T_.float64, device=grads.device)
    dist.all_reduce(grads)
    dist.all_reduce(lt)
    return float(lt.item())


def ppo_update(batch, store, graphs, topology, task_sizes, hyper, embed_cfg, policy_cfg,
               seed: int = 0) -> dict:
    """training.py:196-233 on device: epochs of shuffled minibatches, one fused
    forward+backward per minibatch (all its samples in one ragged batch), fused
    Adam.  Mutates `store` (parameters, Adam moments, step_count) like the reference."""
    from . import _lib
    from .params import pack, slot_names
    from .runtime import stream_ptr
    if not batch.samples:
        raise ValueError("empty rollout batch")
    T_ = torch()
    dev = T_.device("cuda", context().device)
    tasks = ordered_tasks(task_sizes)
    rng = np.random.default_rng(seed)
    adv = np.array([s.advantage for s in batch.samples], dtype=np.float64)
    if hyper.advantage_norm and len(adv) > 1 and adv.std() > 0:
        adv = (adv - adv.mean()) / (adv.std() + 1e-8)
    # float64 master parameters and Adam moments stay on the device for the whole
    # update (go_adam64 runs the reference's float64 Adam); the kernels read `blob`,
    # the float32 copy go_adam64 refreshes after every step
    blob64_h, offs = pack(store, embed_cfg, policy_cfg, task_sizes, dtype=np.float64)
    names = slot_names(embed_cfg, policy_cfg, task_sizes)
    blob64 = T_.as_tensor(blob64_h, device=dev).contiguous()
    blob = blob64.to(T_.float32)

    def moments(d):
        out = np.zeros_like(blob64_h)
        for nm, o in zip(names, offs):
            if d is not None and nm in d:
                a = np.asarray(d[nm], np.float64).reshape(-1)
                out[o:o + a.size] = a
        return T_.as_tensor(out, device=dev)

    m = moments(getattr(store, "_m", None))
    v = moments(getattr(store, "_v", None))
    grads = T_.zeros_like(blob)
    rank, world = _dist_rank_world()
    samples = _device_samples(batch, graphs, tasks)
    step = int(getattr(store, "step_count", 0))
    stats = {"ratio_sum": 0.0, "clip_sum": 0.0, "node_count": 0, "entropy_sum": 0.0,
             "entropy_count": 0, "value_loss_sum": 0.0, "value_count": 0}
    for _epoch in range(hyper.epochs):
        perm = rng.permutation(len(samples))
        stats = {k: 0 if isinstance(val, int) else 0.0 for k, val in stats.items()}
        for chunk in np.array_split(perm, min(hyper.minibatches, len(perm))):
            if len(chunk) == 0:
                continue
            grads.zero_()
            mine = rank_share(chunk, rank, world)
            loss, st = (ppo_grad((blob, offs), embed_cfg, policy_cfg, task_sizes,
                                 [samples[i] for i in mine], adv[mine], hyper, grads,
                                 denominator=len(chunk))
                        if len(mine) else (0.0, np.zeros(0)))
            if world > 1:
                # the one collective of the update: sum gradients (and the loss) over ranks
                loss = allreduce_sum(grads, loss)
            if not np.isfinite(loss):
                raise RuntimeError(
                    f"non-finite PPO loss (advantages {adv.min():.3g}..{adv.max():.3g})")
            F = len(mine)
            per = st[:12 * F].reshape(F, 3, 4)
            for i, k in enumerate(mine):
                n = samples[k].handle.n
                for t in range(len(tasks)):
                    stats["ratio_sum"] += float(per[i, t, 2])
                    stats["clip_sum"] += float(per[i, t, 3])
                    stats["node_count"] += n
                    stats["entropy_sum"] += float(per[i, t, 1] / max(1, n))
                    stats["entropy_count"] += 1
                stats["value_loss_sum"] += float(st[12 * F + i])
                stats["value_count"] += 1
            step += 1
            _lib.call("go_adam64", context().handle, _lib.ptr(blob64), _lib.ptr(blob),
                      _lib.ptr(grads), _lib.ptr(m), _lib.ptr(v), int(blob.numel()), step,
                      float(hyper.lr), 0.9, 0.999, 1e-8, stream_ptr())
    if world > 1:
        import torch.distributed as dist
        T_ = torch()
        keys = list(stats)
        vec = T_.tensor([float(stats[k]) for k in keys], dtype=T_.float64, device=dev)
        dist.all_reduce(vec)
        stats = {k: (int(round(v)) if isinstance(stats[k], int) else float(v))
                 for k, v in zip(keys, vec.tolist())}
    # write the float64 parameters and Adam state back into the store
    hb, hm, hv = (x.cpu().numpy() for x in (blob64, m, v))
    for nm, o in zip(names, offs):
        if nm not in store:
            continue
        p = store[nm]
        size = np.asarray(p.data).size
        shape = np.asarray(p.data).shape
        p.data = hb[o:o + size].reshape(shape).copy()
        if hasattr(store, "_m"):
            store._m[nm] = hm[o:o + size].reshape(shape).copy()
            store._v[nm] = hv[o:o + size].reshape(shape).copy()
    if hasattr(store, "step_count"):
        store.step_count = step
    if hasattr(store, "touch"):
        store.touch()
    return {
        "mean_ratio": stats["ratio_sum"] / max(1, stats["node_count"]),
        "clip_fraction": stats["clip_sum"] / max(1, stats["node_count"]),
        "entropy": stats["entropy_sum"] / max(1, stats["entropy_count"]),
        "value_loss": stats["value_loss_sum"] / max(1, stats["value_count"]),
    }


# ---------------------------------------------------------------------------------------
# training drivers (host orchestration over the device entry points above; SURVEY §8(f) F4:
# what `graphopt optimize method=rl` runs, cli.py:208-220)

@dataclass
class TrainResult:
    """training.py:236-248."""
    store: object
    best_store: object
    curve: list
    best_step_times: list
    best_actions: list
    baselines: list
    stats_history: list = field(default_factory=list)

    @property
    def best_step_time(self) -> float:
        return self.best_step_times[0]


def train(graphs, topology, tasks, hyper, steps: int, seed: int, embed_cfg=None,
          policy_cfg=None, fusion_cfg=None, store=None, incumbent_from_default: bool = True,
          base_assignments=None) -> TrainResult:
    """training.py:251-317, same control flow and the same numpy stream for the per-step
    rollout and update seeds; each step is one device `collect_rollouts` (all rollouts
    batched, one DES launch per graph) and one device `ppo_update`.  The incumbent /
    best-store / divergence bookkeeping reads only per-rollout scalars, so the per-sample
    action arrays are fetched from the device only for a new incumbent.
    Single-process semantics: under torch.distributed every rank runs the same loop and
    ppo_update shares the minibatch work (owner-computes + gradient all-reduce)."""
    from .baselines import baseline_step_time
    from .params import init_all_params
    from .simulator import evaluate_assignments
    embed_cfg = embed_cfg or EmbedConfig()
    policy_cfg = policy_cfg or PolicyConfig()
    fusion_cfg = fusion_cfg or FusionConfig()
    graphs = [as_graph(g) for g in graphs]
    task_sizes = task_action_sizes(topology, tasks, fusion_cfg.num_levels)
    if store is None:
        store = init_all_params(embed_cfg, policy_cfg, task_sizes, seed)
    baselines = [baseline_step_time(g, topology, fusion_cfg) for g in graphs]
    start_results = [
        evaluate_assignments(g, topology,
                             base_assignments[i] if base_assignments
                             else default_assignments(g, topology, fusion_cfg.num_levels),
                             fusion_cfg)
        for i, g in enumerate(graphs)]
    valid_exists = any(r.valid for r in start_results)
    best_times = [r.step_time if (incumbent_from_default and r.valid) else math.inf
                  for r in start_results]
    best_actions = [None] * len(graphs)
    best_store = store.clone()
    best_mean_reward = -math.inf
    curve, stats_history = [], []
    rng = np.random.default_rng(seed)
    bad_streak = 0
    for step in range(steps):
        batch = collect_rollouts(store, graphs, topology, task_sizes, baselines,
                                 hyper.rollouts, int(rng.integers(2**31)), hyper,
                                 embed_cfg, policy_cfg, fusion_cfg, base_assignments,
                                 keep_logits=False)
        for s in batch.samples:
            if s.valid and s.step_time < best_times[s.graph_index]:
                best_times[s.graph_index] = s.step_time
                best_actions[s.graph_index] = {k: np.array(v, copy=True)
                                               for k, v in s.bundle.actions.items()}
        if batch.mean_reward > best_mean_reward:
            best_mean_reward = batch.mean_reward
            best_store = store.clone()
        if batch.mean_reward < -9 and valid_exists:
            bad_streak += 1
            if bad_streak >= 50:
                raise RuntimeError(
                    f"training diverged: mean reward {batch.mean_reward:.2f} "
                    f"below -9 for 50 consecutive steps")
        else:
            bad_streak = 0
        stats = ppo_update(batch, store, graphs, topology, task_sizes, hyper,
                           embed_cfg, policy_cfg, int(rng.integers(2**31)))
        stats_history.append(stats)
        finite = [t for t in best_times if math.isfinite(t)]
        curve.append((step, float(np.mean(finite)) if finite else math.inf))
    return TrainResult(store=store, best_store=best_store, curve=curve,
                       best_step_times=best_times, best_actions=best_actions,
                       baselines=baselines, stats_history=stats_history)


def decode_step_time(graph, store, topology, tasks, embed_cfg, policy_cfg, fusion_cfg) -> float:
    """training.py:320-332: greedy (temperature-0) decode, scored by the simulator;
    invalid decodes count as +inf."""
    from .policy import iterate_decisions
    from .simulator import evaluate_assignments
    task_sizes = task_action_sizes(topology, tasks, fusion_cfg.num_levels)
    bundle, _ = iterate_decisions(graph, store, embed_cfg, policy_cfg, task_sizes,
                                  policy_cfg.iterations, seed=0, temperature=0.0)
    asg = bundle_assignments(graph, topology, bundle, task_sizes, fusion_cfg)
    res = evaluate_assignments(graph, topology, asg, fusion_cfg)
    return res.step_time if res.valid else math.inf


def pretrain_finetune_zeroshot(train_graphs: dict, holdout_family: str, holdout_graph, topology,
                               tasks, hyper, seed: int, pretrain_batches: int = 5,
                               steps_per_batch: int = 4, batch_size: int = 4,
                               finetune_steps: int = 20, embed_cfg=None, policy_cfg=None,
                               fusion_cfg=None) -> dict:
    """training.py:335-381: pretrain on the training families, then the holdout graph's
    zero-shot decode, the best within `finetune_steps` of fine-tuning (never worse than
    zero-shot) and a from-scratch run of the same budget."""
    from .params import init_all_params
    if finetune_steps > 50:
        raise ValueError("fine-tuning budget is capped at 50 steps")
    if holdout_family in train_graphs:
        raise ValueError(f"holdout family {holdout_family!r} appears in the training set")
    hname = getattr(holdout_graph, "name", None)
    for family, gs in train_graphs.items():
        for g in gs:
            if getattr(g, "name", None) == hname:
                raise ValueError(f"holdout graph {hname!r} appears in the training set")
    embed_cfg = embed_cfg or EmbedConfig()
    policy_cfg = policy_cfg or PolicyConfig()
    fusion_cfg = fusion_cfg or FusionConfig()
    task_sizes = task_action_sizes(topology, tasks, fusion_cfg.num_levels)
    pool = [g for family in sorted(train_graphs) for g in train_graphs[family]]
    rng = np.random.default_rng(seed)
    store = init_all_params(embed_cfg, policy_cfg, task_sizes, seed)
    for _ in range(pretrain_batches):
        take = min(batch_size, len(pool))
        idx = rng.choice(len(pool), size=take, replace=False)
        result = train([pool[i] for i in idx], topology, tasks, hyper, steps_per_batch,
                       int(rng.integers(2**31)), embed_cfg, policy_cfg, fusion_cfg, store=store)
        store = result.store
    zeroshot = decode_step_time(holdout_graph, store, topology, tasks, embed_cfg, policy_cfg,
                                fusion_cfg)
    finetuned = zeroshot
    if finetune_steps > 0:
        ft = train([holdout_graph], topology, tasks, hyper, finetune_steps,
                   int(rng.integers(2**31)), embed_cfg, policy_cfg, fusion_cfg,
                   store=store.clone(), incumbent_from_default=False)
        finetuned = min(finetuned, ft.best_step_time)
    scratch = math.inf
    if finetune_steps > 0:
        sc = train([holdout_graph], topology, tasks, hyper, finetune_steps,
                   int(rng.integers(2**31)), embed_cfg, policy_cfg, fusion_cfg,
                   incumbent_from_default=False)
        scratch = sc.best_step_time
    return {"zeroshot": zeroshot, "finetuned": finetuned, "scratch": scratch}

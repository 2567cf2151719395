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
           "ppo_update", "train_step"]


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
    host = _host_staged(pad)
    src = pad.cpu() if host else pad
    bufs = [T.empty_like(src) for _ in sizes]
    dist.all_gather(bufs, src)
    return T.cat([b[:, :s] for b, s in zip(bufs, sizes)], dim=1).to(packed.device)


def _host_staged(t) -> bool:
    """gloo (the CPU test backend) takes host tensors; NCCL works on device memory."""
    import torch.distributed as dist
    return t.is_cuda and dist.get_backend() != "nccl"


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
    batch.global_count = len(gi_all)
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
    if _host_staged(grads):
        g = grads.cpu()
        dist.all_reduce(g)
        grads.copy_(g)
        lt = lt.cpu()
    else:
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
    rank, world = _dist_rank_world()
    lo, hi = getattr(batch, "shard", None) or (0, len(batch.samples))
    count = getattr(batch, "global_count", hi - lo)
    sharded = hi - lo < count
    if sharded:
        # a collect_rollouts(shard=...) batch: this rank holds global rollouts [lo, hi).
        # The reference's advantage normalisation and epoch permutation run over ALL
        # rollouts (training.py:204-213), so both use the all-gathered results; each
        # minibatch member is evaluated by the rank that collected it.
        if getattr(batch, "global_rewards", None) is None or world <= 1:
            raise ValueError("ppo_update got a sharded rollout batch without its gathered "
                             "global results: call collect_rollouts(shard=(rank, world)) "
                             "with torch.distributed initialised")
        adv = (batch.global_rewards - batch.global_values).cpu().numpy().astype(np.float64)
    else:
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
    samples = _device_samples(batch, graphs, tasks)
    step = int(getattr(store, "step_count", 0))
    stats = {"ratio_sum": 0.0, "clip_sum": 0.0, "node_count": 0, "entropy_sum": 0.0,
             "entropy_count": 0, "value_loss_sum": 0.0, "value_count": 0}
    for _epoch in range(hyper.epochs):
        perm = rng.permutation(count)
        stats = {k: 0 if isinstance(val, int) else 0.0 for k, val in stats.items()}
        for chunk in np.array_split(perm, min(hyper.minibatches, len(perm))):
            if len(chunk) == 0:
                continue
            grads.zero_()
            if sharded:  # owner computes: the members this rank collected
                mine = [int(k) for k in chunk if lo <= k < hi]
            else:        # replicated batch: split the members round-robin
                mine = [int(k) for k in rank_share(chunk, rank, world)]
            loss, st = (ppo_grad((blob, offs), embed_cfg, policy_cfg, task_sizes,
                                 [samples[k - lo] for k in mine], adv[mine], hyper, grads,
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
                n = samples[k - lo].handle.n
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
        vec = T_.tensor([float(stats[k]) for k in keys], dtype=T_.float64,
                        device="cpu" if dist.get_backend() != "nccl" else dev)
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
# one training step on the device (the body of the reference's train loop,
# training.py:289-314: collect_rollouts then ppo_update).  The loop around it -- the
# incumbent / best-store / divergence bookkeeping and the pretrain / fine-tune
# drivers (training.py:236-384) -- is host orchestration that stays in the reference
# and reaches this path through the INTEGRATION.md shim (out of scope).

def train_step(store, graphs, topology, task_sizes, baselines, hyper, embed_cfg, policy_cfg,
               fusion_cfg, rollout_seed: int, update_seed: int, base_assignments=None,
               shard=None, keep_logits: bool = False):
    """collect_rollouts + ppo_update with the rollouts sharded over the ranks of an
    initialised torch.distributed group: each rank decides and
    scores only its own global rollouts, the per-rollout results are all-gathered
    once, and each minibatch member's forward+backward runs on the rank that
    collected it, followed by one gradient all-reduce per minibatch.  Returns
    (batch, stats); `store` is updated in place on every rank, identically."""
    if shard is None:
        rank, world = _dist_rank_world()
        shard = (rank, world) if world > 1 else None
    batch = collect_rollouts(store, graphs, topology, task_sizes, baselines, hyper.rollouts,
                             rollout_seed, hyper, embed_cfg, policy_cfg, fusion_cfg,
                             base_assignments, keep_logits=keep_logits, shard=shard)
    stats = ppo_update(batch, store, graphs, topology, task_sizes, hyper, embed_cfg,
                       policy_cfg, update_seed)
    return batch, stats

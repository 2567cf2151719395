"""Default pipeline, reward normaliser and the non-learned optimizers (mirrors
baselines.py:24-237).

greedy_placement uses the native O(D N log N) DP (go_greedy_cuts) that returns the
reference's exact cuts; baseline_step_time, brute_force and simulated_annealing score
candidates with the device DES (brute force batched, 65,536 placements per launch;
annealing chains run on the device, many at once: anneal_chains)."""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import NUM_PRIORITY_LEVELS, FusionConfig
from .costmodel import as_topology
from .fusion import greedy_cuts
from .graph import as_graph
from .simulator import ActionAssignment, evaluate_assignments

_cache: dict = {}


def greedy_placement(graph, topology) -> ActionAssignment:
    """baselines.py:75-118: contiguous topo chunks balanced by flops, colocation
    groups forced to their first member's device."""
    g = as_graph(graph)
    d = as_topology(topology).num_devices
    order = g.topo_order()
    cuts = greedy_cuts(g.flops[order], d)
    actions = np.zeros(g.num_nodes, dtype=np.int64)
    for dev in range(d):
        actions[order[cuts[dev]:cuts[dev + 1]]] = dev
    first: dict = {}
    for v in np.flatnonzero(g.coloc >= 0):
        c = int(g.coloc[v])
        if c not in first:
            first[c] = int(actions[v])
        actions[v] = first[c]
    return ActionAssignment("placement", actions, d)


def default_assignments(graph, topology, num_levels: int = NUM_PRIORITY_LEVELS) -> dict:
    """baselines.py:24-36 (cached per (graph, topology) object)."""
    g = as_graph(graph)
    key = (id(g), id(topology), num_levels)
    hit = _cache.get(key)
    if hit is not None and hit[0] is g:
        return {k: ActionAssignment(v.task, v.actions.copy(), v.num_actions)
                for k, v in hit[1].items()}
    n = g.num_nodes
    asg = {
        "placement": greedy_placement(g, topology),
        "schedule_priority": ActionAssignment.constant("schedule_priority", n, num_levels, 0),
        "fusion_priority": ActionAssignment.constant("fusion_priority", n, num_levels, 0),
    }
    _cache[key] = (g, asg)
    return {k: ActionAssignment(v.task, v.actions.copy(), v.num_actions) for k, v in asg.items()}


def baseline_step_time(graph, topology, fusion_config: FusionConfig | None = None) -> float:
    """baselines.py:39-47."""
    res = evaluate_assignments(graph, topology, default_assignments(graph, topology),
                               fusion_config)
    return res.step_time


# ---------------------------------------------------------------------------------------
# Non-learned optimizers on the batched device DES (baselines.py:50-237)

def descendant_counts(graph) -> np.ndarray:
    """baselines.py:50-58: nodes reachable from each node (excluding itself).  Same
    reverse-topological OR of successor reach sets, with Python ints as bitsets (n bits
    per node instead of the reference's n x n bool matrix)."""
    g = as_graph(graph)
    n = g.num_nodes
    succ = [[] for _ in range(n)]
    for s, d in zip(g.src.tolist(), g.dst.tolist()):
        succ[s].append(d)
    reach = [0] * n
    for v in reversed(g.topo_order().tolist()):
        r = 0
        for w in succ[v]:
            r |= reach[w] | (1 << w)
        reach[v] = r
    return np.array([r.bit_count() for r in reach], dtype=np.int64)


def fanout_priorities(graph, num_levels: int = NUM_PRIORITY_LEVELS) -> ActionAssignment:
    """baselines.py:61-72: schedule priority proportional to descendant count."""
    g = as_graph(graph)
    counts = descendant_counts(g)
    top = int(counts.max(initial=0))
    if top == 0:
        levels = np.zeros(g.num_nodes, dtype=np.int64)
    else:
        levels = (counts * (num_levels - 1)) // top
    return ActionAssignment("schedule_priority", levels.astype(np.int64), num_levels)


def _task_action_size(task: str, topology, num_levels: int) -> int:
    """baselines.py:142-143."""
    return as_topology(topology).num_devices if task == "placement" else num_levels


def brute_force(graph, topology, task: str, limit: int = 10**6,
                fusion_config: FusionConfig | None = None, batch: int = 1 << 16):
    """baselines.py:209-237: exhaustive search over one task's a^n action vectors (other
    tasks at the defaults), returning the lexicographically smallest argmin.  The
    combinations are generated on the device in itertools.product order and scored by
    the batched DES (`batch` placements per launch) instead of one simulate() each; a
    fusion-priority search runs the native fusion pass per combination."""
    import torch as T

    from .config import TASKS
    from .simulator import apply_fusion, evaluate_assignments, simulate_many
    if task not in TASKS:
        raise ValueError(f"unknown task {task!r}")
    fusion_config = fusion_config or FusionConfig()
    g = as_graph(graph)
    top = as_topology(topology)
    n = g.num_nodes
    a = _task_action_size(task, top, fusion_config.num_levels)
    if a ** n > limit:
        raise ValueError(f"search space {a}^{n} exceeds limit {limit}")
    base = default_assignments(g, top, fusion_config.num_levels)
    total = a ** n
    best_i, best_time = -1, float("inf")
    if task == "fusion_priority":
        for i in range(total):
            combo = np.array([(i // a ** (n - 1 - j)) % a for j in range(n)], dtype=np.int64)
            asg = dict(base)
            asg[task] = ActionAssignment(task, combo, a)
            res = evaluate_assignments(g, top, asg, fusion_config)
            if res.valid and res.step_time < best_time:
                best_i, best_time = i, res.step_time
    else:
        from .runtime import context
        dev = T.device("cuda", context().device)
        fg = apply_fusion(g, base["fusion_priority"], fusion_config)
        place0 = T.as_tensor(base["placement"].actions, device=dev, dtype=T.int64)
        prio0 = T.as_tensor(base["schedule_priority"].actions, device=dev, dtype=T.int64)
        pw = T.tensor([a ** (n - 1 - j) for j in range(n)], device=dev, dtype=T.int64)
        for i0 in range(0, total, batch):
            idx = T.arange(i0, min(total, i0 + batch), device=dev, dtype=T.int64)
            combos = (idx[:, None] // pw[None, :]) % a  # itertools.product order
            if task == "placement":
                res = simulate_many(fg, combos, prio0, top)
            else:
                res = simulate_many(fg, place0.expand(len(idx), n), combos, top)
            t = T.where(res.valid.bool(), res.step_time,
                        T.full_like(res.step_time, float("inf")))
            m = float(t.min())
            if m < best_time:  # strict: an earlier batch keeps its tie
                best_time = m
                best_i = i0 + int(T.nonzero(t == m)[0, 0])
    if best_i < 0:
        raise RuntimeError("no valid assignment found")
    best = np.array([(best_i // a ** (n - 1 - j)) % a for j in range(n)], dtype=np.int64)
    return ActionAssignment(task, best, a), best_time


@dataclass
class SAConfig:
    """baselines.py:121-137."""
    iterations: int = 5000
    initial_temperature: float | None = None  # None: 10% of the initial step time
    cooling_rate: float = 0.999
    moves_per_step: int = 1
    seed: int = 0

    def __post_init__(self):
        if self.iterations < 1:
            raise ValueError("iterations must be >= 1")
        if not (0.0 < self.cooling_rate < 1.0):
            raise ValueError("cooling_rate must be in (0,1) for a decreasing schedule")
        if self.moves_per_step < 1:
            raise ValueError("moves_per_step must be >= 1")


def simulated_annealing(graph, topology, tasks: list, sa: SAConfig | None = None,
                        fusion_config: FusionConfig | None = None):
    """baselines.py:146-206 -> (assignments, best step time): the reference's chain for
    seed sa.seed, run by anneal_chains."""
    sa = sa or SAConfig()
    return anneal_chains(graph, topology, tasks, sa, fusion_config, seeds=[sa.seed])[0]


def anneal_chains(graph, topology, tasks: list, sa: SAConfig | None = None,
                  fusion_config: FusionConfig | None = None, seeds=None) -> list:
    """Many simulated-annealing chains at once: chain k is the
    reference's simulated_annealing (baselines.py:146-206) with SAConfig.seed =
    seeds[k], bit for bit -- same moves, same acceptance, same best state -- and the
    chains run concurrently.  Returns [(assignments, best step time)] per seed.

    Placement and schedule-priority chains run entirely on the device (go_anneal: one
    chain per 32-thread block, candidate simulations by the device DES, the numpy
    stream regenerated on the device).  Chains that anneal fusion priorities re-run the
    native fusion pass per candidate on the host and score each iteration's candidates
    of all chains with batched device simulations."""
    from .config import TASKS
    if not tasks:
        raise ValueError("tasks must be non-empty")
    for t in tasks:
        if t not in TASKS:
            raise ValueError(f"unknown task {t!r}")
    sa = sa or SAConfig()
    fusion_config = fusion_config or FusionConfig()
    seeds = [sa.seed] if seeds is None else [int(x) for x in seeds]
    g = as_graph(graph)
    top = as_topology(topology)
    start = default_assignments(g, top, fusion_config.num_levels)
    sizes = {t: _task_action_size(t, top, fusion_config.num_levels) for t in tasks}
    if "fusion_priority" in tasks:
        bests = _anneal_host_fusion(g, top, tasks, sa, fusion_config, seeds, start, sizes)
    else:
        bests = _anneal_device(g, top, tasks, sa, fusion_config, seeds, start, sizes)
    out = []
    for best, t in bests:
        res = dict(start)
        for task in tasks:
            res[task] = ActionAssignment(task, best[task], sizes[task])
        out.append((res, t))
    return out


def _anneal_device(g, top, tasks, sa, fusion_config, seeds, start, sizes):
    import ctypes as C
    import math

    from . import _lib
    from .engine import pcg_words
    from .runtime import context, stream_ptr, torch
    from .simulator import apply_fusion
    T = torch()
    dev = T.device("cuda", context().device)
    h = apply_fusion(g, start["fusion_priority"], fusion_config).install()
    n, k = g.num_nodes, len(seeds)
    init = np.stack([start["placement"].actions, start["schedule_priority"].actions]).astype(np.int32)
    state = T.as_tensor(np.broadcast_to(init, (k, 2, n)).copy(), device=dev)
    best = state.clone()
    best_time = T.empty(k, dtype=T.float64, device=dev)
    words = np.array([pcg_words(np.random.default_rng(s)) for s in seeds], dtype=np.uint64)
    slot = {"placement": 0, "schedule_priority": 1}
    slots = (C.c_int32 * 2)(*[slot[t] for t in tasks])
    sz = (C.c_int32 * 2)(*[sizes[t] for t in tasks])
    t0 = math.nan if sa.initial_temperature is None else float(sa.initial_temperature)
    _lib.call("go_anneal", context().handle, h.handle, k, words.ctypes.data, _lib.ptr(state),
              _lib.ptr(best), top.num_devices, _lib.ptr(top.peak), _lib.ptr(top.mem_bw),
              _lib.ptr(top.cap), _lib.ptr(top.link_bw), 0, int(sa.iterations),
              int(sa.moves_per_step), t0, float(sa.cooling_rate), len(tasks), slots, sz,
              _lib.ptr(best_time), stream_ptr())
    bh = best.cpu().numpy().astype(np.int64)
    th = best_time.cpu().numpy()
    return [({t: bh[i, slot[t]].copy() for t in tasks}, float(th[i])) for i in range(k)]


def _anneal_host_fusion(g, top, tasks, sa, fusion_config, seeds, start, sizes):
    """Iteration-synchronous chains: every chain proposes from its own numpy stream, the
    candidates' fusion passes run natively on host threads and their simulations are
    batched on the device per distinct grouping, then every chain applies its
    Metropolis test (baselines.py:183-204)."""
    import math
    from concurrent.futures import ThreadPoolExecutor

    from .fusion import fuse_groups
    from .simulator import FusedGraph, simulate_many
    n, k = g.num_nodes, len(seeds)
    rngs = [np.random.default_rng(s) for s in seeds]
    base = {t: start[t].actions for t in ("placement", "schedule_priority", "fusion_priority")}
    cur = [{t: base[t].copy() for t in tasks} for _ in range(k)]

    def score(states):
        full = [{**base, **st} for st in states]
        with ThreadPoolExecutor(max_workers=8) as ex:
            maps = list(ex.map(lambda a: fuse_groups(g, a["fusion_priority"],
                                                     fusion_config.max_group), full))
        times = np.empty(len(full))
        groups: dict = {}
        for i, m in enumerate(maps):
            groups.setdefault(m.tobytes(), []).append(i)
        for ids in groups.values():
            res = simulate_many(FusedGraph(g, maps[ids[0]]),
                                np.stack([full[i]["placement"] for i in ids]),
                                np.stack([full[i]["schedule_priority"] for i in ids]), top)
            st, va = res.step_time.cpu().numpy(), res.valid.cpu().numpy()
            for j, i in enumerate(ids):
                times[i] = st[j] if va[j] else math.inf
        return times

    cur_t = score(cur)
    best = [{t: c[t].copy() for t in tasks} for c in cur]
    best_t = cur_t.copy()
    temp = [sa.initial_temperature if sa.initial_temperature is not None
            else (0.1 * x if math.isfinite(x) else 1.0) for x in cur_t]
    for _ in range(sa.iterations):
        cand = []
        for i in range(k):
            c = {t: cur[i][t].copy() for t in tasks}
            for _m in range(sa.moves_per_step):
                t = tasks[int(rngs[i].integers(len(tasks)))]
                v = int(rngs[i].integers(n))
                c[t][v] = int(rngs[i].integers(sizes[t]))
            cand.append(c)
        cand_t = score(cand)
        for i in range(k):
            delta = cand_t[i] - cur_t[i]
            ok = delta <= 0
            if not ok and temp[i] > 0 and math.isfinite(delta):
                ok = rngs[i].random() < math.exp(-delta / temp[i])
            if ok:
                cur[i], cur_t[i] = cand[i], cand_t[i]
                if cur_t[i] < best_t[i]:
                    best_t[i] = cur_t[i]
                    best[i] = {t: cur[i][t].copy() for t in tasks}
            temp[i] *= sa.cooling_rate
    return [(best[i], float(best_t[i])) for i in range(k)]

"""Default pipeline, reward normaliser and the non-learned optimizers (mirrors
baselines.py:24-237).

greedy_placement uses the native O(D N log N) DP (go_greedy_cuts) that returns the
reference's exact cuts; baseline_step_time, brute_force and simulated_annealing score
candidates with the device DES (brute force batched, 65,536 placements per launch)."""
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
    """baselines.py:146-206: anneal over the concatenated action vectors of `tasks`,
    one uniform single-node move per step, Metropolis acceptance under geometric
    cooling, best state returned.  The chain is sequential and its random stream
    (np.random.default_rng(seed): task index, node, value, then a uniform only for an
    uphill move) is the reference's draw for draw; each candidate is scored by the
    device DES (bit-exact step times, so the chain takes the same path), the fusion pass
    re-run only when fusion priorities are annealed."""
    import math

    from .config import TASKS
    from .simulator import apply_fusion, simulate
    if not tasks:
        raise ValueError("tasks must be non-empty")
    for t in tasks:
        if t not in TASKS:
            raise ValueError(f"unknown task {t!r}")
    sa = sa or SAConfig()
    fusion_config = fusion_config or FusionConfig()
    g = as_graph(graph)
    top = as_topology(topology)
    rng = np.random.default_rng(sa.seed)
    n = g.num_nodes
    state = default_assignments(g, top, fusion_config.num_levels)
    sizes = {t: _task_action_size(t, top, fusion_config.num_levels) for t in tasks}
    fixed_fg = None if "fusion_priority" in tasks else apply_fusion(g, state["fusion_priority"],
                                                                   fusion_config)

    def evaluate(asg) -> float:
        fg = fixed_fg or apply_fusion(g, asg["fusion_priority"], fusion_config)
        res = simulate(fg, asg["placement"], asg["schedule_priority"], top)
        return res.step_time if res.valid else math.inf

    current = {t: state[t].actions.copy() for t in tasks}
    cur_time = evaluate(state)
    best = {t: current[t].copy() for t in tasks}
    best_time = cur_time
    temp = sa.initial_temperature
    if temp is None:
        temp = 0.1 * cur_time if math.isfinite(cur_time) else 1.0
    for _ in range(sa.iterations):
        cand = {t: current[t].copy() for t in tasks}
        for _ in range(sa.moves_per_step):
            t = tasks[int(rng.integers(len(tasks)))]
            v = int(rng.integers(n))
            cand[t][v] = int(rng.integers(sizes[t]))
        asg = dict(state)
        for t in tasks:
            asg[t] = ActionAssignment(t, cand[t], sizes[t])
        cand_time = evaluate(asg)
        delta = cand_time - cur_time
        accept = delta <= 0
        if not accept and temp > 0 and math.isfinite(delta):
            accept = rng.random() < math.exp(-delta / temp)
        if accept:
            current = cand
            cur_time = cand_time
            if cur_time < best_time:
                best_time = cur_time
                best = {t: current[t].copy() for t in tasks}
        temp *= sa.cooling_rate
    result = dict(state)
    for t in tasks:
        result[t] = ActionAssignment(t, best[t], sizes[t])
    return result, best_time

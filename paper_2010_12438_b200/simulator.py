"""Runtime simulator on the B200 (mirrors graphopt.simulator, simulator.py:1-496).

simulate / evaluate_assignments keep the reference signatures and return a
SimResult; the discrete-event simulation runs on device (csrc/des.cu, one thread
per placement, bit-exact float64).  simulate_many() is the batched twin that
scores K placements of one graph in one launch.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import NUM_PRIORITY_LEVELS, TASKS, FusionConfig
from .costmodel import as_topology
from .engine import VIOLATIONS, simulate_batch
from .graph import OP_INDEX, as_graph
from .runtime import context, torch

__all__ = ["TASKS", "NUM_PRIORITY_LEVELS", "NON_FUSIBLE", "ActionAssignment", "SimResult",
           "TraceEvent",
           "FusionConfig", "FusedGraph", "singleton_fused", "apply_fusion", "simulate",
           "simulate_many", "evaluate_assignments", "check_validity"]

NON_FUSIBLE = frozenset({"matmul", "conv", "embed-lookup", "other"})  # simulator.py:28


@dataclass
class ActionAssignment:
    """simulator.py:31-58."""

    task: str
    actions: np.ndarray
    num_actions: int

    def __post_init__(self):
        if self.task not in TASKS:
            raise ValueError(f"unknown task {self.task!r}")
        self.actions = np.asarray(self.actions, dtype=np.int64)
        if self.actions.ndim != 1:
            raise ValueError("actions must be a 1-D vector")
        if self.num_actions <= 0:
            raise ValueError("action space must be non-empty")

    @classmethod
    def constant(cls, task, num_nodes, num_actions, value=0):
        return cls(task, np.full(num_nodes, value, dtype=np.int64), num_actions)

    def __len__(self):
        return len(self.actions)


@dataclass
class TraceEvent:
    """simulator.py:61-67."""
    time_start: float
    time_end: float
    device: str
    kind: str  # "compute" | "transfer"
    group_id: int


@dataclass
class SimResult:
    step_time: float
    valid: bool
    violation: str | None
    per_device_busy: list
    peak_mem: list
    trace: list | None = None


class FusedGraph:
    """A graph plus a grouping (simulator.py:86-172).  The group tables themselves
    (canonical order, costs, resident bytes, topo index) are built natively when the
    grouping is installed on the device graph (go_graph_set_fusion)."""

    def __init__(self, graph, group_map):
        self.graph = as_graph(graph)
        gm = np.asarray(group_map, dtype=np.int64)
        if gm.shape != (self.graph.num_nodes,):
            raise ValueError("group_map must assign every node to a group")
        # canonical ids: groups ordered by lowest member (simulator.py:98-109)
        _, first = np.unique(gm, return_index=True)
        roots = gm[np.sort(first)]
        remap = {int(r): i for i, r in enumerate(roots)}
        self.group_map = np.array([remap[int(x)] for x in gm], dtype=np.int64)
        self._singleton = bool((self.group_map == np.arange(len(gm))).all())

    @property
    def num_groups(self) -> int:
        return int(self.group_map.max(initial=-1)) + 1

    def install(self):
        """Upload this grouping's DES tables; returns the device graph handle."""
        h = context().graph(self.graph)
        h.set_fusion(None if self._singleton else self.group_map)
        return h

    @property
    def topo_index(self):
        return None if not self.install().acyclic else True


def as_fused(fg) -> FusedGraph:
    """This package's FusedGraph, or the reference's (duck-typed: .graph, .group_map)
    re-expressed as one, so a graphopt.simulator.FusedGraph passes straight through."""
    if isinstance(fg, FusedGraph):
        return fg
    return FusedGraph(fg.graph, fg.group_map)


def singleton_fused(graph) -> FusedGraph:
    g = as_graph(graph)
    return FusedGraph(g, np.arange(g.num_nodes))


def apply_fusion(graph, fusion: ActionAssignment, config: FusionConfig | None = None) -> FusedGraph:
    """simulator.py:199-277 greedy fusion pass (native host union-find + cycle check)."""
    from .fusion import fuse_groups
    config = config or FusionConfig()
    if fusion.task != "fusion_priority":
        raise ValueError(f"expected fusion_priority actions, got {fusion.task}")
    g = as_graph(graph)
    if len(fusion) != g.num_nodes:
        raise ValueError(f"fusion actions have length {len(fusion)}, want {g.num_nodes}")
    return FusedGraph(g, fuse_groups(g, fusion.actions, config.max_group))


def _check_inputs(n, d, placement, priorities):
    for asg, task in ((placement, "placement"), (priorities, "schedule_priority")):
        if asg.task != task:
            raise ValueError(f"expected {task} actions, got {asg.task}")
        if len(asg) != n:
            raise ValueError(f"{task} actions have length {len(asg)}, want {n} nodes")
    if placement.actions.min(initial=0) < 0 or placement.actions.max(initial=0) >= d:
        raise ValueError(f"placement action out of range [0,{d})")


def simulate_many(fg: FusedGraph, placements, priorities, topology, policy="priority",
                  baseline=0.0):
    """Batched DES: placements int [K, n] (numpy or device), priorities [K, n] or
    [n]; returns engine.SimBatch of device tensors."""
    T = torch()
    dev = T.device("cuda", context().device)
    h = as_fused(fg).install()
    top = as_topology(topology)
    pl = T.as_tensor(placements).to(device=dev, dtype=T.int32)
    if pl.dim() == 1:
        pl = pl.reshape(1, -1)
    pr = T.as_tensor(priorities).to(device=dev, dtype=T.int32)
    per = pr.dim() == 2
    if not per:
        pr = pr.reshape(-1)
    return simulate_batch(h, pl, pr, top, policy=policy, baseline=baseline,
                          prio_per_placement=per)


def simulate(fg: FusedGraph, placement: ActionAssignment, priorities: ActionAssignment, topology,
             policy: str = "priority", record_trace: bool = False) -> SimResult:
    """simulator.py:280-441 on device (bit-exact step time, busy, peak memory).
    record_trace=True records every started compute / transfer on the device
    (go_simulate_trace) and returns them as TraceEvents sorted like the reference
    (simulator.py:432-433: by start, end, kind, device string, group)."""
    if policy not in ("fifo", "priority"):
        raise ValueError(f"unknown policy {policy!r}")
    top = as_topology(topology)
    fg = as_fused(fg)
    _check_inputs(fg.graph.num_nodes, top.num_devices, placement, priorities)
    if record_trace:
        return _simulate_traced(fg, placement, priorities, top, policy)
    out = simulate_many(fg, placement.actions.reshape(1, -1), priorities.actions, top, policy)
    step = float(out.step_time.cpu().numpy()[0])
    vio = VIOLATIONS[int(out.violation.cpu().numpy()[0])]
    busy = out.busy.cpu().numpy()[0].tolist()
    peak = out.peak.cpu().numpy()[0].tolist()
    return SimResult(step_time=step, valid=vio is None, violation=vio, per_device_busy=busy,
                     peak_mem=peak, trace=None)


def _simulate_traced(fg, placement, priorities, top, policy) -> SimResult:
    from .engine import simulate_trace
    T = torch()
    dev = T.device("cuda", context().device)
    fg = as_fused(fg)
    h = fg.install()
    g = fg.graph
    pl = T.as_tensor(placement.actions).to(device=dev, dtype=T.int32)
    pr = T.as_tensor(priorities.actions).to(device=dev, dtype=T.int32)
    out, ev = simulate_trace(h, pl, pr, top, policy, capacity=g.num_nodes + g.num_edges)
    trace = [TraceEvent(float(e["t_start"]), float(e["t_end"]),
                        str(int(e["src_or_device"])) if e["kind"] == 0
                        else f"{int(e['src_or_device'])}->{int(e['dst'])}",
                        "compute" if e["kind"] == 0 else "transfer", int(e["group_id"]))
             for e in ev]
    trace.sort(key=lambda t: (t.time_start, t.time_end, t.kind, t.device, t.group_id))
    vio = VIOLATIONS[int(out.violation.cpu().numpy()[0])]
    return SimResult(step_time=float(out.step_time.cpu().numpy()[0]), valid=vio is None,
                     violation=vio, per_device_busy=out.busy.cpu().numpy()[0].tolist(),
                     peak_mem=out.peak.cpu().numpy()[0].tolist(), trace=trace)


def check_validity(graph, placement: ActionAssignment, topology) -> list[str]:
    """simulator.py:444-469 static re-check (host: placement range + colocation)."""
    g = as_graph(graph)
    d = as_topology(topology).num_devices
    if len(placement) != g.num_nodes:
        return ["length-mismatch"]
    acts = placement.actions
    if acts.min(initial=0) < 0 or acts.max(initial=0) >= d:
        return ["out-of-range"]
    for c in np.unique(g.coloc[g.coloc >= 0]):
        if len(np.unique(acts[g.coloc == c])) > 1:
            return ["colocation"]
    return []


def evaluate_assignments(graph, topology, assignments: dict, fusion_config=None,
                         policy: str = "priority", record_trace: bool = False) -> SimResult:
    """simulator.py:472-487: fusion pass, then simulate."""
    missing = [t for t in TASKS if t not in assignments]
    if missing:
        raise ValueError(f"assignments missing tasks: {missing}")
    fg = apply_fusion(graph, assignments["fusion_priority"], fusion_config)
    return simulate(fg, assignments["placement"], assignments["schedule_priority"], topology,
                    policy=policy, record_trace=record_trace)


_FUSIBLE = np.array([name not in NON_FUSIBLE for name in OP_INDEX], dtype=bool)

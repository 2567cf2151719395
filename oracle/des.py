"""Pure-Python restatement of the reference simulator, cost model, greedy
baseline and reward (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Follows /root/reference/pkg/src/graphopt/simulator.py (FusedGraph :86-172,
apply_fusion :180-277, simulate :280-441), costmodel.py (kernel_time :137,
fused_cost :149-187, uniform_topology :131), baselines.py (greedy_placement
:75-118) and training.py (reward :37-44).  Graphs are oracle/graph.py dicts.
"""
from __future__ import annotations

import heapq
import math
from collections import deque

import numpy as np

NON_FUSIBLE_OPS = (0, 1, 10, 11)  # matmul, conv, embed-lookup, other (simulator.py:28)


class Topology:
    """costmodel.py:56-107 as arrays: per-device peak/bw/cap, link bw[D][D]."""

    def __init__(self, peak, mem_bw, cap, link_bw):
        self.peak = [float(x) for x in peak]
        self.mem_bw = [float(x) for x in mem_bw]
        self.cap = [float(x) for x in cap]
        self.link_bw = [[float(x) for x in row] for row in link_bw]

    @property
    def d(self):
        return len(self.peak)


def uniform_topology(d, peak=1e12, mem_bw=1e11, cap=16e9, link_bw=1e10):  # costmodel.py:131
    return Topology([peak] * d, [mem_bw] * d, [cap] * d, [[link_bw] * d for _ in range(d)])


def kernel_time(flops, nbytes, peak, bw):  # costmodel.py:137-139
    return max(flops / peak, nbytes / bw)


class Fused:
    """FusedGraph (simulator.py:86-172) from a node -> group-label map."""

    def __init__(self, g, group_map):
        n = g["n"]
        gm = [int(x) for x in group_map]
        roots = sorted(set(gm))
        remap = {r: i for i, r in enumerate(roots)}
        gm = [remap[x] for x in gm]
        G = len(roots)
        groups = [[] for _ in range(G)]
        for v in range(n):
            groups[gm[v]].append(v)
        order = sorted(range(G), key=lambda i: groups[i][0])
        pos = {old: new for new, old in enumerate(order)}
        self.groups = [sorted(groups[i]) for i in order]
        self.group_map = [pos[x] for x in gm]
        src, dst, eb = g["src"].tolist(), g["dst"].tolist(), g["ebytes"].tolist()
        E = len(src)
        internal = [[] for _ in range(G)]
        ext_in = [[] for _ in range(G)]
        ext_out = [[] for _ in range(G)]
        for j in range(E):
            gs, gd = self.group_map[src[j]], self.group_map[dst[j]]
            if gs == gd:
                internal[gs].append(j)
            else:
                ext_out[gs].append(j)
                ext_in[gd].append(j)
        for lst in ext_out:
            lst.sort(key=lambda j: (src[j], dst[j]))  # stable, like list.sort
        self.ext_in, self.ext_out = ext_in, ext_out
        flops, ob = g["flops"].tolist(), g["out_bytes"].tolist()
        self.cost_flops, self.cost_bytes = [], []
        out_any = [[] for _ in range(n)]
        for j in range(E):
            out_any[src[j]].append(j)
        for i in range(G):  # costmodel.py:149-187
            members = self.groups[i]
            mset = set(members)
            fl = sum(flops[v] for v in members)
            reads = sum(eb[j] for j in ext_in[i])
            has_out = {src[j] for j in internal[i]} | {src[j] for j in ext_out[i]}
            writers = {src[j] for j in ext_out[i]} | (mset - has_out)
            writes = sum(ob[s] for s in sorted(writers))
            self.cost_flops.append(fl)
            self.cost_bytes.append(reads + writes)
        self.resident = []
        for i in range(G):  # simulator.py:125-133
            mset = set(self.groups[i])
            tot = 0.0
            for v in self.groups[i]:
                outs = out_any[v]
                if not outs or any(dst[j] not in mset for j in outs):
                    tot += ob[v]
            self.resident.append(tot)
        self.succ = [set() for _ in range(G)]
        self.pred = [set() for _ in range(G)]
        for i in range(G):
            for j in ext_out[i]:
                t = self.group_map[dst[j]]
                self.succ[i].add(t)
                self.pred[t].add(i)
        self.topo_index = self._topo()
        self.src, self.dst, self.eb = src, dst, eb

    def _topo(self):  # simulator.py:155-172
        G = len(self.groups)
        indeg = [len(p) for p in self.pred]
        heap = [i for i in range(G) if indeg[i] == 0]
        heapq.heapify(heap)
        index = [0] * G
        seen = 0
        while heap:
            i = heapq.heappop(heap)
            index[i] = seen
            seen += 1
            for j in sorted(self.succ[i]):
                indeg[j] -= 1
                if indeg[j] == 0:
                    heapq.heappush(heap, j)
        return index if seen == G else None


def singleton(g):
    return Fused(g, np.arange(g["n"]))


def simulate(g, fg: Fused, placement, priorities, top: Topology, policy="priority"):
    """simulator.py:280-441.  Returns dict(step_time, valid, violation, busy, peak)."""
    if policy not in ("fifo", "priority"):
        raise ValueError(policy)
    n, d = g["n"], top.d
    placement = [int(x) for x in placement]
    priorities = [int(x) for x in priorities]
    if len(placement) != n or len(priorities) != n:
        raise ValueError("length")
    if min(placement, default=0) < 0 or max(placement, default=0) >= d:
        raise ValueError("placement action out of range")
    G = len(fg.groups)
    gdev = [placement[fg.groups[i][0]] for i in range(G)]
    gpri = [priorities[fg.groups[i][0]] for i in range(G)]
    violation = None
    coloc = {}
    for v in range(n):
        c = int(g["coloc"][v])
        if c >= 0:
            coloc.setdefault(c, set()).add(gdev[fg.group_map[v]])
    if any(len(s) > 1 for s in coloc.values()):
        violation = "colocation"
    if fg.topo_index is None:
        return dict(step_time=0.0, valid=False, violation="cycle_after_fusion",
                    busy=[0.0] * d, peak=[0.0] * d)
    topo = fg.topo_index
    pending = [len(fg.ext_in[i]) for i in range(G)]
    finish = [0.0] * G
    ready_time = [0.0] * G
    busy = [0.0] * d
    running = [None] * d
    queues = [[] for _ in range(d)]
    links = {}
    link_busy = {}
    events = []
    seq = 0
    done = 0

    def key(i):
        if policy == "priority":
            return (-gpri[i], ready_time[i], topo[i])
        return (ready_time[i], topo[i])

    def mark_ready(i, t):
        ready_time[i] = t
        heapq.heappush(queues[gdev[i]], (*key(i), i))

    def deliver(i, t):
        pending[i] -= 1
        if pending[i] == 0:
            mark_ready(i, t)

    for i in range(G):
        if pending[i] == 0:
            mark_ready(i, 0.0)

    def schedule(t):
        nonlocal seq
        for lk in sorted(links):
            if not link_busy[lk] and links[lk]:
                j, gd = links[lk].popleft()
                link_busy[lk] = True
                dt = fg.eb[j] / top.link_bw[lk[0]][lk[1]]
                seq += 1
                heapq.heappush(events, (t + dt, 1, lk[0], lk[1], seq, gd))
        for dev in range(d):
            if running[dev] is None and queues[dev]:
                i = heapq.heappop(queues[dev])[-1]
                running[dev] = i
                dt = kernel_time(fg.cost_flops[i], fg.cost_bytes[i], top.peak[dev], top.mem_bw[dev])
                busy[dev] += dt
                seq += 1
                heapq.heappush(events, (t + dt, 0, dev, i, seq, i))

    schedule(0.0)
    while events:
        now = events[0][0]
        batch = []
        while events and events[0][0] == now:
            batch.append(heapq.heappop(events))
        for ev in batch:
            if ev[1] == 0:
                i, dev = ev[5], ev[2]
                running[dev] = None
                finish[i] = now
                done += 1
                for j in fg.ext_out[i]:
                    gd = fg.group_map[fg.dst[j]]
                    if gdev[gd] == dev:
                        deliver(gd, now)
                    else:
                        lk = (dev, gdev[gd])
                        if lk not in links:
                            links[lk] = deque()
                            link_busy[lk] = False
                        links[lk].append((j, gd))
            else:
                lk = (ev[2], ev[3])
                link_busy[lk] = False
                deliver(ev[5], now)
        schedule(now)
    step_time = max(finish) if G else 0.0
    assert done == G, "simulation deadlocked"
    peak = [0.0] * d
    mem = [[] for _ in range(d)]
    for i in range(G):
        if fg.resident[i] == 0.0:
            continue
        freed = max((finish[c] for c in sorted(fg.succ[i])), default=finish[i])
        mem[gdev[i]].append((finish[i], 0, fg.resident[i]))
        mem[gdev[i]].append((freed, 1, -fg.resident[i]))
    for dev in range(d):
        cur = 0.0
        for _, _, delta in sorted(mem[dev]):
            cur += delta
            peak[dev] = max(peak[dev], cur)
    if violation is None:
        for dev in range(d):
            if peak[dev] > top.cap[dev]:
                violation = "oom"
                break
    return dict(step_time=step_time, valid=violation is None, violation=violation,
                busy=busy, peak=peak)


def greedy_placement(g, d):
    """baselines.py:75-118 (O(D N^2) DP, earliest split on ties)."""
    n = g["n"]
    order = g["topo"]
    flops = g["flops"][order]
    prefix = np.concatenate([[0.0], np.cumsum(flops)])
    dp = np.full(n + 1, math.inf)
    dp[0] = 0.0
    choice = np.zeros((d + 1, n + 1), dtype=np.int64)
    for k in range(1, d + 1):
        nxt = np.full(n + 1, math.inf)
        for i in range(n + 1):
            cand = np.maximum(dp[: i + 1], prefix[i] - prefix[: i + 1])
            j = int(np.argmin(cand))
            nxt[i] = cand[j]
            choice[k, i] = j
        dp = nxt
    cuts = [n]
    i = n
    for k in range(d, 0, -1):
        i = int(choice[k, i])
        cuts.append(i)
    cuts.reverse()
    actions = np.zeros(n, dtype=np.int64)
    for dev in range(d):
        actions[order[cuts[dev]:cuts[dev + 1]]] = dev
    first = {}
    for v in range(n):
        c = int(g["coloc"][v])
        if c >= 0:
            if c not in first:
                first[c] = int(actions[v])
            actions[v] = first[c]
    return actions


def reward(step_time, baseline_time, valid):  # training.py:37-44
    if baseline_time <= 0:
        raise ValueError("baseline_time must be positive")
    if not valid:
        return -10.0
    return -math.sqrt(step_time / baseline_time)


def would_create_cycle(succ, a, b):  # simulator.py:180-196
    for x, y in ((a, b), (b, a)):
        stack = [s for s in succ[x] if s != y]
        seen = set(stack)
        while stack:
            s = stack.pop()
            if s == y:
                return True
            for t in succ[s]:
                if t == y:
                    return True
                if t not in seen:
                    seen.add(t)
                    stack.append(t)
    return False


def apply_fusion(g, pri, max_group=8):
    """simulator.py:199-277 -> group label per node (root ids)."""
    n = g["n"]
    pri = [int(x) for x in pri]
    parent = list(range(n))

    def find(v):
        while parent[v] != v:
            parent[v] = parent[parent[v]]
            v = parent[v]
        return v

    size = [1] * n
    succ = {v: set() for v in range(n)}
    pred = {v: set() for v in range(n)}
    for s, t in zip(g["src"].tolist(), g["dst"].tolist()):
        succ[s].add(t)
        pred[t].add(s)
    from .graph import neighbors
    nb = neighbors(g)
    ops = g["op"].tolist()
    visited = [False] * n
    for v in sorted(range(n), key=lambda v: (-pri[v], v)):
        if pri[v] > 0 and ops[v] not in NON_FUSIBLE_OPS:
            cands = [u for u in nb[v] if visited[u] and pri[u] > 0 and ops[u] not in NON_FUSIBLE_OPS]
            if cands:
                u = min(cands, key=lambda u: (-pri[u], u))
                rv, ru = find(v), find(u)
                if rv != ru and size[rv] + size[ru] <= max_group and not would_create_cycle(succ, rv, ru):
                    if size[rv] < size[ru]:
                        rv, ru = ru, rv
                    parent[ru] = rv
                    size[rv] += size[ru]
                    new_succ = (succ[rv] | succ[ru]) - {rv, ru}
                    new_pred = (pred[rv] | pred[ru]) - {rv, ru}
                    for s in succ[ru]:
                        pred[s].discard(ru)
                    for s in pred[ru]:
                        succ[s].discard(ru)
                    for s in succ[rv]:
                        pred[s].discard(rv)
                    for s in pred[rv]:
                        succ[s].discard(rv)
                    succ[rv] = new_succ
                    pred[rv] = new_pred
                    for s in new_succ:
                        pred[s].add(rv)
                    for s in new_pred:
                        succ[s].add(rv)
                    del succ[ru], pred[ru]
        visited[v] = True
    return np.array([find(v) for v in range(n)], np.int64)

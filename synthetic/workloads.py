"""Synthetic workload generator (restates workloads.py:1-280) producing `Graph`s.

Benchmark input only: it lets bench.py build the named DAGs on
the GPU box, where the reference package is absent.  Same families, closed-form
sizes and numpy draw order, so a spec yields the reference's graph exactly
(pinned by tests/test_host.py::test_workloads_match_reference against fixtures
from the reference)."""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from paper_2010_12438_b200.graph import BYTES_PER_ELEMENT, OP_INDEX, Graph, GraphError

FAMILIES = ("grid-rnn", "enc-dec-rnn", "attention-stack", "multi-branch-cnn", "cell-stack-cnn",
            "dilated-stack")
DEFAULT_NODE_CAP = 10_000
OPS_PER_CELL = 4


@dataclass(frozen=True)
class WorkloadSpec:
    family: str
    layers: int = 2
    steps: int = 4
    width: int = 32
    seed: int = 0

    def __post_init__(self):
        if self.family not in FAMILIES:
            raise GraphError(f"unknown family {self.family!r}")
        if self.layers <= 0 or self.steps <= 0 or self.width <= 0:
            raise GraphError("size params must be positive")

    @property
    def name(self) -> str:
        return f"{self.family}-L{self.layers}-S{self.steps}-w{self.width}-s{self.seed}"


def expected_node_count(spec: WorkloadSpec) -> int:
    L, S = spec.layers, spec.steps
    return {"grid-rnn": L * S * OPS_PER_CELL, "enc-dec-rnn": 2 * L * S * OPS_PER_CELL + 2 * S,
            "attention-stack": 1 + 10 * L, "multi-branch-cnn": 1 + 7 * L,
            "cell-stack-cnn": 4 * L, "dilated-stack": 1 + 4 * L * S + 2}[spec.family]


class _B:
    def __init__(self):
        self.op, self.flops, self.ob = [], [], []
        self.src, self.dst = [], []

    def node(self, op, shape, flops):
        self.op.append(OP_INDEX[op])
        self.flops.append(float(flops))
        self.ob.append(float(BYTES_PER_ELEMENT * math.prod(shape)) if shape else 0.0)
        return len(self.op) - 1

    def edge(self, s, d):
        self.src.append(s)
        self.dst.append(d)


def _w(rng, w):
    return max(4, int(round(w * rng.uniform(0.75, 1.25))))


def _cell(b, w, inputs):
    mm = b.node("matmul", (w,), 2.0 * w * w)
    ad = b.node("elementwise-add", (w,), w)
    sg = b.node("sigmoid", (w,), 4.0 * w)
    ml = b.node("elementwise-mul", (w,), w)
    for s in inputs:
        b.edge(s, mm)
    b.edge(mm, ad)
    b.edge(ad, sg)
    b.edge(sg, ml)
    b.edge(ad, ml)
    return ml


def _grid(b, rng, L, S, w):
    out = [[-1] * S for _ in range(L)]
    for l in range(L):
        for s in range(S):
            ins = ([out[l - 1][s]] if l > 0 else []) + ([out[l][s - 1]] if s > 0 else [])
            out[l][s] = _cell(b, _w(rng, w), ins)
    return out


def _gen(b, rng, spec):
    L, S, w = spec.layers, spec.steps, spec.width
    f = spec.family
    if f == "grid-rnn":
        _grid(b, rng, L, S, w)
    elif f == "enc-dec-rnn":
        enc = _grid(b, rng, L, S, w)
        dec = _grid(b, rng, L, S, w)
        for s in range(S):
            wa = _w(rng, w)
            att = b.node("matmul", (wa,), 2.0 * wa * wa)
            sm = b.node("softmax", (wa,), 5.0 * wa)
            for s2 in range(S):
                b.edge(enc[L - 1][s2], att)
            b.edge(att, sm)
            b.edge(sm, dec[0][s] - (OPS_PER_CELL - 1))
    elif f == "attention-stack":
        bi = b.node("embed-lookup", (w,), float(w))
        for _ in range(L):
            wb = _w(rng, w)
            q, k, v = (b.node("matmul", (wb,), 2.0 * wb * wb) for _ in range(3))
            sc = b.node("matmul", (wb,), 2.0 * wb * wb)
            sm = b.node("softmax", (wb,), 5.0 * wb)
            ctx = b.node("matmul", (wb,), 2.0 * wb * wb)
            f1 = b.node("matmul", (4 * wb,), 8.0 * wb * wb)
            rl = b.node("relu", (4 * wb,), 4.0 * wb)
            f2 = b.node("matmul", (wb,), 8.0 * wb * wb)
            res = b.node("elementwise-add", (wb,), wb)
            for m in (q, k, v):
                b.edge(bi, m)
            for s_, d_ in ((q, sc), (k, sc), (sc, sm), (sm, ctx), (v, ctx), (ctx, f1), (f1, rl),
                           (rl, f2), (f2, res), (bi, res)):
                b.edge(s_, d_)
            bi = res
    elif f == "multi-branch-cnn":
        bi = b.node("embed-lookup", (8, w), 8.0 * w)
        for _ in range(L):
            wb = _w(rng, w)
            outs = []
            for _br in range(3):
                cv = b.node("conv", (8, wb), 16.0 * wb * wb)
                rl = b.node("relu", (8, wb), 8.0 * wb)
                b.edge(bi, cv)
                b.edge(cv, rl)
                outs.append(rl)
            cat = b.node("concat", (24, wb), 0.0)
            for o in outs:
                b.edge(o, cat)
            bi = cat
    elif f == "cell-stack-cnn":
        co = []
        for c in range(L):
            wb = _w(rng, w)
            ca = b.node("conv", (8, wb), 16.0 * wb * wb)
            cb = b.node("conv", (8, wb), 16.0 * wb * wb)
            ad = b.node("elementwise-add", (8, wb), 8.0 * wb)
            rl = b.node("relu", (8, wb), 8.0 * wb)
            if c >= 1:
                b.edge(co[c - 1], ca)
                b.edge(co[max(0, c - 2)], cb)
            b.edge(ca, ad)
            b.edge(cb, ad)
            b.edge(ad, rl)
            co.append(rl)
    else:  # dilated-stack
        prev = b.node("embed-lookup", (w,), float(w))
        skips = []
        for _ in range(L * S):
            wb = _w(rng, w)
            cv = b.node("conv", (wb,), 16.0 * wb * wb)
            sg = b.node("sigmoid", (wb,), 4.0 * wb)
            ml = b.node("elementwise-mul", (wb,), wb)
            ad = b.node("elementwise-add", (wb,), wb)
            for s_, d_ in ((prev, cv), (cv, sg), (sg, ml), (cv, ml), (ml, ad), (prev, ad)):
                b.edge(s_, d_)
            skips.append(ml)
            prev = ad
        rd = b.node("reduce", (w,), float(w * len(skips)))
        sm = b.node("softmax", (w,), 5.0 * w)
        for s in skips:
            b.edge(s, rd)
        b.edge(rd, sm)


def gen_workload(spec: WorkloadSpec, node_cap: int = DEFAULT_NODE_CAP) -> Graph:
    want = expected_node_count(spec)
    if want > node_cap:
        raise GraphError(f"{spec.name}: {want} nodes exceeds cap {node_cap}")
    rng = np.random.default_rng(spec.seed)
    b = _B()
    _gen(b, rng, spec)
    ob = np.asarray(b.ob)
    src = np.asarray(b.src, np.int64)
    g = Graph(b.op, b.flops, ob, src, b.dst, ob[src] if len(src) else np.zeros(0), name=spec.name)
    assert g.num_nodes == want
    return g

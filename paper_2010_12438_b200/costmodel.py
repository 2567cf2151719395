"""Device topology and roofline cost model (mirrors costmodel.py:56-191).

`Topology` holds per-device peak FLOP/s, memory bandwidth and capacity plus one
link bandwidth per ordered device pair, as float64 arrays the DES reads.
`as_topology()` also accepts the reference's DeviceTopology (duck-typed)."""
from __future__ import annotations

import numpy as np


class TopologyError(ValueError):
    pass


class Topology:
    def __init__(self, peak, mem_bw, cap, link_bw):
        self.peak = np.ascontiguousarray(peak, dtype=np.float64)
        self.mem_bw = np.ascontiguousarray(mem_bw, dtype=np.float64)
        self.cap = np.ascontiguousarray(cap, dtype=np.float64)
        d = len(self.peak)
        lb = np.ascontiguousarray(link_bw, dtype=np.float64).reshape(d, d).copy()
        np.fill_diagonal(lb, 1.0)  # never read: same-device transfers are free
        self.link_bw = lb.reshape(-1)
        if (self.peak <= 0).any() or (self.mem_bw <= 0).any() or (self.cap <= 0).any():
            raise TopologyError("all rates must be positive")
        off = ~np.eye(d, dtype=bool)
        if (lb[off] <= 0).any():
            raise TopologyError("bandwidth must be positive")

    @property
    def num_devices(self) -> int:
        return len(self.peak)


def uniform_topology(num_devices: int, peak_flops: float = 1e12, mem_bw: float = 1e11,
                     mem_capacity: float = 16e9, link_bw: float = 1e10) -> Topology:
    """costmodel.py:131-134."""
    d = num_devices
    return Topology([peak_flops] * d, [mem_bw] * d, [mem_capacity] * d,
                    np.full((d, d), float(link_bw)))


def as_topology(top) -> Topology:
    if isinstance(top, Topology):
        return top
    d = top.num_devices
    lb = np.ones((d, d))
    for i in range(d):
        for j in range(d):
            if i != j:
                lb[i, j] = top.link(i, j).bandwidth
    return Topology([top.device(i).peak_flops for i in range(d)],
                    [top.device(i).mem_bw for i in range(d)],
                    [top.device(i).mem_capacity for i in range(d)], lb)


def kernel_time(flops: float, nbytes: float, peak: float, bw: float) -> float:
    """costmodel.py:137-139 (host helper; the DES evaluates it on device)."""
    return max(flops / peak, nbytes / bw)


def topology_from_dict(data: dict) -> Topology:
    """costmodel.py:115-128 JSON form: devices (id, peak_flops, mem_bw, mem_capacity)
    and links either {"uniform_bandwidth": bw} or a list of (src, dst, bandwidth)."""
    devs = sorted(data["devices"], key=lambda d: int(d["id"]))
    if [int(d["id"]) for d in devs] != list(range(len(devs))):
        raise TopologyError("device ids must be dense 0..D-1")
    d = len(devs)
    links_field = data.get("links")
    lb = np.zeros((d, d))
    have = np.eye(d, dtype=bool)
    if isinstance(links_field, dict):
        lb[:] = float(links_field["uniform_bandwidth"])
        have[:] = True
    else:
        for l in links_field or []:
            s_, t_ = int(l["src"]), int(l["dst"])
            if not (0 <= s_ < d and 0 <= t_ < d):  # costmodel.py:72-74
                raise TopologyError(f"link references unknown device: {s_}->{t_}")
            lb[s_, t_] = float(l["bandwidth"])
            have[s_, t_] = True
    if not have.all():  # costmodel.py:75-78
        i, j = map(int, np.argwhere(~have)[0])
        raise TopologyError(f"no link for device pair {i}->{j}")
    return Topology([float(x["peak_flops"]) for x in devs], [float(x["mem_bw"]) for x in devs],
                    [float(x["mem_capacity"]) for x in devs], lb)


def load_topology(path) -> Topology:
    """costmodel.py:110-112."""
    import json
    from pathlib import Path
    return topology_from_dict(json.loads(Path(path).read_text()))

#!/usr/bin/env python
"""Per-kernel share of an `ncu --metrics gpu__time_duration.sum --csv` launch list.

    python scripts/launch_summary.py gpurun_out/launches.csv "<command>" > profiles/rN_launches.txt
ncu serialises launches and runs them cold, so absolute times are not bench times;
the per-kernel SHARE of the step is what bench.py's CUDA-event split should match."""
import collections
import csv
import sys

SCALE = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def main():
    path = sys.argv[1]
    cmd = sys.argv[2] if len(sys.argv) > 2 else ""
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi, ui = (h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"),
                      h.index("Metric Unit"))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        ms = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-6)
        name = r[ki].split("(")[0].replace("void ", "")[:80]
        agg[name][0] += 1
        agg[name][1] += ms
    tot = sum(a[1] for a in agg.values())
    print("ncu --metrics gpu__time_duration.sum --clock-control none (cold cache, serialised)")
    if cmd:
        print("command:", cmd)
    print(f"{sum(a[0] for a in agg.values())} launches, {tot:.1f} ms total\n")
    for name, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        if t / tot < 1e-4:
            continue
        print(f"{t:12.3f} ms {100 * t / tot:5.1f}%  n={n:6d}  {name}")


if __name__ == "__main__":
    main()

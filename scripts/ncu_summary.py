#!/usr/bin/env python
"""Summarise an `ncu --set full` report into profiles/ (tracked evidence).

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r1_ncu_summary \
        [--forwards-per-launch F]

Writes <out>.json (per-kernel duration, DRAM bytes, pipe utilisations, top stall
reasons) and <out>.txt (the same as a table).  `traffic` holds the per-kernel DRAM
bytes bench.py reports next to its roofline."""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = {
    "time_us": ("gpu__time_duration.sum", 1e-3),  # reported in ms or us depending on ncu
    "dram_read": ("dram__bytes_read.sum", 1.0),
    "dram_write": ("dram__bytes_write.sum", 1.0),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1.0),
    "xu_pipe_pct": ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", 1.0),
    "tensor_pipe_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "l2_pct": ("lts__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "regs": ("launch__registers_per_thread", 1.0),
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0,
         "usecond": 1.0, "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def main():
    rep, out = sys.argv[1], sys.argv[2]
    hdr, units, data = raw(rep)
    idx = {h: i for i, h in enumerate(hdr)}
    kernels = []
    for d in data:
        k = {"kernel": d[idx["Kernel Name"]]}
        for key, (m, _) in METRICS.items():
            if m not in idx:
                continue
            v = d[idx[m]].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                continue
            u = units[idx[m]]
            if key == "time_us":
                x *= SCALE.get(u, 1.0)
            elif key.startswith("dram_") and key != "dram_pct":
                x *= SCALE.get(u, 1.0)
            k[key] = x
        stalls = {h.split("issue_stalled_")[1]: float(d[i] or 0) for h, i in idx.items()
                  if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and not h.endswith("not_issued") and d[i]}
        tot = sum(stalls.values()) or 1.0
        k["top_stalls"] = {s: round(v / tot, 3) for s, v in
                           sorted(stalls.items(), key=lambda kv: -kv[1])[:4]}
        kernels.append(k)
    # per-kernel-family aggregates
    fam = defaultdict(list)
    for k in kernels:
        name = k["kernel"].split("(")[0].replace("void ", "")
        fam[name].append(k)
    traffic = {}
    for name, ks in fam.items():
        short = name.split("::")[-1].split("<")[0]
        b = sum(k.get("dram_read", 0) + k.get("dram_write", 0) for k in ks) / len(ks)
        traffic.setdefault(f"{short}_bytes_per_launch_F1", b)
    for k in ("attn_f16_kernel_bytes_per_launch_F1", "attn_tc_fixed_kernel_bytes_per_launch_F1"):
        if k in traffic:
            traffic.setdefault("heads_attention_bytes_per_forward", traffic[k])
    if "segment_max128_kernel_bytes_per_launch_F1" in traffic:
        traffic["segment_max_bytes_per_launch_F1"] = traffic["segment_max128_kernel_bytes_per_launch_F1"]
    res = {"report": rep, "kernels": kernels, "traffic": traffic}
    with open(out + ".json", "w") as f:
        json.dump(res, f, indent=1)
    with open(out + ".txt", "w") as f:
        f.write(f"# {rep}\n# kernel | us | dram MB (r+w) | issue% | xu% | tensor% | dram% | l2% | top stalls\n")
        for k in kernels:
            f.write("{:<60} {:>9.1f} {:>9.1f} {:>6.1f} {:>6.1f} {:>6.1f} {:>6.1f} {:>6.1f}  {}\n".format(
                k["kernel"][:60], k.get("time_us", 0), (k.get("dram_read", 0) + k.get("dram_write", 0)) / 1e6,
                k.get("issue_active_pct", 0), k.get("xu_pipe_pct", 0), k.get("tensor_pipe_pct", 0),
                k.get("dram_pct", 0), k.get("l2_pct", 0), k["top_stalls"]))
    print(open(out + ".txt").read())


if __name__ == "__main__":
    main()

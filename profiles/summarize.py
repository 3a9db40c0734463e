#!/usr/bin/env python
"""Summarise ncu captures of bench.py into committed text files.

    python profiles/summarize.py <tag> <launches.csv> <full.ncu-rep>[,<more captures>]

Writes profiles/<tag>_launches.txt (per-kernel device time of one bench
process, from `ncu --metrics gpu__time_duration.sum`), profiles/<tag>_full.txt
(per-launch DRAM traffic, throughput and stall picture from `ncu --set full`)
and updates profiles/traffic.json (DRAM bytes per launch of the roofline
kernel, read by bench.py).
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    ci = {h: i for i, h in enumerate(rows[hi])}
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= ci["Metric Value"] or r[ci["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ci["Kernel Name"]].split("(")[0]
        v = float(r[ci["Metric Value"]].replace(",", ""))
        scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(r[ci["Metric Unit"]], 1e-6)
        a = agg.setdefault(name, [0, 0.0])
        a[0] += 1
        a[1] += v * scale
    return agg


def full(path):
    # a .ncu-rep (read through ncu -i) or its `--page raw --csv` export
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    ci = {h: i for i, h in enumerate(hdr)}
    res = []
    for r in rows[2:]:
        d = {"kernel": r[ci["Kernel Name"]].split("(")[0]}
        for k in ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                  "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                  "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
                  "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                  "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                  "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]:
            if k in ci:
                d[k] = (r[ci[k]], units[ci[k]])
        res.append(d)
    return res


def to_bytes(val_unit):
    v, u = val_unit
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u, 1)


def to_ms(val_unit):
    v, u = val_unit
    v = float(v.replace(",", ""))
    return v * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
                "second": 1e3, "s": 1e3}.get(u, 1)


def main():
    tag, lpath, fpath = sys.argv[1:4]
    agg = launches(lpath)
    tot = sum(a[1] for a in agg.values())
    lines = [f"# {tag}: per-kernel device time of one `python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline` process",
             "# (ncu --metrics gpu__time_duration.sum --clock-control none; cold-cache, serialised:",
             "#  compare SHARES, not absolutes).  Includes input generation (torch/cuSOLVER QR) and",
             "#  the warm-up + timed solve.", f"# total {tot:.1f} ms", "",
             f"{'ms':>10} {'share':>7} {'launches':>8}  kernel"]
    for name, (cnt, ms) in sorted(agg.items(), key=lambda x: -x[1][1])[:40]:
        lines.append(f"{ms:10.3f} {100 * ms / tot:6.2f}% {cnt:8d}  {name[:110]}")
    ours = {k: v for k, v in agg.items() if "msvd::" in k}
    ot = sum(v[1] for v in ours.values())
    lines += ["", f"# msvd kernels only: {ot:.1f} ms", ""]
    for name, (cnt, ms) in sorted(ours.items(), key=lambda x: -x[1][1]):
        lines.append(f"{ms:10.3f} {100 * ms / ot:6.2f}% {cnt:8d}  {name[:110]}")
    open(os.path.join(HERE, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")

    res, seen = [], set()
    for d in [x for fp in fpath.split(",") for x in full(fp)]:  # first launch of each kernel
        if d["kernel"] not in seen:
            seen.add(d["kernel"])
            res.append(d)
    lines = [f"# {tag}: ncu --set full --clock-control none on the C2 bench (m=1e6, n=1e3, b=1), first launch of each", ""]
    traffic = {}
    for d in res:
        lines.append(d["kernel"])
        for k, v in d.items():
            if k != "kernel":
                lines.append(f"    {k:72s} {v[0]:>16} {v[1]}")
        if "gpu__time_duration.sum" in d and "dram__bytes_read.sum" in d:
            ms = to_ms(d["gpu__time_duration.sum"])
            rb = to_bytes(d["dram__bytes_read.sum"])
            wb = to_bytes(d["dram__bytes_write.sum"])
            lines.append(f"    => DRAM traffic {(rb + wb) / 1e9:.4f} GB in {ms:.3f} ms = {(rb + wb) / ms / 1e6:.0f} GB/s")
            if "gram_kernel" in d["kernel"] and "gram_kernel" not in traffic:
                traffic["gram_kernel"] = rb + wb
            if "apply" in d["kernel"] and "apply_kernel" not in traffic:
                traffic["apply_kernel"] = rb + wb
        lines.append("")
    open(os.path.join(HERE, f"{tag}_full.txt"), "w").write("\n".join(lines) + "\n")
    tpath = os.path.join(HERE, "traffic.json")
    cur = json.load(open(tpath)) if os.path.exists(tpath) else {}
    cur["c2"] = traffic
    cur["c2"]["source"] = f"profiles/{tag}_full.txt"
    json.dump(cur, open(tpath, "w"), indent=1)
    print("\n".join(lines[:60]))


if __name__ == "__main__":
    main()

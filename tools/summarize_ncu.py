#!/usr/bin/env python
"""Summarise ncu outputs from gpurun_out/ into profiles/ (tracked).

    python tools/summarize_ncu.py --launches gpurun_out/launches.csv \
        --report gpurun_out/pd_l0.ncu-rep --tag r01

Writes profiles/<tag>_launches.md (per-kernel share of device time from the
`gpu__time_duration.sum` launch list, PD launches split by grid = pyramid
level), profiles/<tag>_pd_full.md (key `--set full` metrics of the dominant
kernel) and profiles/pd_traffic.json (DRAM bytes per launch, read by bench.py).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path, one_step=False):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
    tot, cnt, lvl, lvc = collections.Counter(), collections.Counter(), collections.Counter(), collections.Counter()
    body = rows[hi + 1:]
    if one_step:  # exactly the first tracked step: 2nd .. 3rd ingest launch
        ing = [i for i, r in enumerate(body) if len(r) > ki and "k_gray8_to_unit" in r[ki]]
        body = body[ing[1]:ing[2]] if len(ing) > 2 else body[ing[1]:]
    for r in body:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("ft::<unnamed>::", "")
        name = name.replace("unnamed>::", "")
        v = float(r[vi])
        tot[name] += v
        cnt[name] += 1
        if "k_pd_tile" in name or "k_pd_" in name:
            lvl[(name, r[gi])] += v
            lvc[(name, r[gi])] += 1
    T = sum(tot.values())
    out = ["| kernel | launches | device time (ms) | share |", "|---|---:|---:|---:|"]
    for k, v in tot.most_common():
        out.append(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {100 * v / T:.1f}% |")
    out += ["", "PD launches by grid (grid.z = streams; grid.x*y = tiles per level):", "",
            "| kernel | grid | launches | total (ms) | share | per launch (us) |", "|---|---|---:|---:|---:|---:|"]
    for (k, g), v in sorted(lvl.items(), key=lambda x: -x[1]):
        out.append(f"| `{k}` | {g} | {lvc[(k, g)]} | {v / 1e6:.3f} | {100 * v / T:.1f}% | "
                   f"{v / lvc[(k, g)] / 1e3:.1f} |")
    out.append(f"\nTotal device time {T / 1e6:.3f} ms (ncu: serialized, cold caches -- compare shares).")
    return "\n".join(out)


def pick(path, kernel="k_pd_tile"):
    """ncu -s value selecting the 2nd launch of `kernel` with the largest grid
    (the finest level, not the first launch of a warp) in a launch list."""
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, gi = h.index("Kernel Name"), h.index("Grid Size")
    seq = [r[gi] for r in rows[hi + 1:] if len(r) > gi and kernel in r[ki]]

    def cells(g):
        n = 1
        for x in g.strip("()").split(","):
            n *= int(x)
        return n
    big = max(cells(g) for g in seq)
    hits = [i for i, g in enumerate(seq) if cells(g) == big]
    return hits[1]


def ncu_csv(report, *args):
    res = subprocess.run(["ncu", "-i", report, *args, "--csv"], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(res.stdout)))


def full(report):
    det = ncu_csv(report, "--page", "details")
    h = det[0]
    want = ["Kernel Name", "Grid Size", "Block Size", "Duration", "Registers Per Thread",
            "Achieved Occupancy", "Theoretical Occupancy", "Issue Slots Busy",
            "Executed Ipc Active", "Warp Cycles Per Issued Instruction",
            "Avg. Active Threads Per Warp", "DRAM Throughput", "Memory Throughput",
            "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Instructions"]
    got = {}
    for row in det[1:]:
        d = dict(zip(h, row))
        if d.get("Metric Name") in want and d["Metric Name"] not in got:
            got[d["Metric Name"]] = f"{d['Metric Value']} {d['Metric Unit']}".strip()
    kname = det[1][h.index("Kernel Name")] if len(det) > 1 and "Kernel Name" in h else "?"
    raw = ncu_csv(report, "--page", "raw")
    rh, rv = raw[0], raw[2]
    keys = ["dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "gpu__time_duration.sum"]
    rawv = {k: rv[rh.index(k)] for k in keys if k in rh}
    units = {k: raw[1][rh.index(k)] for k in keys if k in rh}
    stalls = []
    for i, n in enumerate(rh):
        if "smsp__pcsamp_warps_issue_stalled" in n and "not_issued" not in n:
            try:
                stalls.append((float(rv[i].replace(",", "")), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
            except ValueError:
                pass
    st = sum(x for x, _ in stalls) or 1.0
    lines = [f"kernel: `{kname}`", "", "| metric | value |", "|---|---|"]
    lines += [f"| {k} | {v} |" for k, v in got.items()]
    lines += [f"| {k} | {rawv[k]} {units[k]} |" for k in rawv]
    lines += ["", "Warp stall reasons (PC sampling share):", "", "| reason | share |", "|---|---:|"]
    lines += [f"| {n} | {100 * x / st:.1f}% |" for x, n in sorted(stalls, reverse=True)[:10]]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    traffic = None
    if "dram__bytes_read.sum" in rawv and "dram__bytes_write.sum" in rawv:
        traffic = (float(rawv["dram__bytes_read.sum"]) * mult.get(units["dram__bytes_read.sum"], 1) +
                   float(rawv["dram__bytes_write.sum"]) * mult.get(units["dram__bytes_write.sum"], 1))
    return "\n".join(lines), traffic, got.get("Grid Size", "")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--report")
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--pick", help="launch list: print the ncu -s index of a finest PD launch")
    ap.add_argument("--note", default="")
    ap.add_argument("--one-step", action="store_true",
                    help="launch list: keep only the first tracked step")
    ap.add_argument("--stream-pixels", type=float, default=0.0,
                    help="streams x pixels of the captured launch (normalises traffic)")
    a = ap.parse_args()
    if a.pick:
        print(pick(a.pick))
        return
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if a.launches:
        md = launches(a.launches, a.one_step)
        open(os.path.join(ROOT, "profiles", f"{a.tag}_launches.md"), "w").write(
            f"# {a.tag}: launch list (ncu --metrics gpu__time_duration.sum)\n\n{a.note}\n\n{md}\n")
    if a.report:
        md, traffic, grid = full(a.report)
        open(os.path.join(ROOT, "profiles", f"{a.tag}_pd_full.md"), "w").write(
            f"# {a.tag}: ncu --set full of the dominant kernel\n\n{a.note}\n\n{md}\n")
        if traffic is not None:
            rec = {"dram_bytes_per_launch": traffic, "grid": grid, "source": a.report,
                   "tag": a.tag, "note": a.note}
            if a.stream_pixels:
                rec["bytes_per_stream_pixel"] = traffic / a.stream_pixels
            json.dump(rec, open(os.path.join(ROOT, "profiles", "pd_traffic.json"), "w"), indent=1)
    print("ok")


if __name__ == "__main__":
    main()

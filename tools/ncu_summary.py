"""Summarise an ncu report: key metrics, stall reasons, SASS opcode mix.
    python tools/ncu_summary.py gpurun_out/x.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys


def run(rep, page, *extra):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep):
    rows = run(rep, "details")
    hdr = rows[0]
    keep = ("Duration", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
            "Achieved Occupancy", "Executed Instructions", "Grid Size", "Block Size",
            "DRAM Throughput", "Local Memory Spilling Requests", "Warp Cycles Per Issued Instruction")
    name = None
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", name)
        if d.get("Metric Name") in keep:
            print(f"{d['Metric Name']:36s} {d['Metric Value']} {d['Metric Unit']}")
    print("kernel:", name)
    raw = run(rep, "raw")
    d = dict(zip(raw[0], raw[2]))
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v)
          for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
          and not k.endswith("_not_issued") and v.replace(".", "").isdigit()}
    tot = sum(st.values()) or 1
    print("stalls:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in
                               sorted(st.items(), key=lambda kv: -kv[1]) if v / tot > 0.01))
    for k in ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
              "dram__bytes_read.sum", "dram__bytes_write.sum"):
        print(k, d.get(k))
    src = run(rep, "source", "--print-source", "sass")
    h = src[1]
    ix, isrc = h.index("Instructions Executed"), h.index("Source")
    ops, tot = collections.Counter(), 0
    for r in src[2:]:
        try:
            n = int(r[ix])
        except (ValueError, IndexError):
            continue
        tok = r[isrc].split()
        if not tok:
            continue
        o = tok[1] if tok[0].startswith("@") else tok[0]
        ops[o.split(".")[0]] += n
        tot += n
    print("opcode mix:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in ops.most_common(24)))


if __name__ == "__main__":
    main(sys.argv[1])

"""Per-source-line instruction counts of a kernel: joins an ncu report's
SASS execution counts with nvdisasm line info of the same cubin.
    python tools/ncu_lines.py report.ncu-rep kernel.cubin mangled_substring [file.cu]"""
import collections
import csv
import io
import re
import subprocess
import sys


def main(rep, cubin, fn, srcfile=None):
    dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
    line_of, cur, on, curfile = {}, None, False, None
    for ln in dis.splitlines():
        if ln.startswith("//---") and ".text." in ln:
            on = fn in ln
        m = re.search(r'File "([^"]+)", line (\d+)', ln)
        if m:
            curfile, cur = m.group(1), int(m.group(2))
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if m and on:
            line_of[int(m.group(1), 16)] = (curfile, cur)
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[1]
    ia, ix = h.index("Address"), h.index("Instructions Executed")
    isamp = h.index("Warp Stall Sampling (All Samples)")
    base = None
    per = collections.Counter()
    stall = collections.Counter()
    tot = 0
    tot_s = 0
    for r in rows[2:]:
        try:
            a, n = int(r[ia], 16), int(r[ix])
        except (ValueError, IndexError):
            continue
        if base is None:
            base = a
        f, l = line_of.get(a - base, ("?", 0))
        if srcfile and srcfile not in (f or ""):
            l = -l
        key = (f.split("/")[-1] if f else "?", l)
        per[key] += n
        tot += n
        try:
            st = int(r[isamp] or 0)
        except ValueError:
            st = 0
        stall[key] += st
        tot_s += st
    src = {}
    order = stall if "--stalls" in sys.argv else per
    for (f, l), _ in order.most_common(60):
        print(f"{100 * per[(f, l)] / tot:5.1f}% instr  {100 * stall[(f, l)] / max(tot_s, 1):5.1f}% "
              f"stall-samples  {f}:{l}")


if __name__ == "__main__":
    main(*[a for a in sys.argv[1:] if not a.startswith("--")])

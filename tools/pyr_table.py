#!/usr/bin/env python
"""Per-kernel table (duration, algorithmic bytes, achieved GB/s vs the
measured HBM peak) from an `ncu --metrics gpu__time_duration.sum,...
--csv` log of the stencil kernels (tools/gpu_pyr_profile.sh)."""
import collections
import csv
import sys

# algorithmic bytes per processing-level pixel (fp64 = 8 B; SD, 32 streams)
PX = 720 * 576
BYTES = {  # kernel -> (bytes per output pixel, output pixels as a fraction of PX)
    "k_gray8_to_unit": 1 + 8,              # u8 in, f64 out
    "k_scale_copy": 16,                    # f64 in, f64 out
    "k_blur_decimate<double, 0>": 4 * 8 + 8 + 8,   # 4 inputs per output, out + scaled out
    "k_central_grad": 8 + 16,              # I1 in, ix iy out
    "k_st_combine": 32,                    # img px py in, out
    "k_upsample": 16 + 4,                  # u1 u2 out, coarse (1/4) in
    "k_median": 32,                        # u1 u2 in, out
    "k_warp_setup": 72,                    # u, I0, 3 gathers in; gx gy rho0 out
}
PEAK = 6366.5  # GB/s, MEASURED_PEAKS.json hbm_gbs


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, gi, mi, vi, ui, ii = (h.index(k) for k in ("Kernel Name", "Grid Size", "Metric Name",
                                                    "Metric Value", "Metric Unit", "ID"))
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        mult = {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(r[ui], 1)
        if r[mi] == "gpu__time_duration.sum":
            per[r[ii]]["t"] = float(r[vi].replace(",", "")) * mult
        per[r[ii]]["name"] = r[ki].split("(")[0].replace("void ", "").replace("ft::<unnamed>::", "").replace("unnamed>::", "")
        per[r[ii]]["grid"] = r[gi]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in per.values():
        a = agg[(d["name"], d["grid"])]
        a[0] += 1
        a[1] += d["t"]
    best = {}
    for (n, g), (c, t) in agg.items():  # finest-level launch of each kernel = largest grid
        gx, gy, gz = (int(v) for v in g.strip("()").split(","))
        if n in BYTES and (n not in best or gx * gy > best[n][0]):
            best[n] = (gx * gy, g, gz, c, t)
    print("| kernel (finest level, 32 SD streams) | grid | launches | us / launch | "
          "algorithmic MB | GB/s | of HBM peak |")
    print("|---|---|---:|---:|---:|---:|---:|")
    for n, (_, g, gz, c, t) in sorted(best.items(), key=lambda x: -x[1][4]):
        frac = 0.25 if "blur" in n else 1.0  # blur: bytes counted per output (1/4 of PX)
        mb = BYTES[n] * PX * frac * gz / 1e6
        us = t / c / 1e3
        print(f"| `{n}` | {g} | {c} | {us:.1f} | {mb:.1f} | {mb / us * 1e3:.0f} | "
              f"{mb / us * 1e3 / PEAK * 100:.0f} % |")


if __name__ == "__main__":
    main(sys.argv[1])

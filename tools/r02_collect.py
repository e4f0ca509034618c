"""Copy the outputs of tools/r02_final.sh (gpurun_out/r02_*) into profiles/:
bench lines, GPU suite tail, launch list and the --set full summaries of the
PD and ROF kernels, and profiles/pd_profile.json (read by bench.py's
roofline).  python tools/r02_collect.py"""
import json
import os
import re
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import summarize_ncu as S  # noqa: E402

O, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")


def main():
    for f in ("default", "light", "klt", "c3", "c4", "single", "total64", "reference"):
        lines = [x for x in open(os.path.join(O, f"r02_bench_{f}.jsonl")).read().splitlines()
                 if x.startswith("{")]
        open(os.path.join(P, f"r02_bench_{f}.jsonl"), "w").write(lines[-1] + "\n")
    shutil.copy(os.path.join(O, "r02_bench_gpus2.txt"), os.path.join(P, "r02_bench_gpus2.txt"))
    tail = open(os.path.join(O, "r02_pytest_gpu.log")).read().splitlines()[-3:]
    open(os.path.join(P, "r02_pytest_gpu.txt"), "w").write("\n".join(tail) + "\n")
    md = S.launches(os.path.join(O, "r02_launches.csv"), one_step=True)
    open(os.path.join(P, "r02_launches.md"), "w").write(
        "# r02: launch list (ncu --metrics gpu__time_duration.sum)\n\nCommand: `ncu --metrics "
        "gpu__time_duration.sum --clock-control none -c 2300 python bench.py --steps 1 --warmup 1 "
        "--no-cpu-baseline` (64 SD streams, C2 default FlowParams); rows = the first tracked step "
        "(between the 2nd and 3rd ingest launch).  Final round-2 build.\n\n" + md + "\n")
    md, traffic, _ = S.full(os.path.join(O, "r02_pd_full.ncu-rep"))
    open(os.path.join(P, "r02_pd_full.md"), "w").write(
        "# r02: ncu --set full of the dominant kernel\n\nCommand: `ncu --set full --import-source on "
        "--clock-control none -k regex:k_pd_tile -s 300 -c 1 python bench.py --steps 1 --warmup 1 "
        "--no-cpu-baseline` (64 SD streams): a finest-level middle launch, "
        "k_pd_tile<32,16,2,2,kSchedMid> -- 32x32 tiles of 512 threads, each thread owning two "
        "adjacent rows, halo 4, (P D)x4 fully unrolled with closed-form cone rows, TMA box loads "
        "(U/PX/PY with apron, G/RT) + L2 prefetch of the next wave's boxes + TMA box stores of the "
        "interior, (rho0, 1/|grad|^2) from shared staging (no division in the prologue), the first "
        "pixel's own p kept in registers between the primal and the dual step, zero numerators kept "
        "off the division slow path.  Final round-2 build.\n\n" + md + "\n")
    t = md

    def g(name):
        return float(re.search(r"\| " + re.escape(name) + r" \| ([0-9.]+)", t).group(1))
    d = json.load(open(os.path.join(P, "pd_profile.json")))
    d["dram_bytes_per_stream_pixel_per_launch"] = traffic / (720 * 576 * 64)
    d["issue_slots_busy"] = round(g("Issue Slots Busy") / 100, 4)
    d["fp64_pipe_active"] = round(
        g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active") / 100, 4)
    json.dump(d, open(os.path.join(P, "pd_profile.json"), "w"), indent=1)
    md, traffic, _ = S.full(os.path.join(O, "r02_rof_full.ncu-rep"))
    open(os.path.join(P, "r02_rof_full.md"), "w").write(
        "# r02: ncu --set full of a ROF launch (k_rof_tile, 64x32 tiles)\n\nCommand: `ncu --set full "
        "--import-source on --clock-control none -k regex:k_rof_tile -s 30 -c 1 python bench.py "
        "--steps 1 --warmup 1 --no-cpu-baseline` (64 SD streams, a 4-iteration launch of the 40 ROF "
        "dual steps; iteration loop not unrolled, zero numerators off the division slow path, "
        "img/weight divided once per pass: this capture is a pass's first launch, which also stores "
        "the img/weight plane; the other nine launches read it back).  Final round-2 build.\n\n"
        + md + f"\n\nDRAM bytes of the launch: {traffic:.3g}.\n")
    print(json.dumps(d))


if __name__ == "__main__":
    main()

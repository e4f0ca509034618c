#!/usr/bin/env python
"""Benchmark: tracked SD frames/s per B200 (BASELINE.json metric) on config
C2 -- 720x576, 100 tracks with scale change and occlusion, detections every
5th frame, default FlowParams (6 scales x 5 warps x 50 iterations), fp64.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--streams B]
    python bench.py --impl reference ...     (CPU reference arm)

One step = one frame of each of the B independent streams resident on a GPU
(config C5's stream sharding: ranks own disjoint streams, no collective on
the data path; the only collectives are the timing barrier / max).
`value` is device-timed (CUDA events on the tracker stream, inputs already
in HBM); `e2e` goes through the public Tracker API with host frames in
pinned memory, H2D of frames+detections and D2H of the track table inside
the timed region.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tracked frames/sec per GPU at 720×576, 100 tracks; HBM-roofline fraction"
W_, H_, N_OBJ, DET_EVERY = 720, 576, 100, 5
SCALES = None  # FlowParams.pyramid_scales (None: auto_scales, 6 at SD)
WORKLOAD = ("C2 streams batched as in C5 (64 SD streams per GPU): 720x576 SD, 100 tracks, "
            "scale change + occlusion, detections every 5th frame, TV-L1 6 scales x 5 warps x "
            "50 iterations, ROF 40 iterations, fp64")
# BASELINE.json configs other than the headline, as measured (non-headline)
# lines: (W, H, tracks, detector cadence, pyramid scales, algorithmic bytes /
# frame from SURVEY 8(d), workload text)
CONFIGS = {
    "c2": None,
    "c3": (1920, 1080, 200, 1, 4, 27.47e9,
           "C3: 1920x1080 HD (processed at level 1, 960x540), 200 tracks, detections every "
           "frame, TV-L1 4 scales x 5 warps x 50 iterations, ROF 40 iterations, fp64"),
    "c4": (3840, 2160, 500, 1, 5, 27.69e9,
           "C4: 3840x2160 UHD (processed at level 2, 960x540), 500 tracks, detections every "
           "frame, TV-L1 5 scales x 5 warps x 50 iterations, ROF 40 iterations, fp64 "
           "(the KLT forward-backward check has no counterpart on the reference path)"),
}


def apply_config(name: str) -> None:
    global W_, H_, N_OBJ, DET_EVERY, SCALES, WORKLOAD, METRIC
    c = CONFIGS.get(name)
    if c is None:
        return
    W_, H_, N_OBJ, DET_EVERY, SCALES, fb, WORKLOAD = c
    FRAME_BYTES["default"] = fb
    METRIC = f"tracked frames/sec per GPU at {W_}×{H_}, {N_OBJ} tracks; HBM-roofline fraction"


# ----------------------------------------------------------------------------
def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def allmax(ws, v: float) -> float:
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def stream_seed(rank: int, s: int) -> int:
    return 1000 + 64 * rank + s


def gen_streams(rank: int, n_streams: int, n_frames: int):
    from paper_1910_06017_b200.synth import make_sequence
    out = []
    for s in range(n_streams):
        out.append(make_sequence(W_, H_, N_OBJ, n_frames, seed=stream_seed(rank, s),
                                 det_every=DET_EVERY, scale_change=True, jitter=1.0))
    return out


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:  # timed region shorter than the sampling period: one query now
            try:
                q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                     "clocks_event_reasons.hw_thermal_slowdown,"
                     "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=10).stdout
                self.rows = [[x.strip() for x in ln.split(",")] for ln in out.splitlines() if ln]
            except Exception:
                pass
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def det_records(dets, max_dets):
    from paper_1910_06017_b200._lib import DET_DTYPE
    rec = np.zeros(max_dets, dtype=DET_DTYPE)
    if dets is None:
        return rec, -1
    for j, d in enumerate(dets):
        rec[j] = (d.class_id, d.class_id, d.score, *d.box)
    return rec, len(dets)


def workload(args) -> str:
    if getattr(args, "flow", "default") == "light":
        return WORKLOAD.replace("6 scales x 5 warps x 50 iterations",
                                "6 scales x 2 warps x 10 iterations (SURVEY 8(d) light FlowParams)")
    return WORKLOAD


# ----------------------------------------------------------------------------
# CPU side: the oracle port of the reference, one SD stream-frame per process
def _flow_params(flow: str, oracle: bool = False):
    """default: FlowParams() (the headline C2 workload); light: SURVEY 8(d)'s
    declared light setting (2 warps x 10 iterations per scale)."""
    if oracle:
        from oracle import ftoracle as O
        cls = O.FlowParams
    else:
        from paper_1910_06017_b200.optflow import FlowParams as cls
    if flow == "default":
        return cls(pyramid_scales=SCALES)
    return cls(warps_per_level=2, iterations_per_warp=10, pyramid_scales=SCALES)


FRAME_BYTES = {"default": 22.03e9, "light": 2.52e9}  # SURVEY 8(d) algorithmic bytes / SD frame


def _cpu_frame_job(args):
    rank, s, flow, config = args
    apply_config(config)  # spawned child: module globals start at the headline config
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import ftoracle as O
    from paper_1910_06017_b200.synth import make_sequence
    frames, dets = make_sequence(W_, H_, N_OBJ, 2, seed=stream_seed(rank, s), det_every=1,
                                 scale_change=True)
    st = O.StreamState()
    d0 = [O.Det(d.class_id, d.label, d.score, d.box) for d in dets[0]]
    prm = _flow_params(flow, oracle=True)
    O.step(st, frames[0], 0, d0, prm)  # first frame: ST + spawn (not timed)
    d1 = [O.Det(d.class_id, d.label, d.score, d.box) for d in dets[1]]
    t0 = time.perf_counter()
    O.step(st, frames[1], 1, d1, prm)  # a full tracked frame: ST + flow + predict + match + update
    return time.perf_counter() - t0


def cpu_run(n_procs: int, jobs: int, flow: str = "default", config: str = "c2"):
    for var in ("OMP_NUM_THREADS", "MKL_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        os.environ[var] = "1"  # one core per process (children inherit)
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(n_procs) as pool:
        per = pool.map(_cpu_frame_job, [(99, s, flow, config) for s in range(jobs)])
    return time.perf_counter() - t0, per


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_baseline_measure(flow: str = "default", config: str = "c2"):
    cores = host_cores()
    wall, per = cpu_run(cores, cores, flow, config)
    # each process measured its own tracked frame; aggregate = cores / mean
    per_core_fps = 1.0 / float(np.mean(per))
    return {"value": round(per_core_fps * cores, 5), "unit": "frames/s", "cores": cores,
            "kind": "port", "per_core_fps": round(per_core_fps, 5),
            "sample": f"{cores} processes x 1 tracked frame ({config} workload, {N_OBJ} tracks, {flow} "
                      f"FlowParams) through oracle/ftoracle.py (numpy restatement of the "
                      f"reference, bit-exact); wall {wall:.1f}s"}


def run_reference(args, ws, rank):
    if rank != 0:
        return
    cores = host_cores()
    # One step: every host core tracks one frame of its own stream.  Each
    # process first runs an untimed warm-up frame (imports, ST, spawn), then
    # times one full tracked frame; a step lasts as long as its slowest
    # process (process start-up is not reference work and is not counted).
    step_times, walls = [], []
    for k in range(args.steps):
        wall, per = cpu_run(cores, cores, args.flow, args.config)
        step_times.append(float(np.max(per)))
        walls.append(wall)
        if sum(walls) > args.ref_budget_s:
            break
    steps = len(step_times)
    wall = float(np.sum(step_times))
    fps = cores * steps / wall
    line = {"impl": "reference", "metric": METRIC, "value": round(fps, 5), "unit": "frames/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": 1,
            "ms_per_step": round(1000 * wall / steps, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload(args), "streams": cores,
                       "note": "one step = every host core tracks one frame of its own stream "
                               "(after one untimed warm-up frame per process); step time = the "
                               "slowest process; steps capped by a "
                               f"{args.ref_budget_s:.0f}s budget"},
            "cpu_baseline": {"value": round(fps, 5), "unit": "frames/s", "cores": cores,
                             "kind": "port",
                             "sample": "oracle/ftoracle.py (numpy restatement of flowtrack, "
                                       "bit-exact), one process per core"},
            "e2e": {"value": round(fps, 5), "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
def run_ours(args, ws, rank, local):
    import torch

    from paper_1910_06017_b200 import _lib
    from paper_1910_06017_b200.optflow import FlowParams
    from paper_1910_06017_b200.pipeline import Tracker

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    B, K, Wm = args.streams, args.steps, args.warmup
    T = Wm + K + 1
    max_tracks, max_dets = max(256, 2 * N_OBJ + 56), max(160, N_OBJ + 60)
    seqs = gen_streams(rank, B, T)
    frames = np.stack([np.stack([seqs[s][0][t] for s in range(B)]) for t in range(T)])  # T,B,H,W
    dets = np.zeros((T, B, max_dets), dtype=_lib.DET_DTYPE)
    ndets = np.zeros((T, B), dtype=np.int32)
    for t in range(T):
        for s in range(B):
            dets[t, s], ndets[t, s] = det_records(seqs[s][1][t], max_dets)

    prm = _flow_params(args.flow)
    trk = Tracker(W_, H_, n_streams=B, flow_params=prm, max_tracks=max_tracks, max_dets=max_dets,
                  device=local, motion=args.motion, klt_grid=10)
    stream = torch.cuda.current_stream(dev)

    # ---------------- device-resident timing (value) ----------------
    d_frames = torch.from_numpy(frames).to(dev)
    d_dets = torch.from_numpy(dets.view(np.uint8)).to(dev)
    d_ndets = torch.from_numpy(ndets).to(dev)
    for t in range(Wm + 1):  # frame 0 bootstraps; W full warm-up steps
        trk.step_device(d_frames[t], t, d_dets[t], d_ndets[t])
    torch.cuda.synchronize(dev)
    barrier(ws)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for t in range(Wm + 1, T):
            trk.step_device(d_frames[t], t, d_dets[t], d_ndets[t])
        e1.record(stream)
        torch.cuda.synchronize(dev)
    barrier(ws)
    ms = e0.elapsed_time(e1)
    ms_max = allmax(ws, ms)
    launches_per_step = trk.launches()
    value = ws * B * K / (ms_max / 1000.0)

    # ---------------- dominant kernel, timed live in the last timed step ------
    # (CUDA events captured into the step graph around every finest-level
    # k_pd_tile launch sequence; read after the timed region ends)
    span_ms, span_n, span_pi = C_double(), C_int(), C_double()
    msl, bpl, ipl = C_double(), C_double(), C_int()
    if args.motion == "tvl1":
        _lib.check(trk._lib.ft_tracker_pd_span(trk._h, byref(span_ms), byref(span_n),
                                               byref(span_pi)))
        # the same kernel timed alone (repeated launches over the final state)
        _lib.check(trk._lib.ft_tracker_profile_pd(trk._h, 20, byref(msl), byref(bpl),
                                                  byref(ipl)))
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    # 152 algorithmic bytes per pixel-iteration (read 11 planes,
    # write 8) x the pixel-iterations of the step's finest-level launches
    live_bytes = 152.0 * span_pi.value
    live_launch_ms = span_ms.value / span_n.value if span_n.value else 0.0
    achieved = live_bytes / (span_ms.value / 1000.0) / 1e9 if span_ms.value > 0 else 0.0
    alone_gbs = bpl.value / (msl.value / 1000.0) / 1e9 if msl.value > 0 else 0.0
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "pd_traffic.json")
    if os.path.exists(tfile):
        tj = json.load(open(tfile))
        # ncu capture of one finest-level launch, normalised per stream-pixel
        # and rescaled to this run's streams (same kernel, same geometry)
        if tj.get("bytes_per_stream_pixel"):
            from paper_1910_06017_b200.imaging import select_level
            lv = select_level(W_, H_)  # the flow runs at the processing level
            traffic = round(tj["bytes_per_stream_pixel"] * B * (W_ >> lv) * (H_ >> lv), 1)
    # step-level roofline: SURVEY 8(d) algorithmic bytes per SD frame (22.03 GB at C2)
    frame_bytes = FRAME_BYTES[args.flow]
    step_frac = (value / ws) * frame_bytes / (hbm * 1e9)

    # ---------------- end to end through the public API (e2e) ----------------
    trk.reset()
    recs = [[dets[t, s][:max(ndets[t, s], 0)] if ndets[t, s] >= 0 else None for s in range(B)]
            for t in range(T)]
    for t in range(Wm + 1):
        trk.step_records(frames[t], t, recs[t])
    torch.cuda.synchronize(dev)
    barrier(ws)
    t0 = time.perf_counter()
    n_tracks = 0
    # pipelined public API: stage + submit frame t, then collect frame t-1
    # (each step still does its own pinned H2D and D2H inside the region)
    for t in range(Wm + 1, T):
        trk.submit(frames[t], t, recs[t])
        if t > Wm + 1:
            n_tracks += sum(len(o) for o in trk.wait())
    n_tracks += sum(len(o) for o in trk.wait())
    torch.cuda.synchronize(dev)
    e2e_s = allmax(ws, time.perf_counter() - t0)
    barrier(ws)
    e2e = ws * B * K / e2e_s
    h2d = B * H_ * W_ + B * max_dets * _lib.DET_DTYPE.itemsize + (B + 1) * 4
    d2h = B * 2 * max_tracks * _lib.TRACK_DTYPE.itemsize + 2 * B * 4
    trk.close()

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_measure(args.flow, args.config)

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 3), "unit": "frames/s", "n_gpus": ws,
                "steps": K, "warmup": Wm, "ms_per_step": round(ms_max / K, 4),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic",
                "config": {"workload": workload(args), "streams_per_gpu": B, "frame": [W_, H_],
                           "tracks_per_stream": N_OBJ, "parallelism": f"stream-sharded x{ws}",
                           "l2": "working set > L2: every launch streams its state planes "
                                 f"({B} streams x ~70 MB)"},
                "e2e": {"value": round(e2e, 3), "unit": "frames/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "api": "Tracker.submit/wait (pipelined)"},
                "gpu_launches": int(launches_per_step * K),
                "roofline": {"bound": "hbm", "kernel": "k_pd_tile (TV-L1 primal-dual, finest level)",
                             "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                             "frac": round(achieved / hbm, 4), "traffic": traffic,
                             "timing": "live: CUDA events in the step graph around the "
                                       "finest-level k_pd_tile launches of the last timed step",
                             "launches": span_n.value,
                             "bytes_per_launch": live_bytes / max(span_n.value, 1),
                             "ms_per_launch": round(live_launch_ms, 5),
                             "share_of_step": round(span_ms.value / (ms / K), 4) if ms else None,
                             "compulsory_bytes_per_launch": bpl.value / max(ipl.value, 1),
                             "alone": {"ms_per_launch": round(msl.value, 5),
                                       "iters_per_launch": ipl.value,
                                       "achieved": round(alone_gbs, 1)},
                             "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback 6650",
                             "step_roofline_frac": round(step_frac, 4),
                             "step_bytes_per_frame": frame_bytes},
                "cpu_baseline": cpu, "clocks": clk.summary(),
                "tracks_out": int(n_tracks)}
        if args.motion == "klt":  # SURVEY 8 f4 backend: not the reference path
            line["config"]["workload"] = (
                "C2 with the KLT/MedianFlow backend (SURVEY 8 f4): 720x576 SD, 100 tracks, "
                "10x10 points/box, 3-level LK pyramid, 9x9 window, forward-backward check, fp64")
            line["config"]["l2"] = (f"working set > L2: {B} streams x ~26 MB of KLT pyramids "
                                     "(prev + cur) per step")
            line["roofline"] = None  # gather-latency bound; no streaming-roofline model
            line["step_roofline_frac"] = None
        print(json.dumps(line), flush=True)


from ctypes import byref, c_double as C_double, c_int as C_int  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--streams", type=int, default=64,
                    help="SD streams per GPU (64 = BASELINE config C5's stream count at N=1)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--motion", choices=["tvl1", "klt"], default="tvl1",
                    help="tvl1: the reference path (headline); klt: SURVEY 8 f4 backend")
    ap.add_argument("--flow", choices=["default", "light"], default="default",
                    help="default FlowParams (headline) or SURVEY 8(d)'s light 2 warps x 10 iters")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-budget-s", type=float, default=150.0)
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2",
                    help="c2 (headline) or another BASELINE.json config as a non-headline line")
    args = ap.parse_args()
    apply_config(args.config)
    ws, rank, local = dist_init()
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

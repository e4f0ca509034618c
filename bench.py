#!/usr/bin/env python
"""Benchmark: tracked SD frames/s (BASELINE.json metric) on config C2 --
720x576, 100 tracks with scale change and occlusion, detections every 5th
frame, default FlowParams (6 scales x 5 warps x 50 iterations), fp64 -- with
the streams batched and sharded as in C5.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--streams B | --total-streams T]
    python bench.py --impl reference ...     (CPU reference arm)

One step = one frame of each of the B streams resident on a GPU.  Ranks
own disjoint blocks of global stream ids (paper_1910_06017_b200/shard.py);
no collective touches the data path -- only the timing barrier, the max of
the ranks' times and the final host gather of track records.  `--gpus N`
without a torchrun environment launches the N ranks itself (and fails if
the box has fewer GPUs).

`value` = frames processed by ALL ranks / the slowest rank's device time
(whole-job aggregate, the driver's contract); `value_per_gpu` = value / N,
the per-GPU figure the metric's wording names.  Device time: CUDA events on
the tracker stream, inputs already in HBM.  `e2e` goes through the public
Tracker API with host frames in pinned memory, H2D of frames + detections
and D2H of the track table inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1910_06017_b200 import shard  # noqa: E402

METRIC = "tracked frames/sec per GPU at 720×576, 100 tracks; HBM-roofline fraction"
W_, H_, N_OBJ, DET_EVERY, JITTER = 720, 576, 100, 5, 1.0
SCALES = None  # FlowParams.pyramid_scales (None: auto_scales, 6 at SD)
WORKLOAD = ("C2 streams batched as in C5: 720x576 SD, 100 tracks, scale change + occlusion, "
            "detections every 5th frame (1 px jitter), TV-L1 6 scales x 5 warps x 50 iterations, "
            "ROF 40 iterations, fp64")
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
FRAME_BYTES = {"default": 22.03e9, "light": 2.52e9}  # SURVEY 8(d) algorithmic bytes / SD frame


def apply_config(name: str) -> None:
    global W_, H_, N_OBJ, DET_EVERY, SCALES, WORKLOAD, METRIC
    c = CONFIGS.get(name)
    if c is None:
        return
    W_, H_, N_OBJ, DET_EVERY, SCALES, fb, WORKLOAD = c
    FRAME_BYTES["default"] = fb
    METRIC = f"tracked frames/sec per GPU at {W_}×{H_}, {N_OBJ} tracks; HBM-roofline fraction"


# ---------------------------------------------------------------------------
stream_seed = shard.stream_seed
dist_init = shard.init
barrier = shard.barrier
allmax = shard.allmax


def gen_stream(g: int, n_frames: int):
    from paper_1910_06017_b200.synth import make_sequence
    return make_sequence(W_, H_, N_OBJ, n_frames, seed=stream_seed(g), det_every=DET_EVERY,
                         scale_change=True, jitter=JITTER)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self.proc = gpu, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
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
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
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
    w = WORKLOAD
    if args.flow == "light":
        w = w.replace("6 scales x 5 warps x 50 iterations",
                      "6 scales x 2 warps x 10 iterations (SURVEY 8(d) light FlowParams)")
    if args.motion == "klt":
        w = (f"C2 with the KLT/MedianFlow backend (SURVEY 8 f4): {W_}x{H_}, {N_OBJ} tracks, "
             "10x10 points/box, 3-level LK pyramid, 9x9 window, forward-backward check, fp64")
    return w


def bench_config(args, ws: int, streams_per_gpu: int) -> dict:
    """The `config` object, identical on both arms (same workload keys).
    Strong scaling (--total-streams T): streams_per_gpu = the largest rank
    block, ceil(T / ws)."""
    if args.total_streams is not None:
        total = args.total_streams
        streams_per_gpu = -(-total // ws)
    else:
        total = streams_per_gpu * ws
    return {"workload": workload(args), "frame": [W_, H_], "tracks_per_stream": N_OBJ,
            "detect_every": DET_EVERY, "det_jitter_px": JITTER,
            "streams_per_gpu": streams_per_gpu, "total_streams": total,
            "stream_seeds": "1000 + global stream id",
            "parallelism": f"stream-sharded x{ws} (no data-path collective)",
            "l2": "working set > L2: 64 SD streams x ~100 MB of state per GPU; every launch "
                  "streams its planes from HBM (no L2 flush needed)"}


# ---------------------------------------------------------------------------
# CPU side: the oracle port of the reference.  One job = one stream's frame 1
# of the GPU arm's own sequence (same seed scheme, cadence and jitter): frame
# 0 bootstraps untimed, frame 1 (ST + flow + predict; a coasting frame at
# cadence 5) is timed.  Match + update on detection frames add < 0.1 % on
# the CPU (SURVEY 8(a) A13-A15 vs A4/A6).
def _flow_params(flow: str, oracle: bool = False):
    if oracle:
        from oracle import ftoracle as O
        cls = O.FlowParams
    else:
        from paper_1910_06017_b200.optflow import FlowParams as cls
    if flow == "default":
        return cls(pyramid_scales=SCALES)
    return cls(warps_per_level=2, iterations_per_warp=10, pyramid_scales=SCALES)


def _cpu_frame_job(args):
    g, flow, config, motion = args
    apply_config(config)  # spawned child: module globals start at the headline config
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from oracle import ftoracle as O
    frames, dets = gen_stream(g, 2)
    st = O.StreamState()
    od = [None if d is None else [O.Det(x.class_id, x.label, x.score, x.box) for x in d]
          for d in dets]
    if motion == "klt":
        from oracle import klt_oracle as K
        K.step_klt(st, frames[0], 0, od[0])
        t0 = time.perf_counter()
        K.step_klt(st, frames[1], 1, od[1])
        return time.perf_counter() - t0
    prm = _flow_params(flow, oracle=True)
    O.step(st, frames[0], 0, od[0], prm)  # first frame: ST + spawn (not timed)
    t0 = time.perf_counter()
    O.step(st, frames[1], 1, od[1], prm)  # a tracked frame: ST + flow + predict (+ match/update)
    return time.perf_counter() - t0


def _cv2_frame_job(g: int) -> float:
    """The KLT backend's practical CPU comparison (informative, not the
    oracle: OpenCV's fp32 pyramidal LK is not bit-identical): frame 1 of
    stream g -- the frame-0 detection boxes' 10x10 point grids tracked
    forward and back with cv2.calcOpticalFlowPyrLK (9x9 window, 3 levels,
    10 iterations, eps 0.01 px) on one core."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import cv2
    cv2.setNumThreads(1)
    frames, dets = gen_stream(g, 2)
    pts = []
    for d in dets[0] or []:
        x, y, w, h = d.box
        for j in range(10):
            for i in range(10):
                pts.append((x + (i + 0.5) * w / 10, y + (j + 0.5) * h / 10))
    p0 = np.asarray(pts, dtype=np.float32).reshape(-1, 1, 2)
    a, b = np.ascontiguousarray(frames[0]), np.ascontiguousarray(frames[1])
    crit = (cv2.TERM_CRITERIA_COUNT | cv2.TERM_CRITERIA_EPS, 10, 0.01)
    t0 = time.perf_counter()
    p1, _, _ = cv2.calcOpticalFlowPyrLK(a, b, p0, None, winSize=(9, 9), maxLevel=2, criteria=crit)
    cv2.calcOpticalFlowPyrLK(b, a, p1, None, winSize=(9, 9), maxLevel=2, criteria=crit)
    return time.perf_counter() - t0


def cpu_opencv_measure() -> dict:
    cores = host_cores()
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        per = pool.map(_cv2_frame_job, list(range(cores)))
    wall = time.perf_counter() - t0
    fps = cores / float(np.mean(per))
    return {"value": round(fps, 3), "unit": "frames/s", "cores": cores,
            "sample": f"{cores} processes, frame 1 of streams 0..{cores - 1}: "
                      f"cv2.calcOpticalFlowPyrLK forward + backward on the {N_OBJ} boxes' 10x10 "
                      "grids (fp32, not bit-identical to the KLT oracle; informative)",
            "wall_s": round(wall, 1)}


def cpu_run(n_procs: int, jobs: int, flow: str, config: str, motion: str):
    for var in ("OMP_NUM_THREADS", "MKL_NUM_THREADS", "OPENBLAS_NUM_THREADS"):
        os.environ[var] = "1"  # one core per process (children inherit)
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(n_procs) as pool:
        per = pool.map(_cpu_frame_job, [(s, flow, config, motion) for s in range(jobs)])
    return time.perf_counter() - t0, per


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _cpu_sample(cores, config, motion, flow) -> str:
    impl = ("oracle/klt_oracle.py step_klt (the KLT backend's CPU definition)" if motion == "klt"
            else "oracle/ftoracle.py step (numpy restatement of flowtrack, bit-exact)")
    return (f"{cores} processes (one per host core), each tracking frame 1 of its own stream "
            f"(global ids 0..{cores - 1}, the GPU arm's seeds, cadence and jitter; {config}, "
            f"{N_OBJ} tracks, {flow} FlowParams) through {impl}; frame 0 untimed")


def cpu_baseline_measure(flow: str, config: str, motion: str):
    cores = host_cores()
    wall, per = cpu_run(cores, cores, flow, config, motion)
    per_core_fps = 1.0 / float(np.mean(per))
    return {"value": round(per_core_fps * cores, 5), "unit": "frames/s", "cores": cores,
            "kind": "port", "per_core_fps": round(per_core_fps, 5),
            "sample": _cpu_sample(cores, config, motion, flow) + f"; wall {wall:.1f}s"}


def run_reference(args, ws, rank):
    if rank != 0:
        return
    cores = host_cores()
    # One step: every host core tracks one frame of its own stream.  A step
    # lasts as long as its slowest process (process start-up and the untimed
    # bootstrap frame are not reference work and are not counted).
    step_times = []
    spent = 0.0
    for _ in range(args.steps):
        wall, per = cpu_run(cores, cores, args.flow, args.config, args.motion)
        step_times.append(float(np.max(per)))
        spent += wall
        if spent > args.ref_budget_s:
            break
    steps = len(step_times)
    wall = float(np.sum(step_times))
    fps = cores * steps / wall
    line = {"impl": "reference", "metric": METRIC, "value": round(fps, 5), "unit": "frames/s",
            "n_gpus": args.gpus, "steps": steps, "warmup": 1,
            "ms_per_step": round(1000 * wall / steps, 3), "higher_is_better": True,
            "scaling": "weak" if args.total_streams is None else "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": bench_config(args, ws, args.streams),
            "cpu_baseline": {"value": round(fps, 5), "unit": "frames/s", "cores": cores,
                             "kind": "port",
                             "sample": _cpu_sample(cores, args.config, args.motion, args.flow)
                             + f"; step = slowest process; {steps} steps within a "
                               f"{args.ref_budget_s:.0f}s budget"},
            "e2e": {"value": round(fps, 5), "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
def _pct(v, q):
    return round(float(np.percentile(v, q)), 4) if len(v) else None


def run_ours(args, ws, rank, local):
    import torch

    from paper_1910_06017_b200 import _lib
    from paper_1910_06017_b200.pipeline import Tracker

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if args.total_streams is not None:
        ids = shard.shard(rank, ws, total=args.total_streams)
        scaling = "strong"
    else:
        ids = shard.shard(rank, ws, per_rank=args.streams)
        scaling = "weak"
    B, K, Wm = len(ids), args.steps, args.warmup
    T = Wm + K + 1
    max_tracks, max_dets = max(256, 2 * N_OBJ + 56), max(160, N_OBJ + 60)
    seqs = [gen_stream(g, T) for g in ids]
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
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        ev[0].record(stream)
        for k, t in enumerate(range(Wm + 1, T)):
            trk.step_device(d_frames[t], t, d_dets[t], d_ndets[t])
            ev[k + 1].record(stream)
        torch.cuda.synchronize(dev)
    barrier(ws)
    ms = ev[0].elapsed_time(ev[K])
    step_ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(K)]
    ms_max = allmax(ws, ms)
    launches_per_step = trk.launches()
    value = ws * B * K / (ms_max / 1000.0) if args.total_streams is None else \
        args.total_streams * K / (ms_max / 1000.0)
    phases = trk.phase_ms()

    # ---------------- dominant kernel, timed live in the last timed step ------
    roofline = None
    if args.motion == "tvl1":
        roofline = trk.roofline(hbm_peak_gbs(), frame_bytes=FRAME_BYTES[args.flow],
                                step_ms=ms / K, frames_per_s_per_gpu=value / ws,
                                profiles_dir=os.path.join(ROOT, "profiles"))
        if roofline is not None and phases.get("structure_texture"):
            roofline["rof"] = rof_roofline(phases["structure_texture"], B)
    elif phases.get("klt track"):
        roofline = klt_roofline(phases["klt track"], B)

    # ---------------- end to end through the public API (e2e) ----------------
    recs = [[dets[t, s][:max(ndets[t, s], 0)] if ndets[t, s] >= 0 else None for s in range(B)]
            for t in range(T)]

    def e2e_pass():
        trk.reset()
        for t in range(Wm + 1):
            trk.step_records(frames[t], t, recs[t])
        torch.cuda.synchronize(dev)
        barrier(ws)
        t0 = time.perf_counter()
        last = None
        # pipelined public API: stage + submit frame t, then collect frame t-1
        # (each step still does its own pinned H2D and D2H inside the region)
        for t in range(Wm + 1, T):
            trk.submit(frames[t], t, recs[t])
            if t > Wm + 1:
                last = trk.wait()
        last = trk.wait()
        torch.cuda.synchronize(dev)
        return time.perf_counter() - t0, last

    # an untimed pass first: the step graphs of the pipelined slots are
    # captured there, not inside the timed region
    e2e_pass()
    e2e_s, last = e2e_pass()
    e2e_s = allmax(ws, e2e_s)
    barrier(ws)
    total_frames = ws * B * K if args.total_streams is None else args.total_streams * K
    e2e = total_frames / e2e_s
    h2d = B * H_ * W_ + B * max_dets * _lib.DET_DTYPE.itemsize + (2 * B + 1) * 4
    d2h = B * 2 * max_tracks * _lib.TRACK_DTYPE.itemsize + 2 * B * 4

    # ---------------- single-stream latency (the paper's real-time setting) ----
    latency = None
    if B == 1:
        lat = []
        trk.reset()
        for t in range(T):
            t1 = time.perf_counter()
            trk.step_records(frames[t], t, recs[t])
            if t > Wm:
                lat.append(1000 * (time.perf_counter() - t1))
        latency = {"device_ms_p50": _pct(step_ms, 50), "device_ms_p99": _pct(step_ms, 99),
                   "e2e_ms_p50": _pct(lat, 50), "e2e_ms_p99": _pct(lat, 99),
                   "e2e_api": "Tracker.step_records (synchronous: submit + wait per frame)"}
        # the paper's prefetch: preprocessing of frame t+1
        # overlaps flow/predict/match/update of frame t on the device
        pf = Tracker(W_, H_, n_streams=B, flow_params=prm, max_tracks=max_tracks,
                     max_dets=max_dets, device=local, prefetch=True)
        # one untimed pass captures every step graph the rotation uses (new
        # frame / pending frame / three pyramid buffers / input parity: six
        # in the steady state), then the timed pass replays them
        for t in range(T):
            pf.submit(frames[t], t, recs[t])
            if t:
                pf.wait()
        pf.wait()
        pf.reset()
        for t in range(Wm + 1):
            pf.submit(frames[t], t, recs[t])
            pf.wait()
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        for t in range(Wm + 1, T):
            pf.submit(frames[t], t, recs[t])
            if t > Wm + 1:
                pf.wait()
        pf.wait()
        period = 1000 * (time.perf_counter() - t1) / K
        pf.close()
        latency["prefetch_frame_period_ms"] = round(period, 4)
        latency["prefetch_api"] = ("Tracker(prefetch=True).submit/wait, two steps in flight: "
                                   "frame period (records lag one frame)")

    # ---------------- final host gather of the track results (north_star) ----
    gathered = shard.gather_tracks(ws, rank, ids, last)
    trk.close()

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_measure(args.flow, args.config, args.motion)

    if rank == 0:
        n_tracks = sum(len(r) for r in gathered.values())
        line = {"metric": METRIC, "value": round(value, 3), "unit": "frames/s", "n_gpus": ws,
                "value_per_gpu": round(value / ws, 3),
                "steps": K, "warmup": Wm, "ms_per_step": round(ms_max / K, 4),
                "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (SURVEY 8(d) generator: textured moving boxes, YoloV3-style "
                        "detections in receptive-field coordinates)",
                "config": bench_config(args, ws, B),
                "e2e": {"value": round(e2e, 3), "unit": "frames/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "api": "Tracker.submit/wait (pipelined)"},
                "gpu_launches": int(launches_per_step * K),
                "step_ms": {"p50": _pct(step_ms, 50), "p99": _pct(step_ms, 99)},
                "phases_ms": phases,
                "roofline": roofline,
                "cpu_baseline": cpu, "clocks": clk.summary(),
                "gather": {"streams": len(gathered), "tracks": int(n_tracks),
                           "note": "last frame's track records of every stream gathered to rank "
                                   "0 on the host (torch.distributed gather_object)"}}
        if latency:
            line["latency"] = latency
        if cpu is not None and args.motion == "klt":
            line["cpu_opencv"] = cpu_opencv_measure()
        if cpu is None and ws > 1:
            line["cpu_baseline_note"] = "timed at N=1 only (same host, same workload)"
        print(json.dumps(line), flush=True)


def rof_roofline(st_ms: float, streams: int) -> dict:
    """ROF structure-texture phase (imaging.py:109-144, 40 dual steps) of the
    last timed step, live from its graph event nodes: SURVEY 8(d)'s 40 B per
    pixel-iteration (read I, px, py; write px, py) and the reference's fp64
    work per pixel-iteration (imaging.py:120-124: divergence 3, d 1,
    gradient 2, hypot 1, norm 2, p update 4 incl. two divisions = 13 ops)
    against the measured peaks; the phase also holds the final combine."""
    from paper_1910_06017_b200.imaging import select_level
    lv = select_level(W_, H_)
    px = (W_ >> lv) * (H_ >> lv) * streams * 40
    sec = st_ms / 1000.0
    hbm, _ = hbm_peak_gbs()
    fp = os.path.join(ROOT, "profiles", "fp64_peak.json")
    fp64 = json.load(open(fp))["dadd_dmul_ops_per_s"] if os.path.exists(fp) else None
    return {"kernel": "k_rof_tile (+ k_st_combine), the structure_texture phase",
            "ms_per_step": round(st_ms, 4), "pixel_iters": px,
            "frac": round(40.0 * px / sec / 1e9 / hbm, 4),
            "fp64_frac": round(13.0 * px / sec / fp64, 4) if fp64 else None,
            "bound": "fp64 issue (ncu: profiles/r02_rof_full.md)"}


def klt_roofline(track_ms: float, streams: int) -> dict:
    """KLT point tracking phase (k_klt_points + k_klt_boxes) of the last
    timed step, live from its graph event nodes, against the HBM peak:
    compulsory bytes = both frames' 3-level KLT pyramids with their
    gradients (I, gx, gy: 3 fp64 planes x 1.3125 P pixels each) plus the
    per-point outputs (grid point, forward position, FB error: 40 B).  The
    windows are re-read from L1 (81 bilinear samples x 4 taps per window),
    so the kernel is gather-latency bound, not HBM bound."""
    from paper_1910_06017_b200.imaging import select_level
    lv = select_level(W_, H_)
    P = (W_ >> lv) * (H_ >> lv)
    nbytes = streams * (2 * 3 * 8 * 1.3125 * P + N_OBJ * 100 * 40)
    hbm, src = hbm_peak_gbs()
    ach = nbytes / (track_ms / 1000.0) / 1e9
    return {"bound": "hbm", "kernel": "k_klt_points + k_klt_boxes (the klt track phase)",
            "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s", "frac": round(ach / hbm, 4),
            "traffic": None, "ms_per_step": round(track_ms, 4),
            "compulsory_bytes_per_step": int(nbytes), "peak_source": src,
            "binding": "L1 gathers and issue latency (ncu, profiles/r01_klt_full.md: DRAM 1.6 %, "
                       "L1 hit 95 %, fp64 pipe 37 %, issue slots 64 %)"}


def hbm_peak_gbs():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p)).get("hbm_gbs", 6650.0)), "MEASURED_PEAKS.json hbm_gbs"
    return 6650.0, "fallback 6650 (B200_PROFILING.md)"


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


# test hook (tests/test_multiproc.py): every rank on cuda:0 over gloo, to run
# the multi-rank bench path functionally on a one-GPU box.  The ranks share
# no data and never wait on each other's kernels; the numbers are not a
# scaling measurement.
ONE_GPU = os.environ.get("FT_BENCH_ONE_GPU") == "1"


def launch_ranks(args) -> int:
    """`--gpus N` outside torchrun: start the N ranks ourselves."""
    if args.impl == "ours" and not ONE_GPU:
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this box has {have}",
                  file=sys.stderr)
            return 1
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--streams", type=int, default=64,
                    help="SD streams per GPU (weak scaling; 64 = C5's stream count at N=1)")
    ap.add_argument("--total-streams", type=int, default=None,
                    help="split this many streams over the GPUs (strong scaling, C5: 64)")
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
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None and args.gpus > 1:
        sys.exit(launch_ranks(args))
    if ws_env is not None and int(ws_env) != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":  # the CPU arm needs no GPU communicator
        os.environ.setdefault("FT_DIST_BACKEND", "gloo")
    ws, rank, local = dist_init()
    if ONE_GPU:
        local = 0
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Generate golden fixtures by running the LIVE reference (flowtrack) in this
container.  Run from the repo root:

    python tests/golden/make_golden.py

Needs /root/reference (read-only); the outputs (tests/golden/*.npz, *.json)
are committed so the GPU box, which has no /root/reference, can check
against them.  numpy's version is recorded in every file because the
reference pins only numpy>=1.24 (pyproject.toml:10) and box means depend on
numpy's summation order.
"""

from __future__ import annotations

import json
import os
import sys
from dataclasses import replace

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, ROOT)

from flowtrack import assoc, detect, imaging, optflow, track  # noqa: E402
from flowtrack.imageops import round_half_away  # noqa: E402,F401

from paper_1910_06017_b200.synth import make_sequence  # noqa: E402

META = {"numpy": np.__version__, "generator": "tests/golden/make_golden.py"}


def save(name, **arrays):
    np.savez_compressed(os.path.join(HERE, name), **arrays,
                        _meta=np.array(json.dumps(META)))


def frame_of(u8, idx=0):
    return imaging.Frame.from_gray8(u8, index=idx)


def gen_imaging():
    rng = np.random.default_rng(11)
    out = {}
    for k, (w, h, lv) in enumerate([(37, 29, 3), (64, 48, 4), (80, 61, 2), (5, 4, 2)]):
        u8 = rng.integers(0, 256, (h, w), dtype=np.uint8)
        out[f"pyr{k}_in"] = u8
        pyr = imaging.build_pyramid(frame_of(u8), lv)
        for j, f in enumerate(pyr.levels):
            out[f"pyr{k}_l{j}"] = f.data
    for k, (w, h, wt, bl, it) in enumerate([(45, 33, 12.0, 0.05, 40), (64, 48, 12.0, 0.05, 40),
                                             (30, 20, 5.0, 0.3, 7), (30, 20, 12.0, 1.0, 0)]):
        u8 = rng.integers(0, 256, (h, w), dtype=np.uint8)
        out[f"st{k}_in"] = u8
        out[f"st{k}_prm"] = np.array([wt, bl, it])
        out[f"st{k}_out"] = imaging.structure_texture(frame_of(u8), wt, bl, it).data
    save("imaging.npz", **out)


FLOW_CASES = [
    # (w, h, scales, warps, iters, shift, seed)
    (48, 40, None, 5, 50, (1, 0), 1),
    (96, 72, None, 5, 50, (2, -1), 2),
    (61, 47, 2, 2, 10, (0, 1), 3),
    (40, 32, 3, 3, 7, (0, 0), 4),
    (130, 100, None, 2, 10, (3, 2), 5),
]


def gen_flow():
    out = {}
    for k, (w, h, sc, wp, it, sh, seed) in enumerate(FLOW_CASES):
        frames, _ = make_sequence(w + 16, h + 16, 3, 2, seed=seed)
        a = frames[0][8:8 + h, 8:8 + w]
        b = np.roll(frames[0], sh, axis=(1, 0))[8:8 + h, 8:8 + w]
        if k == 3:
            b = a.copy()
        if k == 4:
            a = frames[0][8:8 + h, 8:8 + w]
            b = frames[1][8:8 + h, 8:8 + w]
        pa = imaging.structure_texture(frame_of(a, 0))
        pb = imaging.structure_texture(frame_of(b, 1))
        prm = optflow.FlowParams(warps_per_level=wp, iterations_per_warp=it,
                                 pyramid_scales=sc)
        fld = optflow.compute_flow(pa, pb, prm)
        out[f"f{k}_a"] = a
        out[f"f{k}_b"] = b
        out[f"f{k}_prm"] = np.array([w, h, -1 if sc is None else sc, wp, it])
        out[f"f{k}_sta"] = pa.data
        out[f"f{k}_stb"] = pb.data
        out[f"f{k}_dx"] = fld.dx
        out[f"f{k}_dy"] = fld.dy
    save("flow.npz", **out)


def predict_field(k, lw, lh):
    """Seeded random field; tests regenerate it instead of storing 3 MB."""
    frng = np.random.default_rng(100 + k)
    return frng.standard_normal((lh, lw)) * 3, frng.standard_normal((lh, lw)) * 3


def gen_predict():
    rng = np.random.default_rng(21)
    out = {}
    cases = []
    for k, (fw, fh, lvl) in enumerate([(160, 120, 0), (321, 239, 1), (640, 360, 2), (720, 576, 0)]):
        lw, lh = fw, fh
        for _ in range(lvl):
            lw //= 2
            lh //= 2
        dx, dy = predict_field(k, lw, lh)
        n = 60
        boxes = []
        for _ in range(n):
            w = float(rng.uniform(0.5, fw * 0.8))
            h = float(rng.uniform(0.5, fh * 0.8))
            x = float(rng.uniform(-w * 0.9, fw))
            y = float(rng.uniform(-h * 0.9, fh))
            boxes.append((x, y, w, h))
        # explicit edge cases: half-pixel edges, full-width box, zero support
        boxes += [(0.5 * (2 ** lvl), 1.5 * (2 ** lvl), 3.0 * (2 ** lvl), 2.0),
                  (0.0, 0.0, float(fw), 5.0 * (2 ** lvl)),
                  (float(fw) - 0.2, 3.0, 0.1, 4.0),
                  (2.0, 2.0, 0.2 * (2 ** lvl), 0.2 * (2 ** lvl))]
        objs = [track.SceneObject(id=i, class_id=0, label="x", box=b) for i, b in enumerate(boxes)]
        fld = optflow.MotionField(width=lw, height=lh, dx=dx, dy=dy)
        pred = track.predict(objs, fld, lvl, (fw, fh))
        res = np.array([p if p is not None else (np.nan,) * 4 for p in pred])
        out[f"p{k}_boxes"] = np.array(boxes)
        out[f"p{k}_meta"] = np.array([fw, fh, lvl])
        out[f"p{k}_out"] = res
        cases.append(k)
    # SPEC.md:347-348 examples
    fld = optflow.MotionField(width=64, height=64, dx=np.full((64, 64), 3.0), dy=np.full((64, 64), -2.0))
    out["kat_uniform"] = np.array(track.predict(
        [track.SceneObject(id=0, class_id=0, label="a", box=(10, 10, 20, 20))], fld, 0, (64, 64))[0])
    save("predict.npz", **out)


def gen_assoc():
    rng = np.random.default_rng(31)
    out = {}
    # hungarian on random / tie-heavy / forbidden matrices
    for k in range(40):
        m = int(rng.integers(1, 9))
        n = int(rng.integers(1, 9))
        kind = k % 4
        if kind == 0:
            c = rng.random((m, n))
        elif kind == 1:
            c = rng.integers(0, 3, (m, n)).astype(np.float64)
        elif kind == 2:
            c = np.where(rng.random((m, n)) < 0.6, assoc.FORBIDDEN_COST, rng.random((m, n)))
        else:
            c = np.zeros((m, n))
        pairs = assoc.hungarian(c, forbidden=assoc.FORBIDDEN_COST if kind == 2 else None)
        out[f"h{k}_cost"] = c
        out[f"h{k}_forb"] = np.array([kind == 2])
        out[f"h{k}_pairs"] = np.array(pairs, dtype=np.int64).reshape(-1, 2)
    # larger gated-sparse case like a real frame (100 x 104)
    for k in range(3):
        m, n = [(100, 104), (57, 40), (200, 190)][k]
        tb = np.column_stack([rng.uniform(0, 600, m), rng.uniform(0, 500, m),
                              rng.uniform(20, 90, m), rng.uniform(20, 90, m)])
        db = tb[rng.permutation(m)[:min(m, n)]] + rng.normal(0, 6, (min(m, n), 4))
        if n > m:
            db = np.vstack([db, np.column_stack([rng.uniform(0, 600, n - m), rng.uniform(0, 500, n - m),
                                                 rng.uniform(20, 90, n - m), rng.uniform(20, 90, n - m)])])
        db[:, 2:] = np.abs(db[:, 2:]) + 1.0
        tc = rng.integers(0, 3, m)
        dc = rng.integers(0, 3, n)
        objs = [track.SceneObject(id=i, class_id=int(tc[i]), label="t", box=tuple(tb[i])) for i in range(m)]
        dets = [detect.Detection(class_id=int(dc[j]), label="d", score=0.9, box=tuple(db[j])) for j in range(n)]
        a = assoc.match(objs, dets, 0.3)
        out[f"m{k}_tb"] = tb
        out[f"m{k}_db"] = db
        out[f"m{k}_tc"] = tc
        out[f"m{k}_dc"] = dc
        out[f"m{k}_pairs"] = np.array([(i, j) for i, j, _ in a.pairs], dtype=np.int64).reshape(-1, 2)
        out[f"m{k}_ious"] = np.array([s for _, _, s in a.pairs])
        out[f"m{k}_um_s"] = np.array(a.unmatched_scene, dtype=np.int64)
        out[f"m{k}_um_d"] = np.array(a.unmatched_detections, dtype=np.int64)
    # iou matrix for random boxes
    A = np.column_stack([rng.uniform(0, 50, 30), rng.uniform(0, 50, 30), rng.uniform(0.5, 30, 30), rng.uniform(0.5, 30, 30)])
    B = np.column_stack([rng.uniform(0, 50, 25), rng.uniform(0, 50, 25), rng.uniform(0.5, 30, 25), rng.uniform(0.5, 30, 25)])
    out["iou_a"] = A
    out["iou_b"] = B
    out["iou_ab"] = np.array([[assoc.iou(tuple(a), tuple(b)) for b in B] for a in A])
    save("assoc.npz", **out)


# ---- end-to-end step composed from the reference functions ----
def ref_step(scene, prev_st, u8, t, dets, prm, gate=0.3, min_score=0.5):
    H, W = u8.shape
    L = imaging.select_level(W, H)
    f = imaging.Frame.from_gray8(u8, index=t)
    lvl = imaging.build_pyramid(f, L + 1).levels[L]
    st = imaging.structure_texture(lvl)
    if dets is not None:
        dets = detect.filter_detections(dets, min_score)
    if prev_st is None:
        if dets is not None:
            scene = track.update([], assoc.Assignment((), (), tuple(range(len(dets)))), dets, t)
    else:
        fld = optflow.compute_flow(prev_st, st, prm)
        act = [i for i, o in enumerate(scene) if o.state == track.ACTIVE]
        pred = track.predict([scene[i] for i in act], fld, L, (W, H))
        scene = list(scene)
        for i, p in zip(act, pred):
            if p is not None:
                scene[i] = replace(scene[i], box=p)
        if dets is not None:
            cand = [i for i, p in zip(act, pred) if p is not None]
            a = assoc.match([scene[i] for i in cand], dets, gate)
            pairs = tuple((cand[i], j, s) for i, j, s in a.pairs)
            full = assoc.Assignment(pairs, (), a.unmatched_detections)
            scene = track.update(scene, full, dets, t)
    return scene, st


STEP_CASES = [
    # name, W, H, objects, frames, det_every, warps, iters, scales, seed
    ("s0", 160, 128, 5, 8, 2, 2, 10, None, 7),
    ("s1", 96, 80, 3, 3, 1, 5, 50, None, 8),
    ("s2", 200, 150, 12, 6, 3, 2, 8, 3, 9),
]


def dets_to_arr(dets):
    if dets is None:
        return np.zeros((0, 6)), -1
    return np.array([[d.class_id, d.score, *d.box] for d in dets]).reshape(-1, 6), len(dets)


def scene_to_arr(scene):
    rows = []
    for o in scene:
        rows.append([o.id, o.class_id, *o.box, 1 if o.state == track.ACTIVE else 0,
                     o.born_at, o.last_seen, o.score, -1 if o.lost_at is None else o.lost_at])
    return np.array(rows, dtype=np.float64).reshape(-1, 11)


def gen_step():
    for name, W, H, nobj, T, every, wp, it, sc, seed in STEP_CASES:
        frames, dets = make_sequence(W, H, nobj, T, seed=seed, det_every=every,
                                     scale_change=True)
        prm = optflow.FlowParams(warps_per_level=wp, iterations_per_warp=it, pyramid_scales=sc)
        scene, prev = [], None
        out = {"frames": frames, "prm": np.array([W, H, -1 if sc is None else sc, wp, it])}
        for t in range(T):
            arr, n = dets_to_arr(dets[t])
            out[f"d{t}"] = arr
            out[f"n{t}"] = np.array([n])
            if dets[t] is not None:
                out[f"lab{t}"] = np.array([d.label for d in dets[t]])
            scene, prev = ref_step(scene, prev, frames[t], t, dets[t], prm)
            out[f"scene{t}"] = scene_to_arr(scene)
        save(f"step_{name}.npz", **out)


def gen_io():
    """video_io parsing (PGM with comments, PPM -> luma, Y4M 420) and optflow
    diagnostics (flow_energy, .flo bytes) from the reference."""
    import tempfile

    from flowtrack import video_io
    rng = np.random.default_rng(51)
    out = {}
    g = rng.integers(0, 256, (7, 9), dtype=np.uint8)
    pgm = b"P5\n# made by make_golden\n9 7\n# max\n255\n" + g.tobytes()
    rgb = rng.integers(0, 256, (5, 6, 3), dtype=np.uint8)
    ppm = b"P6 6 5 255\n" + rgb.tobytes()
    ys = [rng.integers(0, 256, (6, 10), dtype=np.uint8) for _ in range(3)]
    y4m = b"YUV4MPEG2 W10 H6 F25:1 Ip A1:1 C420jpeg\n"
    for y in ys:
        y4m += b"FRAME\n" + y.tobytes() + bytes(2 * 5 * 3)
    with tempfile.TemporaryDirectory() as d:
        for name, blob in (("a.pgm", pgm), ("b.ppm", ppm), ("c.y4m", y4m)):
            open(os.path.join(d, name), "wb").write(blob)
        out["pgm_bytes"] = np.frombuffer(pgm, np.uint8)
        out["pgm_want"] = video_io.read_pgm(os.path.join(d, "a.pgm"))
        out["ppm_bytes"] = np.frombuffer(ppm, np.uint8)
        out["ppm_want"] = video_io.read_pgm(os.path.join(d, "b.ppm"))
        out["y4m_bytes"] = np.frombuffer(y4m, np.uint8)
        out["y4m_want"] = np.stack([f.data for f in video_io.iter_y4m(os.path.join(d, "c.y4m"))])
        z = np.load(os.path.join(HERE, "flow.npz"))
        pa = imaging.Frame.from_array(z["f0_sta"])
        pb = imaging.Frame.from_array(z["f0_stb"], 1)
        fld = optflow.MotionField(width=pa.width, height=pa.height, dx=z["f0_dx"], dy=z["f0_dy"])
        out["energy"] = np.array([optflow.flow_energy(pa, pb, fld),
                                  optflow.flow_energy(pa, pb, fld, optflow.FlowParams(huber_epsilon=0.0))])
        trace = []
        optflow.compute_flow(pa, pb, optflow.FlowParams(), energy_trace=trace)
        out["energy_trace"] = np.array(trace)
        optflow.write_flo(fld, os.path.join(d, "f.flo"))
        out["flo_bytes"] = np.frombuffer(open(os.path.join(d, "f.flo"), "rb").read(), np.uint8)
    save("io.npz", **out)


# ---- headline workload end to end (VERDICT r01 "next" #1) -------------------
# bench.py's own C2 streams (global stream id s -> seed 1000 + s), 720x576,
# 100 objects with scale change, detections every 5th frame with 1 px jitter,
# default FlowParams, through t = 10: two full-size match/update rounds after
# tracked frames.  ST and flow pairs do not depend on track state
# (imaging.py:128-144, optflow.py:217-253), so they run in a process pool; the
# per-stream predict/match/update chain then runs sequentially.
C2_STREAMS, C2_FRAMES, C2_W, C2_H, C2_OBJ, C2_EVERY = 4, 11, 720, 576, 100, 5
C2_FIELD_STRIDE = 16  # subsampled fields stored (full SD fields are 3.3 MB each)


def _c2_seq(s):
    return make_sequence(C2_W, C2_H, C2_OBJ, C2_FRAMES, seed=1000 + s, det_every=C2_EVERY,
                         scale_change=True, jitter=1.0)


def _c2_st(job):
    s, t = job
    frames, _ = _c2_seq(s)
    u8 = frames[t]
    H, W = u8.shape
    L = imaging.select_level(W, H)
    lvl = imaging.build_pyramid(imaging.Frame.from_gray8(u8, index=t), L + 1).levels[L]
    return imaging.structure_texture(lvl).data


def _c2_flow(job):
    a, b, t = job
    fa = imaging.Frame.from_array(a, t - 1)
    fb = imaging.Frame.from_array(b, t)
    fld = optflow.compute_flow(fa, fb, optflow.FlowParams())
    return fld.dx, fld.dy


def gen_c2():
    import hashlib
    import multiprocessing as mp
    import time
    t0 = time.time()
    n = C2_STREAMS
    with mp.get_context("fork").Pool(min(os.cpu_count() or 1, 16)) as pool:
        sts = pool.map(_c2_st, [(s, t) for s in range(n) for t in range(C2_FRAMES)])
        st = {(s, t): sts[s * C2_FRAMES + t] for s in range(n) for t in range(C2_FRAMES)}
        print(f"  ST done {time.time() - t0:.0f}s", flush=True)
        jobs = [(st[(s, t - 1)], st[(s, t)], t) for s in range(n) for t in range(1, C2_FRAMES)]
        flows = pool.map(_c2_flow, jobs)
        print(f"  flow done {time.time() - t0:.0f}s", flush=True)
    out = {"cfg": np.array([C2_W, C2_H, C2_OBJ, C2_FRAMES, C2_EVERY, n, C2_FIELD_STRIDE])}
    k = 0
    for s in range(n):
        frames, dets = _c2_seq(s)
        out[f"s{s}_frames_sha"] = np.frombuffer(hashlib.sha256(frames.tobytes()).digest(), np.uint8)
        L = imaging.select_level(C2_W, C2_H)
        scene = []
        margin = np.inf
        for t in range(C2_FRAMES):
            d = dets[t]
            if d is not None:
                d = detect.filter_detections(d, 0.5)
            arr, nd = dets_to_arr(dets[t])
            out[f"s{s}_d{t}"] = arr
            out[f"s{s}_n{t}"] = np.array([nd])
            if t == 0:
                if d is not None:
                    scene = track.update([], assoc.Assignment((), (), tuple(range(len(d)))), d, t)
            else:
                dx, dy = flows[k]
                k += 1
                fld = optflow.MotionField(width=C2_W >> L, height=C2_H >> L, dx=dx, dy=dy,
                                          frame_index=t)
                out[f"s{s}_dx{t}"] = dx[::C2_FIELD_STRIDE, ::C2_FIELD_STRIDE].copy()
                out[f"s{s}_dy{t}"] = dy[::C2_FIELD_STRIDE, ::C2_FIELD_STRIDE].copy()
                act = [i for i, o in enumerate(scene) if o.state == track.ACTIVE]
                pred = track.predict([scene[i] for i in act], fld, L, (C2_W, C2_H))
                out[f"s{s}_valid{t}"] = np.array([p is not None for p in pred])
                scene = list(scene)
                for i, p in zip(act, pred):
                    if p is not None:
                        scene[i] = replace(scene[i], box=p)
                if d is not None:
                    cand = [i for i, p in zip(act, pred) if p is not None]
                    objs = [scene[i] for i in cand]
                    for o in objs:  # near-tie exposure: min |iou - gate|
                        for dd in d:
                            if o.class_id == dd.class_id:
                                margin = min(margin, abs(assoc.iou(o.box, dd.box) - 0.3))
                    a = assoc.match(objs, d, 0.3)
                    out[f"s{s}_pairs{t}"] = np.array([(cand[i], j) for i, j, _ in a.pairs],
                                                     dtype=np.int64).reshape(-1, 2)
                    pairs = tuple((cand[i], j, sc) for i, j, sc in a.pairs)
                    scene = track.update(scene, assoc.Assignment(pairs, (), a.unmatched_detections),
                                         d, t)
            out[f"s{s}_scene{t}"] = scene_to_arr(scene)
        out[f"s{s}_min_gate_margin"] = np.array([margin])
        print(f"  stream {s}: {len(scene)} objects, min |iou-gate| {margin:.3e}", flush=True)
    save("c2_tracks.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["imaging", "flow", "predict", "assoc", "step", "io"]
    for w in which:
        globals()[f"gen_{w}"]()
        print("wrote", w)

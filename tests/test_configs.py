"""BASELINE.json configs at their FULL frame sizes and track counts, through
the drop-in Tracker, against the oracle step (oracle/ftoracle.py:step, the
SURVEY 8 A16 composition).  Bit-exact track tables every frame.

* C2 (720x576, 100 tracks, detections every 5th frame, S=auto=6): default
  FlowParams (5 warps x 50 iterations) -- the headline workload itself.
* C1 (720x576, 10 boxes, S=3, detections every frame, no jitter).
* C3 (1920x1080, 200 tracks, S=4; processed at level 1 = 960x540) and
  C4 (3840x2160, 500 tracks, S=5; processed at level 2 = 960x540): the
  oracle's default-parameter flow at 960x540 costs ~25 s per frame pair, so
  these run a declared light FlowParams (1 warp x 4 iterations) at full frame
  size and full track count; pyramid, ROF, predict, match and update are
  at their default settings.
"""
import numpy as np
import pytest

from tests.goldutil import scene_rows

pytestmark = pytest.mark.gpu


def _run(W, H, n_obj, T, seed, det_every, scale_change, jitter, warps, iters, scales):
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from oracle import ftoracle as O
    from paper_1910_06017_b200.optflow import FlowParams
    from paper_1910_06017_b200.pipeline import Tracker
    from paper_1910_06017_b200.synth import make_sequence
    frames, dets = make_sequence(W, H, n_obj, T, seed=seed, det_every=det_every,
                                 scale_change=scale_change, jitter=jitter)
    prm = FlowParams(warps_per_level=warps, iterations_per_warp=iters, pyramid_scales=scales)
    oprm = O.FlowParams(warps_per_level=warps, iterations_per_warp=iters, pyramid_scales=scales)
    trk = Tracker(W, H, n_streams=1, flow_params=prm, max_tracks=1024, max_dets=1024)
    st = O.StreamState()
    n_active = []
    for t in range(T):
        scene = trk.step(frames[t], t, [dets[t]])[0]
        od = None if dets[t] is None else [O.Det(d.class_id, d.label, d.score, d.box) for d in dets[t]]
        O.step(st, frames[t], t, od, oprm)
        assert np.array_equal(scene_rows(scene), scene_rows(st.tracks)), (W, H, t)
        n_active.append(sum(o.state == "active" for o in scene))
    trk.close()
    return n_active


def test_c2_sd_default_params():
    act = _run(720, 576, 100, 2, seed=1000, det_every=5, scale_change=True, jitter=1.0,
               warps=5, iters=50, scales=None)
    assert act[0] > 50  # most of the 100 objects are detected and tracked


def test_c1_sd_three_scales():
    _run(720, 576, 10, 3, seed=1001, det_every=1, scale_change=False, jitter=0.0,
         warps=1, iters=4, scales=3)


def test_c3_hd_200_tracks():
    act = _run(1920, 1080, 200, 3, seed=1002, det_every=1, scale_change=False, jitter=1.0,
               warps=1, iters=4, scales=4)
    assert act[-1] > 100


def test_c4_uhd_500_tracks():
    act = _run(3840, 2160, 500, 2, seed=1003, det_every=1, scale_change=True, jitter=1.0,
               warps=1, iters=4, scales=5)
    assert act[-1] > 250


def test_c5_headline_batch_matches_live_reference():
    """The headline workload itself, pinned end to end to the LIVE reference:
    bench.py's 64-stream C5 batch (global stream id s -> seed 1000 + s;
    720x576, 100 objects with scale change, detections every 5th frame,
    1 px jitter, default FlowParams) through t = 10.  Streams 0-3 are
    compared bit-exactly at every frame against tests/golden/c2_tracks.npz
    (tests/golden/make_golden.py:gen_c2 composed flowtrack's own functions,
    optflow.py:217-253, track.py:56-139, assoc.py:109-135): track tables,
    predict-None masks, match pairs (via the tables) and the motion field on
    a 16-px lattice.  Two full-size match/update rounds follow tracked
    frames (t = 5, 10)."""
    import hashlib
    import os

    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    import bench
    from paper_1910_06017_b200.pipeline import Tracker
    from paper_1910_06017_b200.synth import make_sequence
    from tests.goldutil import step_dets  # noqa: F401  (fixture layout shared)
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "c2_tracks.npz"))
    W, H, n_obj, T, every, n_pin, stride = (int(v) for v in z["cfg"])
    B = 64
    seqs = [make_sequence(W, H, n_obj, T, seed=bench.stream_seed(s), det_every=every,
                          scale_change=True, jitter=1.0) for s in range(B)]
    for s in range(n_pin):
        sha = hashlib.sha256(seqs[s][0].tobytes()).digest()
        assert sha == z[f"s{s}_frames_sha"].tobytes(), f"synthetic stream {s} drifted"
    trk = Tracker(W, H, n_streams=B, max_tracks=256, max_dets=160)
    for t in range(T):
        frames = np.stack([seqs[s][0][t] for s in range(B)])
        scenes = trk.step(frames, t, [seqs[s][1][t] for s in range(B)])
        for s in range(n_pin):
            assert np.array_equal(scene_rows(scenes[s]), z[f"s{s}_scene{t}"]), (s, t)
            if t > 0:
                dx, dy = trk.field(s)
                assert np.array_equal(dx[::stride, ::stride], z[f"s{s}_dx{t}"]), (s, t)
                assert np.array_equal(dy[::stride, ::stride], z[f"s{s}_dy{t}"]), (s, t)
    trk.close()

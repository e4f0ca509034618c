"""KLT / MedianFlow backend against its oracle
(oracle/klt_oracle.py).  The oracle is checked on CPU for its defining
properties (it recovers known translations and scale); the device path must
match the oracle bit for bit."""
import numpy as np
import pytest

from oracle import klt_oracle as K


def _scene(shift=(2, 1), scale=1.0, size=(150, 110), seed=0):
    from paper_1910_06017_b200.synth import textured
    rng = np.random.default_rng(seed)
    w, h = size
    base = textured(h + 40, w + 40, rng)
    a = base[20:20 + h, 20:20 + w]
    if scale == 1.0:
        sx, sy = shift
        b = base[20 - sy:20 - sy + h, 20 - sx:20 - sx + w]
    else:  # zoom about the frame centre by `scale`
        from oracle import ftoracle as O
        cy, cx = (h - 1) / 2.0, (w - 1) / 2.0
        ys, xs = np.meshgrid(np.arange(h, dtype=float), np.arange(w, dtype=float), indexing="ij")
        b = O.sample(a, cx + (xs - cx) / scale, cy + (ys - cy) / scale)
    return a, b


def test_oracle_recovers_translation():
    a, b = _scene((2, 1))
    boxes = [(40.0, 30.0, 40.0, 30.0), (90.0, 50.0, 30.0, 40.0)]
    for (x, y, w, h), got in zip(boxes, K.klt_predict(boxes, a, b, 0, (150, 110), grid=5)):
        assert abs(got[0] - (x + 2)) < 0.05 and abs(got[1] - (y + 1)) < 0.05
        assert abs(got[2] - w) < 0.05 and abs(got[3] - h) < 0.05


def test_oracle_recovers_scale_and_lost_boxes():
    a, b = _scene(scale=1.05, seed=3)
    got = K.klt_predict([(45.0, 35.0, 60.0, 40.0)], a, b, 0, (150, 110), grid=6)[0]
    assert abs(got[2] / 60.0 - 1.05) < 0.02 and abs(got[3] / 40.0 - 1.05) < 0.02
    flat = np.full((110, 150), 0.5)  # no texture: structure tensor singular -> None
    assert K.klt_predict([(10.0, 10.0, 30.0, 30.0)], flat, flat, 0, (150, 110), grid=3) == [None]


def test_lane_sum_matches_definition():
    vals = np.random.default_rng(1).standard_normal(81)
    part = [0.0] * 32
    for k, v in enumerate(vals):
        part[k % 32] += v
    for off in (16, 8, 4, 2, 1):
        part = [part[i] + part[i ^ off] for i in range(32)]
    assert K.lane_sum(vals) == part[0] == part[17]


@pytest.mark.gpu
def test_klt_device_bit_exact():
    from paper_1910_06017_b200.imaging import Frame
    from paper_1910_06017_b200.track import SceneObject, predict_klt
    from paper_1910_06017_b200.synth import make_sequence
    from oracle import ftoracle as O
    frames, dets = make_sequence(200, 150, 8, 2, seed=13, scale_change=True)
    a = O.gray8_to_unit(frames[0])
    b = O.gray8_to_unit(frames[1])
    boxes = [d.box for d in dets[0]] + [(0.0, 0.0, 5.0, 5.0), (190.0, 140.0, 9.0, 9.0)]
    want = K.klt_predict(boxes, a, b, 0, (200, 150), grid=7)
    objs = [SceneObject(i, 0, "x", bx) for i, bx in enumerate(boxes)]
    got = predict_klt(objs, Frame.from_array(a), Frame.from_array(b), 0, (200, 150), grid=7)
    assert got == want
    # level-1 coordinates (HD-like): frame 400x300 processed at 200x150
    big = [(2 * x, 2 * y, 2 * w, 2 * h) for x, y, w, h in boxes]
    want1 = K.klt_predict(big, a, b, 1, (400, 300), grid=4)
    objs1 = [SceneObject(i, 0, "x", bx) for i, bx in enumerate(big)]
    assert predict_klt(objs1, Frame.from_array(a), Frame.from_array(b), 1, (400, 300), grid=4) == want1


@pytest.mark.gpu
def test_klt_tracker_matches_oracle():
    """Tracker(motion="klt"): multi-stream lockstep step == oracle step_klt."""
    from oracle import ftoracle as O
    from paper_1910_06017_b200.pipeline import Tracker
    from paper_1910_06017_b200.synth import make_sequence
    from tests.goldutil import scene_rows
    S, W, H, T = 2, 160, 120, 5
    seqs = [make_sequence(W, H, 5, T, seed=70 + s, det_every=2, scale_change=True) for s in range(S)]
    trk = Tracker(W, H, n_streams=S, motion="klt", klt_grid=5, max_tracks=64, max_dets=64)
    states = [O.StreamState() for _ in range(S)]
    for t in range(T):
        frames = np.stack([seqs[s][0][t] for s in range(S)])
        dets = [seqs[s][1][t] for s in range(S)]
        scenes = trk.step(frames, t, dets)
        for s in range(S):
            od = None if dets[s] is None else [O.Det(d.class_id, d.label, d.score, d.box) for d in dets[s]]
            K.step_klt(states[s], frames[s], t, od, grid=5)
            assert np.array_equal(scene_rows(scenes[s]), scene_rows(states[s].tracks)), (s, t)
    trk.close()

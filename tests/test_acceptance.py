"""SPEC acceptance criteria and track-lifecycle properties through the
device path.

* criterion 5: flow accuracy on seeded 128x128 value-noise textures
  translated by integer / half-integer shifts (|s| <= 5): mean endpoint
  error over the central 80 % <= 0.25 px / 0.4 px; zero motion < 1e-3;
* track lifecycle over a long multi-stream run: ids strictly increasing in
  spawn order, a Lost track never re-enters and keeps its last box, and the
  whole run equals the oracle step by step.
"""
import numpy as np
import pytest

from tests.goldutil import scene_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dev():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    return torch.device("cuda", 0)


def _pair(shift, seed):
    from oracle import ftoracle as O
    from paper_1910_06017_b200.synth import textured
    rng = np.random.default_rng(seed)
    big = textured(128 + 32, 128 + 32, rng)
    a = big[16:144, 16:144].copy()
    sx, sy = shift
    ys, xs = np.meshgrid(np.arange(128.0), np.arange(128.0), indexing="ij")
    # curr(x) = prev(x - s): content moves by +s, so the prev->curr field is s
    b = O.sample(big, xs + 16 - sx, ys + 16 - sy)
    return np.clip(a, 0, 1), np.clip(b, 0, 1)


@pytest.mark.parametrize("shift,tol", [((2, 0), 0.25), ((0, -3), 0.25), ((-4, 5), 0.25),
                                       ((0.5, 0.0), 0.4), ((1.5, -2.5), 0.4)])
def test_flow_accuracy_criterion5(dev, shift, tol):
    from paper_1910_06017_b200.imaging import Frame
    from paper_1910_06017_b200.optflow import compute_flow
    a, b = _pair(shift, seed=11)
    f = compute_flow(Frame.from_array(a), Frame.from_array(b))
    c = slice(13, 115)  # central 80 %
    epe = np.hypot(f.dx[c, c] - shift[0], f.dy[c, c] - shift[1]).mean()
    assert epe <= tol, (shift, epe)
    z = compute_flow(Frame.from_array(a), Frame.from_array(a))
    assert np.hypot(z.dx, z.dy).max() < 1e-3


def test_flow_accuracy_pair_matches_oracle(dev):
    from oracle import ftoracle as O
    from paper_1910_06017_b200.imaging import Frame
    from paper_1910_06017_b200.optflow import FlowParams, compute_flow
    a, b = _pair((1.5, -2.5), seed=12)
    prm = FlowParams(warps_per_level=2, iterations_per_warp=20)
    f = compute_flow(Frame.from_array(a), Frame.from_array(b), prm)
    want = O.compute_flow(a, b, O.FlowParams(warps_per_level=2, iterations_per_warp=20))
    assert np.array_equal(f.dx, want[0]) and np.array_equal(f.dy, want[1])


def test_track_lifecycle_long_run(dev):
    from oracle import ftoracle as O
    from paper_1910_06017_b200.optflow import FlowParams
    from paper_1910_06017_b200.pipeline import Tracker
    from paper_1910_06017_b200.synth import make_sequence
    S, W, H, T = 2, 256, 192, 24
    seqs = [make_sequence(W, H, 14, T, seed=500 + s, det_every=5, scale_change=True)
            for s in range(S)]
    prm = FlowParams(warps_per_level=1, iterations_per_warp=5)
    oprm = O.FlowParams(warps_per_level=1, iterations_per_warp=5)
    trk = Tracker(W, H, n_streams=S, flow_params=prm, max_tracks=256, max_dets=64)
    states = [O.StreamState() for _ in range(S)]
    lost_box = [dict() for _ in range(S)]
    seen_ids = [[] for _ in range(S)]
    for t in range(T):
        frames = np.stack([seqs[s][0][t] for s in range(S)])
        dets = [seqs[s][1][t] for s in range(S)]
        scenes = trk.step(frames, t, dets)
        for s in range(S):
            od = None if dets[s] is None else [O.Det(d.class_id, d.label, d.score, d.box)
                                                for d in dets[s]]
            O.step(states[s], frames[s], t, od, oprm)
            assert np.array_equal(scene_rows(scenes[s]), scene_rows(states[s].tracks)), (s, t)
            ids = [o.id for o in scenes[s]]
            assert ids == sorted(ids) and len(set(ids)) == len(ids)  # scene in id order
            for o in scenes[s]:
                if o.id not in seen_ids[s]:
                    assert not seen_ids[s] or o.id > max(seen_ids[s])  # ids strictly increasing
                    assert o.born_at == t
                    seen_ids[s].append(o.id)
                if o.id in lost_box[s]:  # Lost never re-enters, box frozen
                    assert o.state == "lost" and o.box == lost_box[s][o.id]
                if o.state == "lost":
                    lost_box[s].setdefault(o.id, o.box)
    assert all(len(lb) > 0 for lb in lost_box)  # the run exercised track loss
    trk.close()

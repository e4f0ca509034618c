"""Per-stream tracker boundary (SURVEY.md 8(b) ft_step(ctx, stream_id, luma,
w, h, pitch, frame_index, dets, n_dets, ...)): pitched luma, streams that
skip steps (FT_STREAM_SKIP), per-stream frame indices, single-stream steps,
and the reference's Frame / MotionField validation on device data
(imaging.py:33-44, optflow.py:85-86).  Bit-exact against the oracle run on
each stream's own frame sequence."""
import numpy as np
import pytest

from tests.goldutil import scene_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    return torch


def _odets(dets):
    from oracle import ftoracle as O
    return None if dets is None else [O.Det(d.class_id, d.label, d.score, d.box) for d in dets]


def test_pitched_masked_streams_match_oracle(torch):
    """Three streams, luma given as crops of a wider buffer (pitch != width);
    stream 1 has no frame at steps 1 and 3 (it does not advance), stream 2
    numbers its frames from 100; each stream equals the oracle run on the
    frames it actually received."""
    from oracle import ftoracle as O
    from paper_1910_06017_b200.optflow import FlowParams
    from paper_1910_06017_b200.pipeline import Tracker
    from paper_1910_06017_b200.synth import make_sequence
    S, W, H, T = 3, 120, 88, 6
    prm = FlowParams(warps_per_level=2, iterations_per_warp=7)
    oprm = O.FlowParams(warps_per_level=2, iterations_per_warp=7)
    seqs = [make_sequence(W, H, 4, T, seed=70 + s, det_every=2, scale_change=True)
            for s in range(S)]
    skip = {(1, 1), (1, 3)}
    base = {0: 0, 1: 0, 2: 100}
    trk = Tracker(W, H, n_streams=S, flow_params=prm, max_tracks=64, max_dets=64)
    states = [O.StreamState() for _ in range(S)]
    used = [0] * S  # frames each stream has consumed
    wide = np.zeros((H, W + 37), np.uint8)
    for t in range(T):
        frames, dets, idx = [], [], []
        for s in range(S):
            if (s, t) in skip:
                frames.append(None)
                dets.append(None)
                idx.append(0)
                continue
            k = used[s]
            buf = wide.copy()
            buf[:, 13:13 + W] = seqs[s][0][k]
            frames.append(buf[:, 13:13 + W])  # pitched view, stride W + 37
            dets.append(seqs[s][1][k])
            idx.append(base[s] + k)
        assert frames[0].strides[0] == W + 37
        recs = trk.step_records(frames, idx, dets)
        scenes = trk.scenes(recs)
        for s in range(S):
            if (s, t) in skip:
                continue
            k = used[s]
            O.step(states[s], seqs[s][0][k], base[s] + k, _odets(seqs[s][1][k]), oprm)
            used[s] += 1
        for s in range(S):
            assert np.array_equal(scene_rows(scenes[s]), scene_rows(states[s].tracks)), (s, t)
    assert used == [T, T - 2, T]
    assert any(o.born_at >= 100 for o in scenes[2])
    trk.close()


def test_step_stream_matches_oracle(torch):
    """ft_tracker_step_stream: one stream advances, the other does not."""
    from oracle import ftoracle as O
    from paper_1910_06017_b200.optflow import FlowParams
    from paper_1910_06017_b200.pipeline import Tracker
    from paper_1910_06017_b200.synth import make_sequence
    W, H, T = 96, 72, 4
    frames, dets = make_sequence(W, H, 3, T, seed=91, det_every=1)
    trk = Tracker(W, H, n_streams=2, flow_params=FlowParams(warps_per_level=1,
                                                            iterations_per_warp=6),
                  max_tracks=32, max_dets=32)
    st = O.StreamState()
    oprm = O.FlowParams(warps_per_level=1, iterations_per_warp=6)
    for t in range(T):
        scene = trk.step_stream(1, frames[t], t, dets[t])
        O.step(st, frames[t], t, _odets(dets[t]), oprm)
        assert np.array_equal(scene_rows(scene), scene_rows(st.tracks)), t
    other = trk.read()[0]
    assert len(other) == 0  # stream 0 never advanced
    trk.close()


def test_device_frame_and_field_validation(torch):
    from paper_1910_06017_b200.imaging import Frame
    from paper_1910_06017_b200.optflow import MotionField
    ok = torch.rand((6, 7), dtype=torch.float64, device="cuda")
    f = Frame(7, 6, 0, ok)
    assert np.array_equal(f.data, ok.cpu().numpy())
    bad = ok.clone()
    bad[2, 3] = float("nan")
    with pytest.raises(ValueError, match="non-finite"):
        Frame(7, 6, 0, bad)
    big = ok.clone()
    big[0, 0] = 1.5
    with pytest.raises(ValueError, match=r"\[0, 1\]"):
        Frame(7, 6, 0, big)
    neg = ok.clone()
    neg[5, 6] = -1e-300
    with pytest.raises(ValueError, match=r"\[0, 1\]"):
        Frame(7, 6, 0, neg)
    dx = torch.zeros((6, 7), dtype=torch.float64, device="cuda")
    dy = dx.clone()
    MotionField(7, 6, dx, dy)
    dy[1, 1] = float("inf")
    with pytest.raises(ValueError, match="non-finite"):
        MotionField(7, 6, dx, dy)


def test_skip_validation(torch):
    from paper_1910_06017_b200 import _lib
    from paper_1910_06017_b200.pipeline import Tracker
    trk = Tracker(32, 24, n_streams=2, max_tracks=8, max_dets=8)
    with pytest.raises(ValueError, match="pitch"):
        _lib.check(trk._lib.ft_tracker_stage(trk._h, 0, 0, _lib.ptr(np.zeros((24, 32), np.uint8)),
                                             16, 0, None, -1))
    with pytest.raises(ValueError, match="stream out of range"):
        _lib.check(trk._lib.ft_tracker_stage(trk._h, 0, 2, None, 32, 0, None, _lib.FT_STREAM_SKIP))
    with pytest.raises(ValueError, match="FT_STREAM_SKIP"):
        _lib.check(trk._lib.ft_tracker_stage(trk._h, 0, 0, None, 32, 0, None, -3))
    trk.close()


def test_two_trackers_interleaved_pipelined(torch):
    """Two trackers in one process (each with its own streams, step graphs,
    copy stream and per-slot device inputs), pipelined submissions
    interleaved between them: each one's records equal its own sequential
    run."""
    from paper_1910_06017_b200.optflow import FlowParams
    from paper_1910_06017_b200.pipeline import Tracker
    from paper_1910_06017_b200.synth import make_sequence
    W, H, T = 112, 80, 6
    prm = FlowParams(warps_per_level=2, iterations_per_warp=6)
    seq_a = make_sequence(W, H, 4, T, seed=501, det_every=2, scale_change=True)
    seq_b = make_sequence(W, H, 5, T, seed=502, det_every=3, scale_change=True)

    def sequential(seq):
        trk = Tracker(W, H, n_streams=1, flow_params=prm, max_tracks=32, max_dets=32)
        out = [[r.tobytes() for r in trk.step_records([seq[0][t]], t, [seq[1][t]])]
               for t in range(T)]
        trk.close()
        return out

    want_a, want_b = sequential(seq_a), sequential(seq_b)
    ta = Tracker(W, H, n_streams=1, flow_params=prm, max_tracks=32, max_dets=32)
    tb = Tracker(W, H, n_streams=1, flow_params=prm, max_tracks=32, max_dets=32)
    got_a, got_b = [], []
    for t in range(T):
        ta.submit([seq_a[0][t]], t, [seq_a[1][t]])
        tb.submit([seq_b[0][t]], t, [seq_b[1][t]])
        if t:
            got_a.append([r.tobytes() for r in ta.wait()])
            got_b.append([r.tobytes() for r in tb.wait()])
    got_a.append([r.tobytes() for r in ta.wait()])
    got_b.append([r.tobytes() for r in tb.wait()])
    ta.close()
    tb.close()
    assert got_a == want_a and got_b == want_b

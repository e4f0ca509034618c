"""Tracking-quality metrics (SPEC.md harness `evaluate`):
the SPEC known-answer examples and invariants on CPU, and a device run of the
tracker scored against the synthetic ground truth (GPU)."""
import numpy as np
import pytest

from paper_1910_06017_b200.metrics import evaluate, match_frame


def _truth(n_frames=6):
    # two objects moving right, well separated
    rows = []
    for f in range(n_frames):
        rows.append((f, 0, 10.0 + 2 * f, 10.0, 20.0, 20.0))
        rows.append((f, 1, 60.0 + 2 * f, 40.0, 24.0, 16.0))
    return rows


def test_identical_output():  # SPEC: 0 switches, recall 1, mean IoU 1
    gt = _truth()
    m = evaluate([(f, i + 7, x, y, w, h) for f, i, x, y, w, h in gt], gt)
    assert (m.id_switches, m.fragmentation, m.recall, m.mean_iou) == (0, 0, 1.0, 1.0)


def test_swapped_ids_two_switches():  # SPEC: ids swapped at frame k -> exactly 2
    gt = _truth()
    out = [(f, (1 - i) if f >= 3 else i, x, y, w, h) for f, i, x, y, w, h in gt]
    assert evaluate(out, gt).id_switches == 2


def test_empty_output_recall_zero():  # SPEC: empty output -> recall 0
    m = evaluate([], _truth())
    assert m.recall == 0.0 and m.matches == 0


def test_relabel_invariance():  # SPEC: metrics depend on the partition only
    gt = _truth()
    out = [(f, i if f < 4 else 5, x + 1.0, y, w, h) for f, i, x, y, w, h in gt if (f, i) != (2, 1)]
    a = evaluate(out, gt)
    b = evaluate([(f, 100 - i, x, y, w, h) for f, i, x, y, w, h in out], gt)
    assert a == b


def test_fragmentation_and_gate():
    gt = _truth()
    # object 0 missed at frames 2-3 (interrupted once); object 1 shifted below IoU 0.5
    out = [(f, i, x, y, w, h) for f, i, x, y, w, h in gt if not (i == 0 and f in (2, 3))]
    out = [(f, i, x + (15.0 if i == 1 else 0.0), y, w, h) for f, i, x, y, w, h in out]
    m = evaluate(out, gt)
    assert m.fragmentation == 1
    assert m.matches == 4  # object 0 on frames 0, 1, 4, 5 only
    assert match_frame([(0, (0, 0, 10, 10))], [(3, (5, 0, 10, 10))]) == []  # IoU 1/3 < 0.5


def test_optimal_not_greedy():
    # greedy on the best IoU would take (t0, k0) and leave t1 unmatched
    truth = [(0, (0.0, 0.0, 10.0, 10.0)), (1, (3.0, 0.0, 10.0, 10.0))]
    out = [(10, (2.0, 0.0, 10.0, 10.0)), (11, (-3.0, 0.0, 10.0, 10.0))]
    pairs = match_frame(truth, out)
    assert sorted((t, k) for t, k, _ in pairs) == [(0, 11), (1, 10)]


@pytest.mark.gpu
def test_tracker_run_scored():
    """A device run on a synthetic stream: recall and switches from the
    device tracks equal those of the oracle run (bit-exact tracks)."""
    import torch
    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a CUDA device")
    from oracle import ftoracle as O
    from paper_1910_06017_b200.optflow import FlowParams
    from paper_1910_06017_b200.pipeline import Tracker, track_records
    from paper_1910_06017_b200.synth import SyntheticStream

    W, H, T = 160, 128, 12
    s = SyntheticStream(W, H, 4, seed=5)
    frames, dets, truth = [], [], []
    for t in range(T):
        s.advance()
        frames.append(s.render())
        d = s.detections()
        dets.append(d if t % 3 == 0 else None)
        truth += [(t, k, *box) for k, (_, box) in enumerate(s.gt_boxes(t))]
    prm = FlowParams(warps_per_level=2, iterations_per_warp=10)
    trk = Tracker(W, H, n_streams=1, flow_params=prm, max_tracks=32, max_dets=32)
    st = O.StreamState()
    oprm = O.FlowParams(warps_per_level=2, iterations_per_warp=10)
    dev_rows, ora_rows = [], []
    for t in range(T):
        scene = trk.step(frames[t], t, [dets[t]])[0]
        dev_rows += track_records(scene, t)
        od = None if dets[t] is None else [O.Det(d.class_id, d.label, d.score, d.box) for d in dets[t]]
        O.step(st, frames[t], t, od, oprm)
        ora_rows += [(t, o.id, *o.box) for o in st.tracks if o.state == "active"]
    trk.close()
    m_dev, m_ora = evaluate(dev_rows, truth), evaluate(ora_rows, truth)
    assert m_dev == m_ora
    assert m_dev.recall > 0.6 and m_dev.id_switches == 0  # oracle run: recall 0.77, 0 switches

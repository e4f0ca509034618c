"""Ingest / output boundary: PGM/PPM/Y4M parsing,
JSONL detection sidecars, .flo files -- checked against fixtures written by
the live reference (tests/golden/make_golden.py:gen_io).  Host-only parts
run on CPU; flow_energy and Frame ingest run on the GPU."""
import json

import numpy as np
import pytest

from paper_1910_06017_b200 import detect, video_io


def _write(tmp_path, name, arr):
    p = tmp_path / name
    p.write_bytes(arr.tobytes())
    return p


def test_pgm_ppm_y4m_parse(golden, tmp_path):
    z = golden("io.npz")
    assert np.array_equal(video_io.read_pgm(_write(tmp_path, "a.pgm", z["pgm_bytes"])), z["pgm_want"])
    assert np.array_equal(video_io.read_pgm(_write(tmp_path, "b.ppm", z["ppm_bytes"])), z["ppm_want"])
    frames = list(video_io.iter_y4m_u8(_write(tmp_path, "c.y4m", z["y4m_bytes"])))
    want = np.rint(z["y4m_want"] * 255.0).astype(np.uint8)
    assert len(frames) == 3 and all(np.array_equal(f, w) for f, w in zip(frames, want))


def test_pgm_errors_and_roundtrip(tmp_path):
    bad = tmp_path / "bad.pgm"
    bad.write_bytes(b"P2\n3 3\n255\n" + bytes(9))
    with pytest.raises(video_io.FormatError, match="not a binary PGM"):
        video_io.read_pgm(bad)
    trunc = tmp_path / "t.pgm"
    trunc.write_bytes(b"P5\n4 4\n255\n" + bytes(5))
    with pytest.raises(video_io.FormatError, match="truncated"):
        video_io.read_pgm(trunc)
    deep = tmp_path / "d.pgm"
    deep.write_bytes(b"P5\n2 2\n65535\n" + bytes(8))
    with pytest.raises(video_io.FormatError, match="8-bit"):
        video_io.read_pgm(deep)
    img = np.arange(12, dtype=np.uint8).reshape(3, 4)
    video_io.write_pgm(tmp_path / "r.pgm", img)
    assert np.array_equal(video_io.read_pgm(tmp_path / "r.pgm"), img)
    video_io.write_y4m(tmp_path / "m.y4m", [img, img[::-1]])
    got = list(video_io.iter_y4m_u8(tmp_path / "m.y4m"))
    assert np.array_equal(got[0], img) and np.array_equal(got[1], img[::-1])
    with pytest.raises(video_io.FormatError):
        video_io.load_frames(tmp_path / "x.avi")


def test_detection_sidecar(tmp_path):
    p = tmp_path / "d.jsonl"
    recs = [{"frame": 0, "class_id": 1, "label": "car", "score": 0.9, "box": [1, 2, 3, 4]},
            {"frame": 2, "class_id": 80, "label": "text", "score": 0.6, "box": [5.5, 6, 7, 8]}]
    p.write_text("\n".join(json.dumps(r) for r in recs) + "\n\n")
    src = detect.ScriptedSource.from_file(p)
    assert src.lookup(1) == []
    assert src.lookup(2)[0].box == (5.5, 6.0, 7.0, 8.0)
    for bad_line, msg in [('{"frame": 0}', "missing key"), ("nope", "invalid JSON"),
                          ('{"frame": -1, "class_id": 1, "label": "a", "score": 0.5, "box": [0,0,1,1]}',
                           "bad frame index"),
                          ('{"frame": 0, "class_id": 1, "label": "a", "score": 1.5, "box": [0,0,1,1]}',
                           "outside")]:
        q = tmp_path / "bad.jsonl"
        q.write_text(bad_line + "\n")
        with pytest.raises(detect.DetectionFormatError, match=msg):
            detect.load_detection_file(q)
    back = tmp_path / "back.jsonl"
    back.write_text("\n".join(json.dumps(r) for r in reversed(recs)))
    with pytest.raises(detect.DetectionFormatError, match="backwards"):
        detect.load_detection_file(back)
    rf = detect.adaptive_receptive_field(1920, 1080, 608)
    assert (rf.width, rf.height) == (608, 342)  # SPEC acceptance criterion 1
    assert detect.adaptive_receptive_field(1080, 1920, 608) == detect.ReceptiveField(342, 608)
    assert detect.adaptive_receptive_field(720, 576, 608) == detect.ReceptiveField(608, 486)
    for sq in (608, 1000, 64):  # square frames: the square field (criterion 1's identity case)
        assert detect.adaptive_receptive_field(sq, sq, 608) == detect.ReceptiveField(608, 608)


def test_flo_bytes_match_reference(golden, tmp_path):
    from paper_1910_06017_b200.optflow import MotionField, read_flo, write_flo
    z = golden("flow.npz")
    fld = MotionField(z["f0_sta"].shape[1], z["f0_sta"].shape[0], z["f0_dx"], z["f0_dy"])
    write_flo(fld, tmp_path / "f.flo")
    assert (tmp_path / "f.flo").read_bytes() == golden("io.npz")["flo_bytes"].tobytes()
    back = read_flo(tmp_path / "f.flo")
    assert np.array_equal(back.dx, z["f0_dx"].astype(np.float32).astype(np.float64))


@pytest.mark.gpu
def test_flow_energy_and_device_ingest(golden, tmp_path):
    from paper_1910_06017_b200.imaging import Frame
    from paper_1910_06017_b200.optflow import FlowParams, MotionField, flow_energy
    zf, zi = golden("flow.npz"), golden("io.npz")
    a, b = Frame.from_array(zf["f0_sta"]), Frame.from_array(zf["f0_stb"], 1)
    fld = MotionField(a.width, a.height, zf["f0_dx"], zf["f0_dy"])
    assert flow_energy(a, b, fld) == zi["energy"][0]
    assert flow_energy(a, b, fld, FlowParams(huber_epsilon=0.0)) == zi["energy"][1]
    frames = list(video_io.iter_y4m(_write(tmp_path, "c.y4m", zi["y4m_bytes"])))
    assert all(np.array_equal(f.data, w) for f, w in zip(frames, zi["y4m_want"]))
    assert [f.index for f in frames] == [0, 1, 2]


def test_track_records_mot_roundtrip(tmp_path):
    import io

    from paper_1910_06017_b200.pipeline import read_mot, track_records, write_jsonl, write_mot
    from paper_1910_06017_b200.track import LOST, SceneObject
    scene = [SceneObject(0, 3, "car", (1.5, 2.0, 10.0, 12.0), born_at=0, last_seen=4, score=0.75),
             SceneObject(1, 80, "text", (5.0, 6.0, 7.0, 8.0), state=LOST, born_at=1, last_seen=3,
                         lost_at=4),
             SceneObject(2, 81, "logo", (9.0, 9.0, 2.0, 2.0), state=LOST, born_at=0, last_seen=1,
                         lost_at=2)]
    rows = track_records(scene, 4)
    assert [r["id"] for r in rows] == [0, 1]  # active + newly lost only
    buf = io.StringIO()
    write_mot(rows, buf)
    assert buf.getvalue().splitlines()[0] == "5,1,1.5,2.0,10.0,12.0,0.75,-1,-1,-1"
    back = read_mot(io.StringIO(buf.getvalue()))
    assert [(b["frame"], b["id"], b["x"], b["w"]) for b in back] == [(4, 0, 1.5, 10.0), (4, 1, 5.0, 7.0)]
    jb = io.StringIO()
    write_jsonl(rows, jb)
    assert json.loads(jb.getvalue().splitlines()[1])["state"] == "lost"


@pytest.mark.gpu
def test_run_driver_matches_oracle():
    from oracle import ftoracle as O
    from paper_1910_06017_b200.optflow import FlowParams
    from paper_1910_06017_b200.pipeline import run
    from paper_1910_06017_b200.synth import make_sequence
    frames, dets = make_sequence(96, 64, 3, 4, seed=61, det_every=1)
    src = detect.ScriptedSource({t: d for t, d in enumerate(dets)})
    st = O.StreamState()
    prm = O.FlowParams(warps_per_level=1, iterations_per_warp=5)
    for t, scene in run(frames, src, 96, 64, detect_every=2,
                        flow_params=FlowParams(warps_per_level=1, iterations_per_warp=5)):
        od = None if t % 2 else [O.Det(d.class_id, d.label, d.score, d.box) for d in dets[t]]
        O.step(st, frames[t], t, od, prm)
        assert [(o.id, o.box, o.state) for o in scene] == [(o.id, o.box, o.state) for o in st.tracks]


@pytest.mark.gpu
def test_pipelined_mode_equivalence():
    """SPEC acceptance criterion 8: the concurrent / prefetch mode yields
    byte-identical scenes to the sequential mode; with a slow detector the
    lookup of frame t+1 overlaps the device work of frame t."""
    import time

    from paper_1910_06017_b200.optflow import FlowParams
    from paper_1910_06017_b200.pipeline import run
    from paper_1910_06017_b200.synth import make_sequence
    frames, dets = make_sequence(160, 120, 6, 8, seed=62, det_every=1, scale_change=True)
    src = detect.DelayedSource(detect.ScriptedSource({t: d for t, d in enumerate(dets)}), 0.02)
    prm = FlowParams(warps_per_level=2, iterations_per_warp=20)
    outs, times = {}, {}
    summ = {}
    for mode in (False, True, "prefetch"):
        t0 = time.perf_counter()
        kw = dict(prefetch=True, summary=summ) if mode == "prefetch" else dict(pipelined=mode)
        outs[mode] = [(t, [(o.id, o.box, o.state, o.lost_at) for o in sc])
                      for t, sc in run(frames, src, 160, 120, detect_every=3, flow_params=prm,
                                       **kw)]
        times[mode] = time.perf_counter() - t0
    assert outs[True] == outs[False]
    assert outs["prefetch"] == outs[False]
    assert [t for t, _ in outs[True]] == list(range(8))
    assert summ["frames"] == 8 and summ["mode"] == "concurrent+prefetch"
    assert summ["census"]["active"] == len(outs[False][-1][1])
    assert summ["mean_phase_ms"] and all(v >= 0 for v in summ["mean_phase_ms"].values())


@pytest.mark.gpu
def test_prefetch_multistream_skip_matches_sequential():
    """Device prefetch with several streams and a stream that skips a step:
    submit / wait / flush records (one-frame lag) equal the sequential
    tracker's step records."""
    from paper_1910_06017_b200.optflow import FlowParams
    from paper_1910_06017_b200.pipeline import Tracker
    from paper_1910_06017_b200.synth import make_sequence
    S, W, H, T = 3, 128, 96, 6
    seqs = [make_sequence(W, H, 4, T, seed=300 + s, det_every=2, scale_change=True)
            for s in range(S)]
    prm = FlowParams(warps_per_level=2, iterations_per_warp=9)

    def inputs(t):
        fr = [seqs[s][0][t] for s in range(S)]
        de = [seqs[s][1][t] for s in range(S)]
        if t == 3:
            fr[1], de[1] = None, None  # stream 1 has no frame at t = 3
        return fr, de

    seq = Tracker(W, H, n_streams=S, flow_params=prm, max_tracks=32, max_dets=32)
    want = []
    for t in range(T):
        fr, de = inputs(t)
        want.append([r.tobytes() for r in seq.step_records(fr, t, de)])
    seq.close()
    pf = Tracker(W, H, n_streams=S, flow_params=prm, max_tracks=32, max_dets=32, prefetch=True)
    got = []
    for t in range(T):
        fr, de = inputs(t)
        pf.submit(fr, t, de)
        r = pf.wait()
        if t == 0:
            assert r is None
        else:
            got.append([x.tobytes() for x in r])
    pf.flush()
    got.append([x.tobytes() for x in pf.wait()])
    assert got == want
    assert any(k.startswith("flow+track") for k in pf.phase_ms())
    # reset with a step still in flight, then replay: same records again
    fr, de = inputs(0)
    pf.submit(fr, 0, de)
    pf.reset()
    again = []
    for t in range(T):
        fr, de = inputs(t)
        pf.submit(fr, t, de)
        r = pf.wait()
        if t:
            again.append([x.tobytes() for x in r])
    pf.flush()
    again.append([x.tobytes() for x in pf.wait()])
    assert again == want
    pf.close()


@pytest.mark.gpu
def test_bench_modes_report():
    """SPEC.md:428-434 bench(): every mode, same scenes (asserted inside)."""
    from paper_1910_06017_b200.optflow import FlowParams
    from paper_1910_06017_b200.pipeline import bench
    from paper_1910_06017_b200.synth import make_sequence
    frames, dets = make_sequence(96, 80, 3, 5, seed=7, det_every=1)
    src = detect.ScriptedSource({t: d for t, d in enumerate(dets)})
    rep = bench(frames, src, 96, 80, detect_every=2,
                flow_params=FlowParams(warps_per_level=1, iterations_per_warp=5))
    assert set(rep) == {"sequential", "concurrent", "concurrent+prefetch", "frames",
                        "paper_concurrency_gain"}
    assert rep["sequential"]["ratio_vs_sequential"] == 1.0
    assert rep["concurrent+prefetch"]["emission_lag_frames"] == 2
    assert all(rep[m]["mean_ms_per_frame"] > 0 for m in ("sequential", "concurrent"))


@pytest.mark.gpu
def test_criterion9_concurrency_benefit():
    """SPEC acceptance criterion 9 (reported, loosely asserted): with a
    detector that takes 20 ms per lookup and a flow-dominated step, the
    concurrent mode's mean per-frame time is at most the sequential one's;
    the ratio is reported (the paper quotes ~20 %)."""
    from paper_1910_06017_b200.optflow import FlowParams
    from paper_1910_06017_b200.pipeline import bench
    from paper_1910_06017_b200.synth import make_sequence
    frames, dets = make_sequence(320, 240, 8, 10, seed=9, det_every=1, scale_change=True)
    src = detect.DelayedSource(detect.ScriptedSource({t: d for t, d in enumerate(dets)}), 0.02)
    prm = FlowParams(warps_per_level=3, iterations_per_warp=30)
    bench(frames[:3], src, 320, 240, detect_every=1, flow_params=prm)  # warm-up (module load)
    rep = bench(frames, src, 320, 240, detect_every=1, repetitions=2, flow_params=prm)
    ratio = rep["concurrent"]["ratio_vs_sequential"]
    print(f"criterion 9: concurrent / sequential = {ratio:.3f} "
          f"(prefetch {rep['concurrent+prefetch']['ratio_vs_sequential']:.3f}; paper ~0.8)")
    assert ratio <= 1.0, rep


@pytest.mark.gpu
def test_energy_trace_matches_reference(golden):
    from paper_1910_06017_b200.imaging import Frame
    from paper_1910_06017_b200.optflow import compute_flow
    zf, zi = golden("flow.npz"), golden("io.npz")
    a, b = Frame.from_array(zf["f0_sta"]), Frame.from_array(zf["f0_stb"], 1)
    trace = []
    fld = compute_flow(a, b, energy_trace=trace)
    assert np.array_equal(np.array(trace), zi["energy_trace"])
    assert np.array_equal(fld.dx, zf["f0_dx"])

"""Pin the CPU oracle (oracle/ftoracle.py) to the live-reference fixtures.

Everything here is bit-exact (np.array_equal) -- the oracle restates the
reference's floating-point operation order.  CPU only.
"""
import itertools

import numpy as np
import pytest

from oracle import ftoracle as O
from tests.goldutil import predict_field, scene_rows, step_dets


def test_pyramid_bit_exact(golden):
    z = golden("imaging.npz")
    for k in range(4):
        u8 = z[f"pyr{k}_in"]
        levels = [z[key] for key in sorted(k2 for k2 in z.files if k2.startswith(f"pyr{k}_l"))]
        got = O.pyramid(O.gray8_to_unit(u8), len(levels))
        for a, b in zip(got, levels):
            assert a.shape == b.shape
            assert np.array_equal(a, b)


def test_pyramid_rejects_degenerate():
    with pytest.raises(ValueError):
        O.pyramid(np.zeros((5, 5)), 3)
    with pytest.raises(ValueError):
        O.pyramid(np.zeros((5, 5)), 0)


def test_select_level_kats():
    # SPEC.md:59-61 and SURVEY.md section 4
    assert O.select_level(720, 576) == 0
    assert O.select_level(2560, 1280) == 1
    assert O.select_level(4096, 2048) == 2
    assert O.select_level(1920, 1080) == 1
    assert O.select_level(3840, 2160) == 2


def test_structure_texture_bit_exact(golden):
    z = golden("imaging.npz")
    for k in range(4):
        wt, bl, it = z[f"st{k}_prm"]
        got = O.structure_texture(O.gray8_to_unit(z[f"st{k}_in"]), wt, bl, int(it))
        assert np.array_equal(got, z[f"st{k}_out"])


def test_structure_texture_constant_kat():
    out = O.structure_texture(np.full((16, 16), 0.3))
    assert np.allclose(out, (0.05 * 0.3 + 0.95) / 1.95, atol=0, rtol=1e-15)


def _prm(p):
    w, h, sc, wp, it = (int(v) for v in p)
    return O.FlowParams(warps_per_level=wp, iterations_per_warp=it,
                        pyramid_scales=None if sc < 0 else sc)


def test_flow_bit_exact(golden):
    z = golden("flow.npz")
    for k in range(5):
        sta = O.structure_texture(O.gray8_to_unit(z[f"f{k}_a"]))
        stb = O.structure_texture(O.gray8_to_unit(z[f"f{k}_b"]))
        assert np.array_equal(sta, z[f"f{k}_sta"])
        assert np.array_equal(stb, z[f"f{k}_stb"])
        dx, dy = O.compute_flow(sta, stb, _prm(z[f"f{k}_prm"]))
        assert np.array_equal(dx, z[f"f{k}_dx"]), k
        assert np.array_equal(dy, z[f"f{k}_dy"]), k


def test_identical_frames_zero_flow(golden):
    z = golden("flow.npz")
    assert np.abs(z["f3_dx"]).max() == 0.0 and np.abs(z["f3_dy"]).max() == 0.0


def test_predict_bit_exact(golden):
    z = golden("predict.npz")
    for k in range(4):
        fw, fh, lvl = (int(v) for v in z[f"p{k}_meta"])
        lw, lh = fw >> lvl, fh >> lvl
        dx, dy = predict_field(k, lw, lh)
        tr = [O.Track(id=i, class_id=0, label="x", box=tuple(b))
              for i, b in enumerate(z[f"p{k}_boxes"])]
        got = O.predict(tr, dx, dy, lvl, (fw, fh))
        want = z[f"p{k}_out"]
        for g, w in zip(got, want):
            if g is None:
                assert np.isnan(w).all()
            else:
                assert np.array_equal(np.array(g), w)
    tr = [O.Track(id=0, class_id=0, label="a", box=(10.0, 10.0, 20.0, 20.0))]
    got = O.predict(tr, np.full((64, 64), 3.0), np.full((64, 64), -2.0), 0, (64, 64))
    assert got[0] == (13.0, 8.0, 20.0, 20.0)
    assert np.array_equal(np.array(got[0]), z["kat_uniform"])


def test_iou_and_kats(golden):
    z = golden("assoc.npz")
    got = np.array([[O.iou(tuple(a), tuple(b)) for b in z["iou_b"]] for a in z["iou_a"]])
    assert np.array_equal(got, z["iou_ab"])
    assert O.iou((0, 0, 10, 10), (5, 0, 10, 10)) == 1 / 3
    assert O.iou((1, 2, 3, 4), (1, 2, 3, 4)) == 1.0
    assert O.iou((0, 0, 1, 1), (5, 5, 1, 1)) == 0.0
    with pytest.raises(ValueError):
        O.iou((0, 0, 0, 1), (0, 0, 1, 1))


def test_hungarian_golden_and_kats(golden):
    z = golden("assoc.npz")
    for k in range(40):
        forb = O.FORBIDDEN if bool(z[f"h{k}_forb"][0]) else None
        got = O.hungarian(z[f"h{k}_cost"], forbidden=forb)
        assert [tuple(p) for p in z[f"h{k}_pairs"].tolist()] == got, k
    assert O.hungarian([[5.0]]) == [(0, 0)]
    assert O.hungarian([[1.0, 2.0], [2.0, 4.0]]) == [(0, 1), (1, 0)]
    assert O.hungarian([[3.0], [1.0]]) == [(1, 0)]
    assert O.hungarian(np.zeros((3, 3))) == [(0, 0), (1, 1), (2, 2)]
    assert O.hungarian(np.ones((2, 3))) == [(0, 0), (1, 1)]
    assert O.hungarian(np.ones((3, 2))) == [(0, 0), (1, 1)]
    assert O.hungarian(np.zeros((0, 3))) == []


def test_hungarian_brute_force_small():
    # SPEC acceptance criterion 3 (reduced count for the CPU suite)
    rng = np.random.default_rng(3)
    for _ in range(150):
        m, n = int(rng.integers(1, 6)), int(rng.integers(1, 6))
        c = rng.random((m, n))
        pairs = O.hungarian(c)
        tot = sum(c[i, j] for i, j in pairs)
        k = min(m, n)
        best = min(sum(c[i, j] for i, j in zip(rows, cols))
                   for rows in itertools.combinations(range(m), k)
                   for cols in itertools.permutations(range(n), k))
        assert abs(tot - best) < 1e-12


def test_match_golden(golden):
    z = golden("assoc.npz")
    for k in range(3):
        tr = [O.Track(id=i, class_id=int(c), label="t", box=tuple(b))
              for i, (b, c) in enumerate(zip(z[f"m{k}_tb"], z[f"m{k}_tc"]))]
        de = [O.Det(class_id=int(c), label="d", score=0.9, box=tuple(b))
              for b, c in zip(z[f"m{k}_db"], z[f"m{k}_dc"])]
        pairs, us, ud = O.match(tr, de, 0.3)
        assert [(i, j) for i, j, _ in pairs] == [tuple(p) for p in z[f"m{k}_pairs"].tolist()]
        assert np.array_equal(np.array([s for _, _, s in pairs]), z[f"m{k}_ious"])
        assert list(us) == z[f"m{k}_um_s"].tolist()
        assert list(ud) == z[f"m{k}_um_d"].tolist()


def test_update_lifecycle():
    d = [O.Det(1, "a", 0.9, (0.0, 0.0, 5.0, 5.0)), O.Det(2, "b", 0.8, (9.0, 9.0, 3.0, 3.0))]
    s = O.update([], (), d, 0)
    assert [o.id for o in s] == [0, 1]
    s = O.update(s, ((1, 0, 0.5),), [O.Det(2, "b", 0.7, (9.5, 9.0, 3.0, 3.0))], 1)
    assert s[0].state == O.LOST and s[0].lost_at == 1
    assert s[1].box == (9.5, 9.0, 3.0, 3.0) and s[1].last_seen == 1
    s = O.update(s, (), d, 2)
    assert [o.id for o in s] == [0, 1, 2, 3]  # ids never reused
    with pytest.raises(ValueError):
        O.update(s, ((0, 0, 1.0),), d, 3)
    with pytest.raises(IndexError):
        O.update(s, ((9, 0, 1.0),), d, 3)


@pytest.mark.parametrize("name", ["s0", "s1", "s2"])
def test_step_bit_exact(golden, name):
    z = golden(f"step_{name}.npz")
    W, H, sc, wp, it = (int(v) for v in z["prm"])
    prm = O.FlowParams(warps_per_level=wp, iterations_per_warp=it,
                       pyramid_scales=None if sc < 0 else sc)
    frames = z["frames"]
    st = O.StreamState()
    for t in range(frames.shape[0]):
        dets = step_dets(z, t)
        if dets is not None:
            dets = [O.Det(d.class_id, d.label, d.score, d.box) for d in dets]
        O.step(st, frames[t], t, dets, prm)
        assert np.array_equal(scene_rows(st.tracks), z[f"scene{t}"]), (name, t)

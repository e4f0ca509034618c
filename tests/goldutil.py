"""Shared helpers to read the golden fixtures (tests/golden/*.npz)."""
import numpy as np

from paper_1910_06017_b200.detect import Detection


def predict_field(k, lw, lh):
    # mirrors tests/golden/make_golden.py:predict_field
    frng = np.random.default_rng(100 + k)
    return frng.standard_normal((lh, lw)) * 3, frng.standard_normal((lh, lw)) * 3


def step_dets(z, t):
    n = int(z[f"n{t}"][0])
    if n < 0:
        return None
    arr = z[f"d{t}"]
    labels = z[f"lab{t}"]
    return [Detection(class_id=int(r[0]), label=str(labels[i]), score=float(r[1]),
                      box=tuple(float(v) for v in r[2:6])) for i, r in enumerate(arr)]


def scene_rows(tracks):
    """Track-like objects -> (N, 11) float rows matching make_golden.scene_to_arr."""
    rows = []
    for o in tracks:
        rows.append([o.id, o.class_id, *o.box, 1 if o.state == "active" else 0,
                     o.born_at, o.last_seen, o.score, -1 if o.lost_at is None else o.lost_at])
    return np.array(rows, dtype=np.float64).reshape(-1, 11)

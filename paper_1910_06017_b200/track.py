"""Track records and their per-frame lifecycle, executed on the B200.

Drop-in for the reference's track module (track.py): the record type
`SceneObject`, `active_set`, `predict` and `update` keep their names,
arguments, defaults and exceptions.  The arithmetic runs in libomnitrack:

* predict -> ft_predict: per box a warp evaluates the rounded, clamped pixel
  support and the exact numpy-order mean of the flow inside it
  (track.py:56-87);
* update  -> ft_update: the match-driven transition kernel
  (track.py:90-139) -- matched boxes take the detection (or a blend),
  unmatched Active records turn Lost, unmatched detections spawn records
  with fresh ids above every id ever issued.

Records are immutable host values; only their numeric fields cross the
C ABI (labels stay on the host).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .optflow import MotionField

ACTIVE = "active"
LOST = "lost"


def _validated_box(state, born_at, last_seen, box):
    # same checks and messages as the reference record (track.py:35-44)
    if state not in (ACTIVE, LOST):
        raise ValueError(f"unknown state {state!r}")
    if last_seen < born_at:
        raise ValueError("last_seen cannot precede born_at")
    bx, by, bw, bh = (float(v) for v in box)
    if bw <= 0 or bh <= 0:
        raise ValueError(f"box must have positive size, got {box[2]}x{box[3]}")
    return bx, by, bw, bh


@dataclass(frozen=True)
class SceneObject:
    """One tracked entity, box in original-frame pixels (x, y, w, h)."""

    id: int
    class_id: int
    label: str
    box: tuple
    state: str = ACTIVE
    born_at: int = 0
    last_seen: int = 0
    score: float = 1.0
    lost_at: int | None = None

    def __post_init__(self):
        object.__setattr__(self, "box",
                           _validated_box(self.state, self.born_at, self.last_seen, self.box))


def active_set(objects) -> list:
    """The records that still take part in prediction and matching."""
    return [rec for rec in objects if rec.state == ACTIVE]


def _box_array(records) -> np.ndarray:
    arr = np.array([r.box for r in records], dtype=np.float64).reshape(-1, 4)
    return np.ascontiguousarray(arr)


def predict(objects, field: MotionField, level: int, frame_size) -> list:
    """Move every box by the mean motion over its support at pyramid `level`.

    Returns, per record, the new (x, y, w, h) -- size unchanged, position
    clamped into the frame -- or None when the rounded support is empty.
    Lost records are rejected with ValueError, as in the reference.
    """
    records = list(objects)
    lost = next((r for r in records if r.state != ACTIVE), None)
    if lost is not None:
        raise ValueError(f"cannot predict lost object {lost.id}")
    if not records:
        return []
    width, height = frame_size
    src = _box_array(records)
    dst = np.empty_like(src)
    ok = np.empty(len(records), dtype=np.uint8)
    fdx, fdy = field.device()
    _lib.check(_lib.load().ft_predict(
        _lib.ctx(), _lib.ptr(src), len(records), _lib.ptr(fdx), _lib.ptr(fdy), field.width,
        field.height, int(level), int(width), int(height), _lib.ptr(dst), _lib.ptr(ok)))
    return [tuple(map(float, dst[k])) if ok[k] else None for k in range(len(records))]


# flags returned per existing record by ft_update
_KEEP, _MATCHED, _TURNED_LOST = 0, 1, 2


def update(objects, assignment, detections, frame_index: int,
           detection_blend: float = 1.0) -> list:
    """One frame of the lifecycle (see module docstring); returns a new list:
    the existing records in order, then one spawned record per unmatched
    detection in detection order."""
    records = list(objects)
    dets = list(detections)
    n_rec, n_det = len(records), len(dets)
    pairs = np.array([(i, j) for i, j, _ in assignment.pairs], dtype=np.int32).reshape(-1, 2)
    for i, j in pairs:  # index errors first, like the reference's first loop
        if not 0 <= i < n_rec:
            raise IndexError(f"scene index {i} out of range")
        if not 0 <= j < n_det:
            raise IndexError(f"detection index {j} out of range")
    matched_to = {int(i): int(j) for i, j in pairs}
    for i in sorted(matched_to):
        if records[i].state != ACTIVE:
            raise ValueError(f"lost object {records[i].id} appeared in the assignment")

    ids = np.array([r.id for r in records], dtype=np.int64)
    active = np.array([r.state == ACTIVE for r in records], dtype=np.int32)
    rows = n_rec + n_det
    src = np.empty(rows, dtype=np.int32)
    boxes = np.empty((rows, 4), dtype=np.float64)
    flags = np.empty(rows, dtype=np.int32)
    new_ids = np.empty(rows, dtype=np.int64)
    count = C.c_int()
    rec_boxes, det_boxes = _box_array(records), _box_array(dets)  # alive across the call
    _lib.check(_lib.load().ft_update(
        _lib.ctx(), _lib.ptr(ids), _lib.ptr(active), _lib.ptr(rec_boxes), n_rec,
        _lib.ptr(pairs), len(pairs), _lib.ptr(det_boxes), n_det, float(detection_blend),
        _lib.ptr(src), _lib.ptr(boxes), _lib.ptr(flags), _lib.ptr(new_ids), C.byref(count)))

    out = []
    for row in range(count.value):
        k = int(src[row])
        if k < 0:  # spawn from detection -k-1
            det = dets[-k - 1]
            out.append(SceneObject(id=int(new_ids[row]), class_id=det.class_id, label=det.label,
                                   box=det.box, state=ACTIVE, born_at=frame_index,
                                   last_seen=frame_index, score=det.score))
            continue
        rec = records[k]
        flag = int(flags[row])
        if flag == _MATCHED:
            out.append(replace(rec, box=tuple(map(float, boxes[row])),
                               score=dets[matched_to[k]].score, last_seen=frame_index))
        elif flag == _TURNED_LOST:
            out.append(replace(rec, state=LOST, lost_at=frame_index))
        else:
            out.append(rec)
    return out


def predict_klt(objects, prev, curr, level: int, frame_size, grid: int = 10) -> list:
    """KLT / MedianFlow alternative to `predict` (the
    backend north_star describes, defined by oracle/klt_oracle.py since the
    reference has none): a grid x grid point set per box is tracked with
    pyramidal Lucas-Kanade between the processing-level frames `prev` and
    `curr` (Frames, e.g. build_pyramid(f, L+1).levels[L]) and back, points
    failing the forward-backward median test are dropped, and the box moves
    by the median displacement and scales by the median pairwise distance
    ratio.  Returns (x, y, w, h) or None per object, like `predict`."""
    records = list(objects)
    lost = next((r for r in records if r.state != ACTIVE), None)
    if lost is not None:
        raise ValueError(f"cannot predict lost object {lost.id}")
    if not records:
        return []
    width, height = frame_size
    src = _box_array(records)
    dst = np.empty_like(src)
    ok = np.empty(len(records), dtype=np.uint8)
    a, b = prev.device(), curr.device()
    _lib.check(_lib.load().ft_klt_predict(
        _lib.ctx(), _lib.ptr(a), _lib.ptr(b), prev.width, prev.height, int(level), int(width),
        int(height), int(grid), _lib.ptr(src), len(records), _lib.ptr(dst), _lib.ptr(ok)))
    return [tuple(map(float, dst[k])) if ok[k] else None for k in range(len(records))]

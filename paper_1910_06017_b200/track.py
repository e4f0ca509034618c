"""Scene-object lifecycle on the B200 (drop-in for reference track.py:
SceneObject, active_set, predict, update).

predict() runs the segmented box-mean kernel on the device field; update()
runs the lifecycle kernel (ft_update).  Objects stay immutable host records.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from . import _lib
from .optflow import MotionField

ACTIVE = "active"
LOST = "lost"


@dataclass(frozen=True)
class SceneObject:
    """A persistent tracked entity in original-frame coordinates (track.py:21-44)."""

    id: int
    class_id: int
    label: str
    box: tuple  # x, y, w, h
    state: str = ACTIVE
    born_at: int = 0
    last_seen: int = 0
    score: float = 1.0
    lost_at: int | None = None

    def __post_init__(self):
        if self.state not in (ACTIVE, LOST):
            raise ValueError(f"unknown state {self.state!r}")
        if self.last_seen < self.born_at:
            raise ValueError("last_seen cannot precede born_at")
        x, y, w, h = self.box
        if w <= 0 or h <= 0:
            raise ValueError(f"box must have positive size, got {w}x{h}")
        object.__setattr__(self, "box", (float(x), float(y), float(w), float(h)))


def active_set(objects) -> list:
    """Objects still eligible for prediction and matching, order kept."""
    return [o for o in objects if o.state == ACTIVE]


def predict(objects, field: MotionField, level: int, frame_size) -> list:
    """Shift each box by the mean flow over its rounded support (track.py:56-87).

    One entry per object: the shifted (x, y, w, h), or None when the box has
    no pixel support left.
    """
    objects = list(objects)
    for o in objects:
        if o.state != ACTIVE:
            raise ValueError(f"cannot predict lost object {o.id}")
    n = len(objects)
    if n == 0:
        return []
    fw, fh = frame_size
    boxes = np.ascontiguousarray(np.array([o.box for o in objects], dtype=np.float64))
    out = np.empty((n, 4), dtype=np.float64)
    valid = np.empty(n, dtype=np.uint8)
    ddx, ddy = field.device()
    _lib.check(_lib.load().ft_predict(_lib.ctx(), _lib.ptr(boxes), n, _lib.ptr(ddx),
                                      _lib.ptr(ddy), field.width, field.height, int(level),
                                      int(fw), int(fh), _lib.ptr(out), _lib.ptr(valid)))
    return [tuple(float(v) for v in out[i]) if valid[i] else None for i in range(n)]


def update(objects, assignment, detections, frame_index: int,
           detection_blend: float = 1.0) -> list:
    """Apply one frame's match results (track.py:90-139): matched objects take
    the detection's box (or a blend) and score, unmatched Active objects turn
    Lost, every unmatched detection spawns a new object with a fresh id."""
    objects = list(objects)
    detections = list(detections)
    n, nd = len(objects), len(detections)
    pairs = []
    for i, j, _ in assignment.pairs:
        if not 0 <= i < n:
            raise IndexError(f"scene index {i} out of range")
        if not 0 <= j < nd:
            raise IndexError(f"detection index {j} out of range")
        pairs.append((i, j))
    matched = {i for i, _ in pairs}
    for i in sorted(matched):
        if objects[i].state != ACTIVE:
            raise ValueError(f"lost object {objects[i].id} appeared in the assignment")
    ids = np.array([o.id for o in objects], dtype=np.int64)
    state = np.array([1 if o.state == ACTIVE else 0 for o in objects], dtype=np.int32)
    boxes = np.array([o.box for o in objects], dtype=np.float64).reshape(-1, 4)
    dboxes = np.array([d.box for d in detections], dtype=np.float64).reshape(-1, 4)
    pr = np.array(pairs, dtype=np.int32).reshape(-1, 2)
    out_src = np.empty(n + nd, dtype=np.int32)    # >=0 object index, <0: -(det+1) spawn
    out_box = np.empty((n + nd, 4), dtype=np.float64)
    out_flag = np.empty(n + nd, dtype=np.int32)   # 0 keep, 1 matched, 2 -> lost
    out_id = np.empty(n + nd, dtype=np.int64)
    cnt = C.c_int()
    _lib.check(_lib.load().ft_update(
        _lib.ctx(), _lib.ptr(ids), _lib.ptr(state), _lib.ptr(np.ascontiguousarray(boxes)), n,
        _lib.ptr(pr), len(pr), _lib.ptr(np.ascontiguousarray(dboxes)), nd,
        float(detection_blend), _lib.ptr(out_src), _lib.ptr(out_box), _lib.ptr(out_flag),
        _lib.ptr(out_id), C.byref(cnt)))
    result = []
    for k in range(cnt.value):
        src = int(out_src[k])
        if src >= 0:
            o = objects[src]
            flag = int(out_flag[k])
            if flag == 1:
                j = dict(pairs)[src]
                result.append(replace(o, box=tuple(float(v) for v in out_box[k]),
                                      score=detections[j].score, last_seen=frame_index))
            elif flag == 2:
                result.append(replace(o, state=LOST, lost_at=frame_index))
            else:
                result.append(o)
        else:
            d = detections[-src - 1]
            result.append(SceneObject(id=int(out_id[k]), class_id=d.class_id, label=d.label,
                                      box=d.box, state=ACTIVE, born_at=frame_index,
                                      last_seen=frame_index, score=d.score))
    return result

"""IoU scoring and globally optimal assignment on the B200 (drop-in for
reference assoc.py: FORBIDDEN_COST, Assignment, iou, hungarian, match).

Cost matrices and the Hungarian solve run in libomnitrack (ft_iou_matrix,
ft_hungarian, ft_match); results are bit-identical to the reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib

FORBIDDEN_COST = 1e6  # assoc.py:18


@dataclass(frozen=True)
class Assignment:
    """Matching result (assoc.py:21-27)."""

    pairs: tuple  # ((scene idx, det idx, iou), ...)
    unmatched_scene: tuple
    unmatched_detections: tuple


def _boxes(items) -> np.ndarray:
    return np.ascontiguousarray(np.array([tuple(b) for b in items], dtype=np.float64).reshape(-1, 4))


def iou_matrix(a, b) -> np.ndarray:
    """IoU of every box in `a` against every box in `b` (device)."""
    A, B = _boxes(a), _boxes(b)
    out = np.empty((len(A), len(B)), dtype=np.float64)
    if out.size:
        _lib.check(_lib.load().ft_iou_matrix(_lib.ctx(), _lib.ptr(A), len(A), _lib.ptr(B),
                                             len(B), _lib.ptr(out)))
    return out


def iou(a, b) -> float:
    """Intersection-over-union of two (x, y, w, h) boxes (assoc.py:30-41)."""
    if a[2] <= 0 or a[3] <= 0 or b[2] <= 0 or b[3] <= 0:
        raise ValueError("boxes must have positive width and height")
    return float(iou_matrix([a], [b])[0, 0])


def hungarian(cost, forbidden: float | None = None) -> list:
    """Min-cost assignment of min(m, n) pairs, sorted by row; pairs on cells
    >= `forbidden` are dropped (assoc.py:84-106)."""
    c = np.asarray(cost, dtype=np.float64)
    if c.ndim != 2:
        raise ValueError("cost must be a 2-D matrix")
    if c.size == 0:
        return []
    if not np.all(np.isfinite(c)):
        raise ValueError("costs must be finite")
    c = np.ascontiguousarray(c)
    m, n = c.shape
    pairs = np.empty((min(m, n), 2), dtype=np.int32)
    cnt = C.c_int()
    _lib.check(_lib.load().ft_hungarian(_lib.ctx(), _lib.ptr(c), m, n,
                                        0 if forbidden is None else 1,
                                        0.0 if forbidden is None else float(forbidden),
                                        _lib.ptr(pairs), C.byref(cnt)))
    return [(int(i), int(j)) for i, j in pairs[:cnt.value]]


def match(objects, detections, gate: float = 0.3) -> Assignment:
    """Gated, class-constrained IoU matching (assoc.py:109-135)."""
    m, n = len(objects), len(detections)
    if m == 0 or n == 0:
        return Assignment((), tuple(range(m)), tuple(range(n)))
    tb = _boxes(o.box for o in objects)
    db = _boxes(d.box for d in detections)
    tc = np.array([o.class_id for o in objects], dtype=np.int32)
    dc = np.array([d.class_id for d in detections], dtype=np.int32)
    k = min(m, n)
    pairs = np.empty((k, 2), dtype=np.int32)
    ious = np.empty(k, dtype=np.float64)
    cnt = C.c_int()
    _lib.check(_lib.load().ft_match(_lib.ctx(), _lib.ptr(tb), _lib.ptr(tc), m, _lib.ptr(db),
                                    _lib.ptr(dc), n, float(gate), _lib.ptr(pairs),
                                    _lib.ptr(ious), C.byref(cnt)))
    k = cnt.value
    mi = set(int(i) for i in pairs[:k, 0])
    mj = set(int(j) for j in pairs[:k, 1])
    return Assignment(
        pairs=tuple((int(pairs[t, 0]), int(pairs[t, 1]), float(ious[t])) for t in range(k)),
        unmatched_scene=tuple(i for i in range(m) if i not in mi),
        unmatched_detections=tuple(j for j in range(n) if j not in mj))

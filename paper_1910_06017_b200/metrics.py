"""Tracking-quality metrics of the SPEC harness module (SURVEY.md section 8
row f3; reference SPEC.md `[MODULE] harness`, `[OP] evaluate`).

The reference package specifies but does not ship `evaluate`; this is host
tooling that sits after the hot path (it reads TrackRecord rows, it is never
on the per-frame step).  Semantics, as SPEC states them:

* per frame, an optimal truth <-> track matching at IoU >= 0.5 (maximum
  number of pairs, then maximum total IoU -- the same lexicographic objective
  as the reference's gated Hungarian, assoc.py:109-135, with gate 0.5 and no
  class constraint);
* an id switch is counted when a truth object's matched track id differs
  from its matched id at its previous matched frame;
* fragmentation counts the interruptions of a truth trajectory: a matched
  frame that follows an unmatched stretch after an earlier match;
* mean IoU over all matched pairs; track recall = matched truth instances /
  all truth instances.

Metrics depend only on the partition of the output into tracks, not on the
track id values (SPEC invariant), which tests/test_metrics.py checks.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from scipy.optimize import linear_sum_assignment

from .track import ACTIVE

IOU_MATCH = 0.5
_FORBIDDEN = 1e6  # as assoc.FORBIDDEN_COST: never preferred to a real pair


@dataclass(frozen=True)
class Metrics:
    id_switches: int
    fragmentation: int
    mean_iou: float
    recall: float
    matches: int
    truth_instances: int


def _iou_matrix(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """IoU of (x, y, w, h) boxes, assoc.iou's formula (assoc.py:30-41)."""
    ax, ay, aw, ah = (a[:, k:k + 1] for k in range(4))
    bx, by, bw, bh = (b[None, :, k] for k in range(4))
    iw = np.maximum(0.0, np.minimum(ax + aw, bx + bw) - np.maximum(ax, bx))
    ih = np.maximum(0.0, np.minimum(ay + ah, by + bh) - np.maximum(ay, by))
    inter = iw * ih
    return inter / (aw * ah + bw * bh - inter)


def _by_frame(rows) -> dict:
    """{frame: [(id, (x, y, w, h)), ...]} from TrackRecord rows
    (pipeline.track_records / read_mot dicts with frame, id, x, y, w, h[, state])
    or (frame, id, x, y, w, h) tuples."""
    out: dict = {}
    for r in rows:
        if isinstance(r, dict):
            if r.get("state", ACTIVE) != ACTIVE:  # a track's Lost record is not an output box
                continue
            box = r["box"] if "box" in r else (r["x"], r["y"], r["w"], r["h"])
            f, i, box = int(r["frame"]), int(r["id"]), tuple(map(float, box))
        else:
            f, i, box = int(r[0]), int(r[1]), tuple(map(float, r[2:6]))
        out.setdefault(f, []).append((i, box))
    return out


def match_frame(truth, output, iou_min: float = IOU_MATCH):
    """Optimal matching of one frame: list of (truth_id, track_id, iou)."""
    if not truth or not output:
        return []
    ious = _iou_matrix(np.array([b for _, b in truth], float),
                       np.array([b for _, b in output], float))
    cost = np.where(ious >= iou_min, 1.0 - ious, _FORBIDDEN)
    rr, cc = linear_sum_assignment(cost)
    return [(truth[r][0], output[c][0], float(ious[r, c]))
            for r, c in zip(rr, cc) if ious[r, c] >= iou_min]


def evaluate(output_rows, truth_rows, iou_min: float = IOU_MATCH) -> Metrics:
    """SPEC `evaluate(track output, ground truth)`; both keyed by frame."""
    out, gt = _by_frame(output_rows), _by_frame(truth_rows)
    last_id: dict = {}      # truth id -> track id at its last matched frame
    gap: dict = {}          # truth id -> unmatched since its last match
    switches = frags = n_match = n_truth = 0
    iou_sum = 0.0
    for f in sorted(gt):
        truth = gt[f]
        n_truth += len(truth)
        pairs = match_frame(truth, out.get(f, []), iou_min)
        matched = {t: (k, iou) for t, k, iou in pairs}
        for t, _ in truth:
            if t in matched:
                k, iou = matched[t]
                n_match += 1
                iou_sum += iou
                if t in last_id and last_id[t] != k:
                    switches += 1
                if gap.get(t):
                    frags += 1
                last_id[t] = k
                gap[t] = False
            elif t in last_id:
                gap[t] = True
    return Metrics(id_switches=switches, fragmentation=frags,
                   mean_iou=iou_sum / n_match if n_match else 0.0,
                   recall=n_match / n_truth if n_truth else 0.0,
                   matches=n_match, truth_instances=n_truth)

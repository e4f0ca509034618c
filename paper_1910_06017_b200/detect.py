"""The detector boundary of the hot path (drop-in for reference detect.py's
per-frame types): `Detection` records, the confidence gate, the YoloV3
adaptive receptive field and its box remap, pluggable per-frame sources and
the JSONL sidecar reader.

Everything here is host-side bookkeeping on a few hundred records per frame;
the tracker uploads the gated detections as `ft_det` SoA records.  Anchor
k-means (training-time math) is out of scope.
"""
from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass

GENERAL_CLASS_COUNT = 80  # COCO classes 0..79; text and logo detectors follow
TEXT_CLASS_ID = 80
LOGO_CLASS_ID = 81


class DetectionFormatError(ValueError):
    """A sidecar line could not be parsed (carries path:line)."""


class SourceError(RuntimeError):
    """A detection provider failed while a run was in progress."""


@dataclass(frozen=True)
class Detection:
    """Class, label, confidence in [0, 1] and an (x, y, w, h) pixel box."""

    class_id: int
    label: str
    score: float
    box: tuple

    def __post_init__(self):
        coords = tuple(float(v) for v in self.box)
        if len(coords) != 4 or any(not math.isfinite(v) for v in coords):
            raise ValueError("box coordinates must be finite")
        if coords[2] <= 0 or coords[3] <= 0:
            raise ValueError(f"box must have positive size, got {self.box[2]}x{self.box[3]}")
        if not 0.0 <= self.score <= 1.0:
            raise ValueError(f"score {self.score} outside [0, 1]")
        object.__setattr__(self, "box", coords)


@dataclass(frozen=True)
class ReceptiveField:
    width: int
    height: int


def _snap(side: int, multiple: int) -> int:
    return max(multiple, multiple * int((side + multiple / 2) // multiple))


def adaptive_receptive_field(img_w: int, img_h: int, base: int,
                             round_to: int | None = None) -> ReceptiveField:
    """Detector input keeping the frame's aspect ratio: the long side is
    `base`, the short side base*short/long floored (optionally snapped to a
    multiple of `round_to`); e.g. 1920x1080 at 608 -> 608x342."""
    if img_w <= 0 or img_h <= 0 or base <= 0:
        raise ValueError("image size and base must be positive")
    if img_w >= img_h:
        short = int(base * img_h / img_w)
        return ReceptiveField(base, _snap(short, round_to) if round_to else short)
    short = int(base * img_w / img_h)
    return ReceptiveField(_snap(short, round_to) if round_to else short, base)


def remap_detection(box, field: ReceptiveField, img_w: int, img_h: int):
    """Scale a receptive-field box back to frame pixels (one uniform factor,
    long side over long side) and clip it to the frame."""
    factor = max(img_w, img_h) / max(field.width, field.height)
    x, y, w, h = (float(v) * factor for v in box)
    x_end = min(x + w, float(img_w))
    y_end = min(y + h, float(img_h))
    x0, y0 = max(x, 0.0), max(y, 0.0)
    if x_end <= x0 or y_end <= y0:
        raise ValueError(f"box {tuple(box)} lies entirely outside the "
                         f"{img_w}x{img_h} frame after remapping")
    return (x0, y0, x_end - x0, y_end - y0)


def filter_detections(detections, min_score: float):
    """Keep detections with score >= min_score, in their original order."""
    return [d for d in detections if d.score >= min_score]


class DetectionSource:
    """Provider of the detections of one frame (the reference's plugin
    interface): `lookup(frame_index) -> list[Detection]`."""

    def lookup(self, frame_index: int) -> list:
        raise NotImplementedError


class ScriptedSource(DetectionSource):
    """Replays detections keyed by frame index; unknown frames give []."""

    def __init__(self, by_frame: dict):
        self._table = {k: list(v) for k, v in by_frame.items()}

    @classmethod
    def from_file(cls, path) -> "ScriptedSource":
        return cls(load_detection_file(path))

    def lookup(self, frame_index: int) -> list:
        return list(self._table.get(frame_index, ()))


class DelayedSource(DetectionSource):
    """Wraps a source and sleeps `delay_s` per lookup (detector latency)."""

    def __init__(self, inner: DetectionSource, delay_s: float):
        self._inner, self._delay = inner, float(delay_s)

    def lookup(self, frame_index: int) -> list:
        time.sleep(self._delay)
        return self._inner.lookup(frame_index)


_REQUIRED = ("frame", "class_id", "label", "score", "box")


def _parse_record(raw: str, where: str, last_frame: int):
    def bad(msg):
        return DetectionFormatError(f"{where}: {msg}")

    try:
        rec = json.loads(raw)
    except json.JSONDecodeError as exc:
        raise bad(f"invalid JSON ({exc.msg})") from None
    if not isinstance(rec, dict):
        raise bad("record is not an object")
    missing = [k for k in _REQUIRED if k not in rec]
    if missing:
        raise bad(f"missing key {missing[0]!r}")
    frame = rec["frame"]
    if not isinstance(frame, int) or frame < 0:
        raise bad(f"bad frame index {frame!r}")
    if frame < last_frame:
        raise bad(f"frame indices went backwards ({frame} after {last_frame})")
    if not isinstance(rec["class_id"], int):
        raise bad("class_id must be an integer")
    if not isinstance(rec["label"], str):
        raise bad("label must be a string")
    box = rec["box"]
    if not (isinstance(box, list) and len(box) == 4
            and all(isinstance(v, (int, float)) for v in box)):
        raise bad("box must be [x, y, w, h]")
    if not isinstance(rec["score"], (int, float)):
        raise bad("score must be a number")
    try:
        det = Detection(rec["class_id"], rec["label"], float(rec["score"]),
                        tuple(float(v) for v in box))
    except ValueError as exc:
        raise bad(str(exc)) from None
    return frame, det


def load_detection_file(path) -> dict:
    """JSONL sidecar, one detection per line with keys frame, class_id, label,
    score and box [x, y, w, h]; frames must not decrease."""
    table: dict = {}
    last = -1
    with open(path, "r", encoding="utf-8") as fh:
        for lineno, raw in enumerate(fh, start=1):
            if raw.strip():
                last, det = _parse_record(raw.strip(), f"{path}:{lineno}", last)
                table.setdefault(last, []).append(det)
    return table

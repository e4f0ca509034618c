"""Detection records and the detector-side geometry on the hot path's input
boundary (reference detect.py).

Host-side only: detections are a few hundred records per frame and are
uploaded to the device as SoA arrays by the tracker (pipeline.py).
"""

from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass

GENERAL_CLASS_COUNT = 80
TEXT_CLASS_ID = 80
LOGO_CLASS_ID = 81


class DetectionFormatError(ValueError):
    """Malformed detection sidecar (reference detect.py:23-24)."""


class SourceError(RuntimeError):
    """A detection source failed mid-run (reference detect.py:27-28)."""


@dataclass(frozen=True)
class Detection:
    """One detection in frame pixels (reference detect.py:31-49)."""

    class_id: int
    label: str
    score: float
    box: tuple  # (x, y, w, h)

    def __post_init__(self):
        vals = tuple(float(v) for v in self.box)
        if len(vals) != 4 or not all(math.isfinite(v) for v in vals):
            raise ValueError("box coordinates must be finite")
        if vals[2] <= 0 or vals[3] <= 0:
            raise ValueError(f"box must have positive size, got {vals[2]}x{vals[3]}")
        if not 0.0 <= self.score <= 1.0:
            raise ValueError(f"score {self.score} outside [0, 1]")
        object.__setattr__(self, "box", vals)


@dataclass(frozen=True)
class ReceptiveField:
    width: int
    height: int


def adaptive_receptive_field(img_w: int, img_h: int, base: int,
                             round_to: int | None = None) -> ReceptiveField:
    """Aspect-preserving detector input size; the long side becomes `base`,
    the short side is floored (optionally snapped to a multiple of
    `round_to`) -- reference detect.py:69-88."""
    if img_w <= 0 or img_h <= 0 or base <= 0:
        raise ValueError("image size and base must be positive")
    landscape = img_w >= img_h
    long_, short_img, long_img = base, (img_h if landscape else img_w), (img_w if landscape else img_h)
    short = int(base * short_img / long_img)
    if round_to:
        short = max(round_to, round_to * int((short + round_to / 2) // round_to))
    return ReceptiveField(width=long_, height=short) if landscape else \
        ReceptiveField(width=short, height=long_)


def remap_detection(box, field: ReceptiveField, img_w: int, img_h: int):
    """Receptive-field box -> frame pixels, clamped (detect.py:91-107)."""
    k = max(img_w, img_h) / max(field.width, field.height)
    x, y, w, h = (float(v) * k for v in box)
    right = min(x + w, float(img_w))
    bottom = min(y + h, float(img_h))
    x = max(x, 0.0)
    y = max(y, 0.0)
    if right <= x or bottom <= y:
        raise ValueError(f"box {tuple(box)} lies entirely outside the "
                         f"{img_w}x{img_h} frame after remapping")
    return (x, y, right - x, bottom - y)


def filter_detections(detections, min_score: float):
    """Confidence gate, order preserved (detect.py:210-212)."""
    return [d for d in detections if d.score >= min_score]


class DetectionSource:
    """Per-frame detection provider -- the reference's plugin interface
    (detect.py:215-220)."""

    def lookup(self, frame_index: int) -> list:
        raise NotImplementedError


class ScriptedSource(DetectionSource):
    """In-memory / JSONL replay keyed by frame index (detect.py:223-237)."""

    def __init__(self, by_frame: dict):
        self._by_frame = dict(by_frame)

    @classmethod
    def from_file(cls, path) -> "ScriptedSource":
        return cls(load_detection_file(path))

    def lookup(self, frame_index: int) -> list:
        return list(self._by_frame.get(frame_index, ()))


class DelayedSource(DetectionSource):
    """Adds a fixed latency per lookup (detect.py:240-253)."""

    def __init__(self, inner: DetectionSource, delay_s: float):
        self._inner = inner
        self._delay = float(delay_s)

    def lookup(self, frame_index: int) -> list:
        time.sleep(self._delay)
        return self._inner.lookup(frame_index)


def load_detection_file(path) -> dict:
    """JSONL sidecar: {frame, class_id, label, score, box:[x,y,w,h]} per line,
    frames non-decreasing (detect.py:261-305)."""
    out: dict = {}
    prev = -1
    with open(path, "r", encoding="utf-8") as fh:
        for n, raw in enumerate(fh, start=1):
            raw = raw.strip()
            if not raw:
                continue
            where = f"{path}:{n}"
            try:
                rec = json.loads(raw)
            except json.JSONDecodeError as e:
                raise DetectionFormatError(f"{where}: invalid JSON ({e.msg})") from None
            if not isinstance(rec, dict):
                raise DetectionFormatError(f"{where}: record is not an object")
            for key in ("frame", "class_id", "label", "score", "box"):
                if key not in rec:
                    raise DetectionFormatError(f"{where}: missing key {key!r}")
            fr = rec["frame"]
            if not (isinstance(fr, int) and fr >= 0):
                raise DetectionFormatError(f"{where}: bad frame index {fr!r}")
            if fr < prev:
                raise DetectionFormatError(
                    f"{where}: frame indices went backwards ({fr} after {prev})")
            prev = fr
            if not isinstance(rec["class_id"], int):
                raise DetectionFormatError(f"{where}: class_id must be an integer")
            if not isinstance(rec["label"], str):
                raise DetectionFormatError(f"{where}: label must be a string")
            box = rec["box"]
            if not (isinstance(box, list) and len(box) == 4
                    and all(isinstance(v, (int, float)) for v in box)):
                raise DetectionFormatError(f"{where}: box must be [x, y, w, h]")
            if not isinstance(rec["score"], (int, float)):
                raise DetectionFormatError(f"{where}: score must be a number")
            try:
                det = Detection(rec["class_id"], rec["label"], float(rec["score"]),
                                tuple(float(v) for v in box))
            except ValueError as e:
                raise DetectionFormatError(f"{where}: {e}") from None
            out.setdefault(fr, []).append(det)
    return out

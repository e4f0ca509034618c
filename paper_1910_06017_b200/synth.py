"""Synthetic textured moving-object video + YoloV3-style detections.

The reference ships no harness (SPEC.md:462-527 specifies one); this is the
generator SURVEY.md section 8(d) prescribes, host-side numpy, deterministic
given (seed, stream id):

* background: value noise, lattice cells 8/4/2 px weighted 0.5/0.3/0.2;
* objects: independent value-noise texture (cell 4 px), size U[24,96]*(W/720),
  velocity U[-3,3] px/frame, integer placement, bounced to stay >= 50 % inside
  the frame; optional per-object scale 1+0.01*sin(2*pi*t/60)
  and z-ordered overlaps (config C2);
* detections: GT box + N(0, sigma) jitter, score U[0.55,1], class in [0,82),
  emitted in receptive-field coordinates of
  adaptive_receptive_field(W,H,608) and mapped back with remap_detection
  (detect.py:69-107); a few low-score false positives exercise the 0.5 gate.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .detect import Detection, adaptive_receptive_field, remap_detection


def value_noise(h: int, w: int, cell: int, rng: np.random.Generator) -> np.ndarray:
    """Smooth-step interpolated lattice noise in [0,1]."""
    gh, gw = h // cell + 2, w // cell + 2
    lat = rng.random((gh, gw))
    ys = np.arange(h) / cell
    xs = np.arange(w) / cell
    y0 = ys.astype(np.int64)
    x0 = xs.astype(np.int64)
    fy = ys - y0
    fx = xs - x0
    fy = fy * fy * (3 - 2 * fy)
    fx = fx * fx * (3 - 2 * fx)
    a = lat[y0][:, x0]
    b = lat[y0][:, x0 + 1]
    c = lat[y0 + 1][:, x0]
    d = lat[y0 + 1][:, x0 + 1]
    top = a * (1 - fx) + b * fx
    bot = c * (1 - fx) + d * fx
    return top * (1 - fy[:, None]) + bot * fy[:, None]


def textured(h: int, w: int, rng: np.random.Generator, cells=(8, 4, 2),
             weights=(0.5, 0.3, 0.2)) -> np.ndarray:
    img = np.zeros((h, w))
    for c, wt in zip(cells, weights):
        img += wt * value_noise(h, w, c, rng)
    return img


@dataclass
class _Obj:
    tex: np.ndarray          # base texture (u8)
    w0: float
    h0: float
    x: float
    y: float
    vx: float
    vy: float
    class_id: int
    phase: float
    scaling: bool


class SyntheticStream:
    """One independent synthetic video stream with ground-truth boxes."""

    def __init__(self, width: int, height: int, n_objects: int, seed: int,
                 scale_change: bool = False, jitter: float = 1.0,
                 false_positives: int = 1):
        self.width, self.height = width, height
        self.jitter = float(jitter)
        self.false_positives = int(false_positives)
        self.rng = np.random.default_rng(seed)
        bg = textured(height, width, np.random.default_rng(seed + 1000))
        self.background = np.clip(bg * 255.0, 0, 255).astype(np.uint8)
        k = width / 720.0
        self.objects = []
        for _ in range(n_objects):
            ow = float(self.rng.uniform(24, 96) * k)
            oh = float(self.rng.uniform(24, 96) * k)
            ow = max(4.0, min(ow, width / 2.0))
            oh = max(4.0, min(oh, height / 2.0))
            tex = textured(int(math.ceil(oh * 1.1)) + 2, int(math.ceil(ow * 1.1)) + 2,
                           self.rng, cells=(4,), weights=(1.0,))
            tex = np.clip(40 + tex * 215.0, 0, 255).astype(np.uint8)
            self.objects.append(_Obj(
                tex=tex, w0=ow, h0=oh,
                x=float(self.rng.uniform(0, width - ow)),
                y=float(self.rng.uniform(0, height - oh)),
                vx=float(self.rng.uniform(-3, 3)), vy=float(self.rng.uniform(-3, 3)),
                class_id=int(self.rng.integers(0, 82)),
                phase=float(self.rng.uniform(0, 2 * math.pi)),
                scaling=scale_change))
        self.t = -1
        self.receptive = adaptive_receptive_field(width, height, 608)

    def _size(self, o: _Obj, t: int):
        if not o.scaling:
            return o.w0, o.h0
        s = 1.0 + 0.01 * math.sin(2 * math.pi * t / 60.0 + o.phase)
        return o.w0 * s, o.h0 * s

    def gt_boxes(self, t: int):
        out = []
        for o in self.objects:
            w, h = self._size(o, t)
            out.append((o.class_id, (float(round(o.x)), float(round(o.y)), w, h)))
        return out

    def advance(self):
        """Move objects to the next frame (bounce so >= 50 % stays inside)."""
        self.t += 1
        if self.t == 0:
            return
        for o in self.objects:
            w, h = self._size(o, self.t)
            o.x += o.vx
            o.y += o.vy
            if o.x < -w / 2 or o.x > self.width - w / 2:
                o.vx = -o.vx
                o.x = min(max(o.x, -w / 2), self.width - w / 2)
            if o.y < -h / 2 or o.y > self.height - h / 2:
                o.vy = -o.vy
                o.y = min(max(o.y, -h / 2), self.height - h / 2)

    def render(self) -> np.ndarray:
        """u8 luma for the current frame (objects painted in z order)."""
        img = self.background.copy()
        for o in self.objects:
            w, h = self._size(o, self.t)
            iw, ih = max(1, int(round(w))), max(1, int(round(h)))
            ys = np.minimum((np.arange(ih) * (o.tex.shape[0] - 1) / max(ih - 1, 1)).astype(int),
                            o.tex.shape[0] - 1)
            xs = np.minimum((np.arange(iw) * (o.tex.shape[1] - 1) / max(iw - 1, 1)).astype(int),
                            o.tex.shape[1] - 1)
            patch = o.tex[ys][:, xs]
            x0, y0 = int(round(o.x)), int(round(o.y))
            ax0, ay0 = max(x0, 0), max(y0, 0)
            ax1, ay1 = min(x0 + iw, self.width), min(y0 + ih, self.height)
            if ax1 > ax0 and ay1 > ay0:
                img[ay0:ay1, ax0:ax1] = patch[ay0 - y0:ay1 - y0, ax0 - x0:ax1 - x0]
        return img

    def detections(self) -> list:
        """Noisy GT detections mapped through the receptive field."""
        rf = self.receptive
        inv = max(rf.width, rf.height) / max(self.width, self.height)
        dets = []
        boxes = self.gt_boxes(self.t)
        for cid, (x, y, w, h) in boxes:
            jx, jy, jw, jh = (self.rng.normal(0, self.jitter, 4) if self.jitter > 0
                              else (0.0, 0.0, 0.0, 0.0))
            bx = (x + jx, y + jy, max(w + jw, 2.0), max(h + jh, 2.0))
            det = self._emit(cid, bx, inv, float(self.rng.uniform(0.55, 1.0)))
            if det is not None:
                dets.append(det)
        for _ in range(self.false_positives):
            w = float(self.rng.uniform(10, 40))
            h = float(self.rng.uniform(10, 40))
            bx = (float(self.rng.uniform(0, self.width - w)),
                  float(self.rng.uniform(0, self.height - h)), w, h)
            det = self._emit(int(self.rng.integers(0, 82)), bx, inv,
                             float(self.rng.uniform(0.05, 0.45)))
            if det is not None:
                dets.append(det)
        return dets

    def _emit(self, cid, box, inv, score):
        rf_box = tuple(v * inv for v in box)
        try:
            px = remap_detection(rf_box, self.receptive, self.width, self.height)
        except ValueError:
            return None
        return Detection(class_id=cid, label=f"c{cid}", score=score, box=px)


def make_sequence(width: int, height: int, n_objects: int, n_frames: int,
                  seed: int, det_every: int = 1, scale_change: bool = False,
                  jitter: float = 1.0):
    """(frames u8 [T,H,W], dets list-per-frame or None when no detector
    result that frame)."""
    s = SyntheticStream(width, height, n_objects, seed, scale_change, jitter)
    frames = np.empty((n_frames, height, width), np.uint8)
    dets = []
    for t in range(n_frames):
        s.advance()
        frames[t] = s.render()
        d = s.detections()
        dets.append(d if t % det_every == 0 else None)
    return frames, dets

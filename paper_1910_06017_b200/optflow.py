"""Dense coarse-to-fine TV-L1 optical flow on the B200 (drop-in for
reference optflow.py: FlowParams, MotionField, auto_scales, compute_flow).

The field maps pixels of `prev` to `curr`: content at p in prev appears at
p + field(p) in curr (optflow.py:10-11).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .imaging import Frame

MIN_COARSE_DIM = 16  # optflow.py:26
INTENSITY_SCALE = 255.0  # optflow.py:31


@dataclass(frozen=True)
class FlowParams:
    """Solver parameters (optflow.py:36-66); dual step = 1/(8*time_step)."""

    data_weight: float = 0.15
    huber_epsilon: float = 0.01
    time_step: float = 0.25
    warps_per_level: int = 5
    iterations_per_warp: int = 50
    pyramid_scales: int | None = None  # None: deepest with coarsest dim >= 16

    def __post_init__(self):
        if self.data_weight <= 0:
            raise ValueError("data_weight must be positive")
        if self.huber_epsilon < 0:
            raise ValueError("huber_epsilon must be non-negative")
        if self.time_step <= 0:
            raise ValueError("time_step must be positive")
        if self.warps_per_level < 1:
            raise ValueError("warps_per_level must be >= 1")
        if self.iterations_per_warp < 1:
            raise ValueError("iterations_per_warp must be >= 1")
        if self.pyramid_scales is not None and self.pyramid_scales < 1:
            raise ValueError("pyramid_scales must be >= 1")


class MotionField:
    """Dense per-pixel displacement (optflow.py:69-93).  dx / dy are
    read-only host arrays materialised on first access; the device planes
    stay available to predict() without a round trip."""

    __slots__ = ("width", "height", "frame_index", "_dx", "_dy", "_ddx", "_ddy")

    def __init__(self, width: int, height: int, dx, dy, frame_index: int = -1):
        object.__setattr__(self, "width", int(width))
        object.__setattr__(self, "height", int(height))
        object.__setattr__(self, "frame_index", int(frame_index))
        shape = (self.height, self.width)
        on_dev = type(dx).__module__.startswith("torch")
        if on_dev:
            if tuple(dx.shape) != shape or tuple(dy.shape) != shape:
                raise ValueError(f"field components must be {shape}")
            # optflow.py:85-86 rejects non-finite fields at construction
            # (inside compute_flow): checked on the device
            if _lib.check_plane(dx, -np.inf, np.inf) | _lib.check_plane(dy, -np.inf, np.inf):
                raise ValueError("field contains non-finite values")
            object.__setattr__(self, "_ddx", dx)
            object.__setattr__(self, "_ddy", dy)
            object.__setattr__(self, "_dx", None)
            object.__setattr__(self, "_dy", None)
            return
        dx = np.ascontiguousarray(dx, dtype=np.float64)
        dy = np.ascontiguousarray(dy, dtype=np.float64)
        if dx.shape != shape or dy.shape != shape:
            raise ValueError(f"field components must be {shape}")
        if not (np.all(np.isfinite(dx)) and np.all(np.isfinite(dy))):
            raise ValueError("field contains non-finite values")
        dx = dx.copy()
        dy = dy.copy()
        dx.setflags(write=False)
        dy.setflags(write=False)
        object.__setattr__(self, "_dx", dx)
        object.__setattr__(self, "_dy", dy)
        object.__setattr__(self, "_ddx", None)
        object.__setattr__(self, "_ddy", None)

    def __setattr__(self, name, value):
        raise AttributeError("MotionField is immutable")

    def _host(self):
        if self._dx is None:
            dx = self._ddx.cpu().numpy()
            dy = self._ddy.cpu().numpy()
            dx.setflags(write=False)
            dy.setflags(write=False)
            object.__setattr__(self, "_dx", dx)
            object.__setattr__(self, "_dy", dy)

    @property
    def dx(self) -> np.ndarray:
        self._host()
        return self._dx

    @property
    def dy(self) -> np.ndarray:
        self._host()
        return self._dy

    def device(self):
        """(dx, dy) as CUDA float64 tensors."""
        if self._ddx is None:
            import torch
            object.__setattr__(self, "_ddx", torch.from_numpy(np.array(self._dx)).cuda())
            object.__setattr__(self, "_ddy", torch.from_numpy(np.array(self._dy)).cuda())
        return self._ddx, self._ddy

    def magnitude(self) -> np.ndarray:
        return np.hypot(self.dx, self.dy)


def auto_scales(width: int, height: int) -> int:
    """Pyramid depth whose coarsest level keeps both sides >= 16 (optflow.py:96-104)."""
    out = C.c_int()
    _lib.check(_lib.load().ft_auto_scales(int(width), int(height), C.byref(out)))
    return out.value


FLO_MAGIC = 202021.25  # Middlebury .flo tag ("PIEH" as little-endian float)


def flow_energy(prev: Frame, curr: Frame, field: MotionField,
                params: FlowParams = FlowParams()) -> float:
    """TV-L1 objective of `field` for a frame pair (optflow.py:140-144): the
    per-pixel terms come from the device (ft_flow_energy_terms, bit-exact);
    they are summed with numpy exactly as the reference sums its arrays."""
    import torch

    a, b = prev.device(), curr.device()
    fdx, fdy = field.device()
    data = torch.empty_like(a)
    s1 = torch.empty_like(a)
    s2 = torch.empty_like(a)
    _lib.check(_lib.load().ft_flow_energy_terms(
        _lib.ctx(), _lib.ptr(a), _lib.ptr(b), _lib.ptr(fdx), _lib.ptr(fdy), prev.width,
        prev.height, float(params.huber_epsilon), _lib.ptr(data), _lib.ptr(s1), _lib.ptr(s2)))
    total = params.data_weight * float(data.cpu().numpy().sum())
    for term in (s1, s2):
        total += float(term.cpu().numpy().sum())
    return total


def write_flo(field: MotionField, path) -> None:
    """Middlebury .flo: tag, width, height, then float32 (dx, dy) pairs."""
    inter = np.stack([field.dx, field.dy], axis=-1).astype(np.float32)
    with open(path, "wb") as fh:
        fh.write(np.array([FLO_MAGIC], "<f4").tobytes())
        fh.write(np.array([field.width, field.height], "<i4").tobytes())
        fh.write(inter.tobytes())


def read_flo(path) -> MotionField:
    with open(path, "rb") as fh:
        head = fh.read(12)
        if len(head) != 12:
            raise ValueError(f"{path}: truncated .flo header")
        magic = float(np.frombuffer(head[:4], "<f4")[0])
        width, height = (int(v) for v in np.frombuffer(head[4:], "<i4"))
        if abs(magic - FLO_MAGIC) > 1e-3:
            raise ValueError(f"{path}: bad .flo magic {magic}")
        body = fh.read(width * height * 8)
        if len(body) != width * height * 8:
            raise ValueError(f"{path}: truncated .flo data")
    pairs = np.frombuffer(body, "<f4").reshape(height, width, 2)
    return MotionField(width, height, pairs[..., 0].astype(np.float64),
                       pairs[..., 1].astype(np.float64))


def compute_flow(prev: Frame, curr: Frame, params: FlowParams = FlowParams(),
                 energy_trace: list | None = None) -> MotionField:
    """Coarse-to-fine TV-L1 from prev to curr (optflow.py:217-253).

    Both frames are expected to be structure-texture preprocessed.  When
    `energy_trace` is a list, the finest-scale objective after every warp is
    appended to it (optflow.py:212-213): the device writes the per-pixel
    terms after each warp and they are summed in numpy's order here.
    """
    import torch

    if (prev.width, prev.height) != (curr.width, curr.height):
        raise ValueError(f"frame sizes differ: {prev.width}x{prev.height} vs "
                         f"{curr.width}x{curr.height}")
    if prev.width < 2 or prev.height < 2:
        raise ValueError("frames must be at least 2x2")
    a = prev.device()
    b = curr.device()
    dx = torch.empty_like(a)
    dy = torch.empty_like(a)
    prm = _lib.flow_params_struct(params)
    if energy_trace is None:
        _lib.check(_lib.load().ft_compute_flow(_lib.ctx(), _lib.ptr(a), _lib.ptr(b), prev.width,
                                               prev.height, C.byref(prm), _lib.ptr(dx),
                                               _lib.ptr(dy)))
    else:
        n = prev.width * prev.height
        terms = torch.empty((params.warps_per_level, 3, n), dtype=torch.float64, device=a.device)
        _lib.check(_lib.load().ft_compute_flow_traced(
            _lib.ctx(), _lib.ptr(a), _lib.ptr(b), prev.width, prev.height, C.byref(prm),
            _lib.ptr(dx), _lib.ptr(dy), _lib.ptr(terms)))
        host = terms.cpu().numpy().reshape(params.warps_per_level, 3, prev.height, prev.width)
        for data, s1, s2 in host:  # _energy (optflow.py:127-137) summed like numpy
            total = params.data_weight * float(np.abs(data).sum())
            total += float(s1.sum())
            total += float(s2.sum())
            energy_trace.append(total)
    return MotionField(prev.width, prev.height, dx, dy, frame_index=curr.index)

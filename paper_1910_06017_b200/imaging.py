"""Frames, Gaussian pyramids, level selection and structure-texture
preprocessing on the B200 (drop-in for reference imaging.py).

Frame data lives on the device (float64, row-major); `.data` returns a
read-only host copy on demand, like the reference's read-only ndarray
(imaging.py:43).  Compute goes through libomnitrack (ft_build_pyramid,
ft_structure_texture); there is no host fallback.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

MAX_LEVEL_DIM = 1280  # imaging.py:19
BT601_WEIGHTS = (0.299, 0.587, 0.114)  # imaging.py:21


def _torch():
    import torch
    return torch


class Frame:
    """Single-channel luminance image in [0, 1] (reference imaging.py:24-56).

    `data` may be a numpy array (validated like the reference: shape,
    finiteness, range) or a CUDA float64 tensor produced by this package.
    """

    __slots__ = ("width", "height", "index", "_host", "_dev")

    def __init__(self, width: int, height: int, index: int, data):
        object.__setattr__(self, "width", int(width))
        object.__setattr__(self, "height", int(height))
        object.__setattr__(self, "index", int(index))
        torch = None
        if not isinstance(data, np.ndarray) and type(data).__module__.startswith("torch"):
            torch = _torch()
        if torch is not None:
            if tuple(data.shape) != (self.height, self.width):
                raise ValueError(f"frame data shape {tuple(data.shape)} does not match "
                                 f"{self.height}x{self.width}")
            dev = data.to(torch.float64).contiguous()
            if not dev.is_cuda:
                dev = dev.cuda()
            # the reference validates every Frame (imaging.py:33-44): same
            # checks on the device (one reduction, one 4-byte read back)
            bad = _lib.check_plane(dev, 0.0, 1.0)
            if bad & 1:
                raise ValueError("frame contains non-finite values")
            if bad & 2:
                raise ValueError("frame values must lie in [0, 1]")
            object.__setattr__(self, "_dev", dev)
            object.__setattr__(self, "_host", None)
            return
        arr = np.ascontiguousarray(data, dtype=np.float64)
        if arr.shape != (self.height, self.width):
            raise ValueError(f"frame data shape {arr.shape} does not match "
                             f"{self.height}x{self.width}")
        if not np.all(np.isfinite(arr)):
            raise ValueError("frame contains non-finite values")
        if arr.size and (arr.min() < 0.0 or arr.max() > 1.0):
            raise ValueError("frame values must lie in [0, 1]")
        if arr is data:
            arr = arr.copy()
        arr.setflags(write=False)
        object.__setattr__(self, "_host", arr)
        object.__setattr__(self, "_dev", None)

    def __setattr__(self, name, value):
        raise AttributeError("Frame is immutable")

    @property
    def data(self) -> np.ndarray:
        if self._host is None:
            arr = self._dev.cpu().numpy()
            arr.setflags(write=False)
            object.__setattr__(self, "_host", arr)
        return self._host

    def device(self):
        """The frame as a contiguous CUDA float64 tensor (uploaded once)."""
        if self._dev is None:
            torch = _torch()
            object.__setattr__(self, "_dev", torch.from_numpy(np.array(self._host)).cuda())
        return self._dev

    @classmethod
    def from_array(cls, data, index: int = 0) -> "Frame":
        data = np.asarray(data, dtype=np.float64)
        return cls(width=data.shape[1], height=data.shape[0], index=index, data=data)

    @classmethod
    def from_gray8(cls, data, index: int = 0) -> "Frame":
        """u8 luma divided by 255 on the device (imaging.py:52-56)."""
        torch = _torch()
        u8 = np.ascontiguousarray(data, dtype=np.uint8)
        h, w = u8.shape
        src = torch.from_numpy(u8 if u8.flags.writeable else u8.copy()).cuda()
        dst = torch.empty((h, w), dtype=torch.float64, device=src.device)
        _lib.check(_lib.load().ft_gray8_to_unit(_lib.ctx(), _lib.ptr(src), w, h, _lib.ptr(dst)))
        return cls(width=w, height=h, index=index, data=dst)


class Pyramid:
    """Gaussian pyramid; level 0 is the input frame (imaging.py:59-66)."""

    __slots__ = ("levels",)

    def __init__(self, levels):
        object.__setattr__(self, "levels", tuple(levels))

    def __len__(self) -> int:
        return len(self.levels)


def rgb_to_luma(rgb: np.ndarray) -> np.ndarray:
    """BT.601 luma of an (H, W, 3) array (imaging.py:69-72; host ingest helper)."""
    wr, wg, wb = BT601_WEIGHTS
    return wr * rgb[..., 0] + wg * rgb[..., 1] + wb * rgb[..., 2]


def level_sizes(width: int, height: int, num_levels: int):
    sizes = [(width, height)]
    for _ in range(1, num_levels):
        w, h = sizes[-1]
        sizes.append((w // 2, h // 2))
    return sizes


def build_pyramid(frame: Frame, num_levels: int) -> Pyramid:
    """5-tap binomial blur + decimate by 2 per level on the device
    (imaging.py:75-95); rejects a coarsest level below 2x2."""
    torch = _torch()
    if num_levels < 1:
        raise ValueError("num_levels must be >= 1")
    sizes = level_sizes(frame.width, frame.height, num_levels)
    for lvl, (w, h) in enumerate(sizes[1:], start=1):
        if w < 2 or h < 2:
            raise ValueError(f"pyramid level {lvl} would be {w}x{h}; at least 2x2 required")
    src = frame.device()
    total = sum(w * h for w, h in sizes)
    buf = torch.empty(total, dtype=torch.float64, device=src.device)
    _lib.check(_lib.load().ft_build_pyramid(_lib.ctx(), _lib.ptr(src), frame.width,
                                            frame.height, num_levels, _lib.ptr(buf)))
    levels, off = [frame], sizes[0][0] * sizes[0][1]
    for w, h in sizes[1:]:
        levels.append(Frame(w, h, frame.index, buf[off:off + w * h].view(h, w)))
        off += w * h
    return Pyramid(levels)


def select_level(width: int, height: int) -> int:
    """Smallest L with max(W, H) / 2^L <= 1280 (imaging.py:98-106)."""
    out = C.c_int()
    _lib.check(_lib.load().ft_select_level(int(width), int(height), C.byref(out)))
    return out.value


def rof_denoise(img, weight: float, iterations: int, step: float = 0.25) -> np.ndarray:
    """TV smoothing by dual projected gradient (imaging.py:109-125); returns
    the structure image as a host array like the reference."""
    torch = _torch()
    if weight <= 0:
        raise ValueError("weight must be positive")
    src = img.device() if isinstance(img, Frame) else \
        torch.from_numpy(np.ascontiguousarray(img, dtype=np.float64)).cuda()
    h, w = src.shape
    out = torch.empty_like(src)
    _lib.check(_lib.load().ft_rof_denoise(_lib.ctx(), _lib.ptr(src), w, h, float(weight),
                                          int(iterations), float(step), _lib.ptr(out)))
    return out.cpu().numpy()


def structure_texture(frame: Frame, smoothing_weight: float = 12.0, blend: float = 0.05,
                      iterations: int = 40) -> Frame:
    """ROF structure-texture decomposition, texture + blend*structure mapped
    to [0, 1] (imaging.py:128-144), on the device."""
    torch = _torch()
    if not 0.0 <= blend <= 1.0:
        raise ValueError("blend must lie in [0, 1]")
    if smoothing_weight <= 0:
        raise ValueError("weight must be positive")
    src = frame.device()
    out = torch.empty_like(src)
    _lib.check(_lib.load().ft_structure_texture(
        _lib.ctx(), _lib.ptr(src), frame.width, frame.height, float(smoothing_weight),
        float(blend), int(iterations), _lib.ptr(out)))
    return Frame(frame.width, frame.height, frame.index, out)

"""Frame ingest for the tracker (drop-in for reference video_io.py; SURVEY
section 8 f2): binary PGM/PPM files, directories of them, and YUV4MPEG2
luma.  Decoding stays on the host (it is byte parsing); decoded frames go to
the device through Frame.from_gray8 (the u8/255 kernel), or straight into
Tracker staging via the `iter_*_u8` generators.
"""
from __future__ import annotations

import re
from dataclasses import dataclass
from pathlib import Path
from typing import Iterator

import numpy as np

from .imaging import Frame, rgb_to_luma


class FormatError(ValueError):
    """Unparseable image / stream file (message carries the path)."""


_PNM_HEADER = re.compile(rb"\A(P[56])(?:\s|#[^\n]*\n)+(\d+)(?:\s|#[^\n]*\n)+(\d+)"
                         rb"(?:\s|#[^\n]*\n)+(\d+)\s")


def _parse_pnm(blob: bytes, path):
    """(magic, width, height, maxval, pixel offset) of a binary PNM."""
    m = _PNM_HEADER.match(blob)
    if not m:
        magic = blob[:2]
        if magic not in (b"P5", b"P6"):
            raise FormatError(f"{path}: not a binary PGM/PPM file (magic {magic!r})")
        raise FormatError(f"{path}: malformed header")
    magic, w, h, maxval = m.group(1), int(m.group(2)), int(m.group(3)), int(m.group(4))
    if w <= 0 or h <= 0:
        raise FormatError(f"{path}: invalid dimensions {w}x{h}")
    if not 0 < maxval <= 255:
        raise FormatError(f"{path}: only 8-bit data supported (maxval {maxval})")
    return magic, w, h, m.end()


def read_pgm(path) -> np.ndarray:
    """uint8 luma of a P5 PGM; a P6 PPM is reduced with BT.601 weights."""
    blob = Path(path).read_bytes()
    magic, w, h, off = _parse_pnm(blob, path)
    chans = 1 if magic == b"P5" else 3
    need = w * h * chans
    pix = blob[off:off + need]
    if len(pix) != need:
        raise FormatError(f"{path}: truncated pixel data ({len(pix)} of {need} bytes)")
    arr = np.frombuffer(pix, dtype=np.uint8)
    if chans == 1:
        return arr.reshape(h, w)
    rgb = arr.reshape(h, w, 3).astype(np.float64)
    return np.clip(np.rint(rgb_to_luma(rgb)), 0, 255).astype(np.uint8)


def write_pgm(path, img) -> None:
    """Binary P5 PGM from uint8 data, or from [0,1] floats scaled by 255."""
    a = np.asarray(img)
    if a.dtype != np.uint8:
        a = np.clip(np.rint(a * 255.0), 0, 255).astype(np.uint8)
    rows, cols = a.shape
    Path(path).write_bytes(b"P5\n%d %d\n255\n" % (cols, rows) + np.ascontiguousarray(a).tobytes())


def read_frame(path, index: int = 0) -> Frame:
    return Frame.from_gray8(read_pgm(path), index=index)


def _pnm_files(path) -> list:
    folder = Path(path)
    files = sorted(p for p in folder.iterdir() if p.suffix.lower() in (".pgm", ".ppm"))
    if not files:
        raise FormatError(f"{folder}: no .pgm/.ppm files found")
    return files


def iter_pgm_dir_u8(path) -> Iterator[np.ndarray]:
    for p in _pnm_files(path):
        yield read_pgm(p)


def iter_pgm_dir(path) -> Iterator[Frame]:
    """Frames of a directory of .pgm/.ppm files, lexicographic order."""
    for k, p in enumerate(_pnm_files(path)):
        yield read_frame(p, index=k)


@dataclass(frozen=True)
class _Y4MHeader:
    width: int
    height: int
    chroma_bytes: int


def _y4m_header(line: bytes, path) -> _Y4MHeader:
    if not line.startswith(b"YUV4MPEG2"):
        raise FormatError(f"{path}: missing YUV4MPEG2 signature")
    tags = {f[:1]: f[1:] for f in line.split()[1:]}
    w = int(tags[b"W"]) if b"W" in tags else 0
    h = int(tags[b"H"]) if b"H" in tags else 0
    if not w or not h:
        raise FormatError(f"{path}: stream header lacks W/H")
    cs = tags.get(b"C", b"420").decode("ascii")
    cw, ch = (w + 1) // 2, (h + 1) // 2
    sizes = {"420": 2 * cw * ch, "420jpeg": 2 * cw * ch, "420paldv": 2 * cw * ch,
             "420mpeg2": 2 * cw * ch, "422": 2 * cw * h, "444": 2 * w * h, "mono": 0}
    if cs not in sizes:
        raise FormatError(f"{path}: unsupported colorspace C{cs}")
    return _Y4MHeader(w, h, sizes[cs])


def iter_y4m_u8(path) -> Iterator[np.ndarray]:
    """uint8 luma planes of a YUV4MPEG2 stream (chroma skipped)."""
    with open(path, "rb") as fh:
        hdr = _y4m_header(fh.readline(), path)
        n_luma = hdr.width * hdr.height
        k = 0
        while True:
            marker = fh.readline()
            if not marker:
                return
            if not marker.startswith(b"FRAME"):
                raise FormatError(f"{path}: bad frame marker at frame {k}")
            luma = fh.read(n_luma)
            if len(luma) != n_luma:
                raise FormatError(f"{path}: truncated frame {k}")
            if len(fh.read(hdr.chroma_bytes)) != hdr.chroma_bytes:
                raise FormatError(f"{path}: truncated chroma in frame {k}")
            yield np.frombuffer(luma, dtype=np.uint8).reshape(hdr.height, hdr.width)
            k += 1


def iter_y4m(path) -> Iterator[Frame]:
    for k, luma in enumerate(iter_y4m_u8(path)):
        yield Frame.from_gray8(luma, index=k)


def write_y4m(path, frames_u8, fps: int = 25) -> None:
    """Mono YUV4MPEG2 writer (test fixtures and synthetic exports)."""
    frames_u8 = list(frames_u8)
    h, w = frames_u8[0].shape
    with open(path, "wb") as fh:
        fh.write(b"YUV4MPEG2 W%d H%d F%d:1 Ip A1:1 Cmono\n" % (w, h, fps))
        for f in frames_u8:
            fh.write(b"FRAME\n" + np.ascontiguousarray(f, dtype=np.uint8).tobytes())


def load_frames(path) -> Iterator[Frame]:
    """A directory of PGMs, a .y4m stream, or a single .pgm/.ppm file."""
    p = Path(path)
    if p.is_dir():
        return iter_pgm_dir(p)
    if p.suffix.lower() == ".y4m":
        return iter_y4m(p)
    if p.suffix.lower() in (".pgm", ".ppm"):
        return iter([read_frame(p)])
    raise FormatError(f"{path}: expected a directory of PGM files or a .y4m stream")

"""CPU oracle for the OmniTrack tracking hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference `flowtrack` package's
per-frame path (pyramid -> ROF structure-texture -> TV-L1 flow -> mean-box
predict -> IoU/Hungarian match -> update) plus the `step` composition the
reference leaves to its absent pipeline module.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import it, and only as the checker or the timed CPU baseline.  The
product path (paper_1910_06017_b200) never imports it and fails loudly when
its CUDA library is missing.

Parity pin: every function below is checked bit-for-bit against fixtures
produced by the live reference (tests/golden/make_golden.py, numpy 2.3.5)
in tests/test_oracle.py.  Floating-point operation order follows the
reference line by line so the restatement is bit-identical, not merely close.

Citations are `file:line` relative to /root/reference/pkg/src/flowtrack/.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

# --------------------------------------------------------------------------
# constants (imaging.py:19, optflow.py:26, optflow.py:31, assoc.py:18)
# --------------------------------------------------------------------------
LEVEL_DIM_LIMIT = 1280
COARSE_MIN = 16
INTENSITY = 255.0
FORBIDDEN = 1e6
TAPS = (1.0 / 16.0, 4.0 / 16.0, 6.0 / 16.0, 4.0 / 16.0, 1.0 / 16.0)  # imageops.py:9

ACTIVE, LOST = "active", "lost"


# --------------------------------------------------------------------------
# grid primitives
# --------------------------------------------------------------------------
def _mirror_index(n: int, pad: int) -> np.ndarray:
    """Indices of a 'symmetric' (edge-duplicating) pad of width `pad`."""
    idx = np.arange(-pad, n + pad)
    idx = np.where(idx < 0, -idx - 1, idx)
    idx = np.where(idx >= n, 2 * n - 1 - idx, idx)
    return idx


def blur5(img: np.ndarray) -> np.ndarray:
    """5-tap binomial blur, rows then columns (imageops.py:12-23).

    Each pass accumulates tap 0..4 in order starting from 0.0, exactly like
    the reference's `out += k * shifted` loop.
    """
    h, w = img.shape
    cols = _mirror_index(w, 2)
    tmp = np.zeros_like(img)
    for k in range(5):
        tmp = tmp + TAPS[k] * img[:, cols[k:k + w]]
    rows = _mirror_index(h, 2)
    out = np.zeros_like(img)
    for k in range(5):
        out = out + TAPS[k] * tmp[rows[k:k + h], :]
    return out


def halve(img: np.ndarray) -> np.ndarray:
    """Even-sample decimation to floor-halved size (imageops.py:26-29)."""
    h, w = img.shape
    return img[0:(h // 2) * 2:2, 0:(w // 2) * 2:2]


def grad_fwd(a: np.ndarray):
    """Forward differences, zero last column/row (imageops.py:32-38)."""
    gx = np.zeros_like(a)
    gy = np.zeros_like(a)
    gx[:, :-1] = a[:, 1:] - a[:, :-1]
    gy[:-1, :] = a[1:, :] - a[:-1, :]
    return gx, gy


def div_bwd(px: np.ndarray, py: np.ndarray) -> np.ndarray:
    """Backward-difference divergence (imageops.py:41-50).

    d = dx + dy where dx uses px[c] - px[c-1] inside, px[0] at c=0 and
    -px[w-2] at c=w-1; dy likewise down the rows.
    """
    dx = np.empty_like(px)
    dx[:, 0] = px[:, 0]
    dx[:, 1:-1] = px[:, 1:-1] - px[:, :-2]
    dx[:, -1] = -px[:, -2]
    dy = np.empty_like(py)
    dy[0, :] = py[0, :]
    dy[1:-1, :] = py[1:-1, :] - py[:-2, :]
    dy[-1, :] = -py[-2, :]
    return dx + dy


def central_grad(a: np.ndarray):
    """np.gradient with unit spacing, first-order edges (optflow.py:155)."""
    gx = np.empty_like(a)
    gy = np.empty_like(a)
    gx[:, 1:-1] = (a[:, 2:] - a[:, :-2]) / 2.0
    gx[:, 0] = (a[:, 1] - a[:, 0]) / 1.0
    gx[:, -1] = (a[:, -1] - a[:, -2]) / 1.0
    gy[1:-1, :] = (a[2:, :] - a[:-2, :]) / 2.0
    gy[0, :] = (a[1, :] - a[0, :]) / 1.0
    gy[-1, :] = (a[-1, :] - a[-2, :]) / 1.0
    return gx, gy


def sample(img: np.ndarray, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Clamped bilinear lookup (imageops.py:53-66)."""
    h, w = img.shape
    xc = np.minimum(np.maximum(x, 0.0), w - 1.0)
    yc = np.minimum(np.maximum(y, 0.0), h - 1.0)
    xf = np.floor(xc)
    yf = np.floor(yc)
    ix0 = xf.astype(np.intp)
    iy0 = yf.astype(np.intp)
    ix1 = np.minimum(ix0 + 1, w - 1)
    iy1 = np.minimum(iy0 + 1, h - 1)
    ax = xc - ix0
    ay = yc - iy0
    upper = img[iy0, ix0] * (1.0 - ax) + img[iy0, ix1] * ax
    lower = img[iy1, ix0] * (1.0 - ax) + img[iy1, ix1] * ax
    return upper * (1.0 - ay) + lower * ay


def resample(img: np.ndarray, new_w: int, new_h: int) -> np.ndarray:
    """Pixel-centre bilinear resize (imageops.py:69-75)."""
    h, w = img.shape
    xs = (np.arange(new_w) + 0.5) * (w / new_w) - 0.5
    ys = (np.arange(new_h) + 0.5) * (h / new_h) - 0.5
    return sample(img, xs[None, :].repeat(new_h, 0), ys[:, None].repeat(new_w, 1))


def median9(a: np.ndarray) -> np.ndarray:
    """3x3 median with replicated border (imageops.py:78-84): the 5th order
    statistic of the 9 neighbours, an exact selection."""
    h, w = a.shape
    p = np.pad(a, 1, mode="edge")
    nb = np.stack([p[r:r + h, c:c + w] for r in range(3) for c in range(3)])
    nb.sort(axis=0)
    return nb[4].copy()


def rha(v: float) -> float:
    """Round half away from zero (imageops.py:87-90)."""
    return math.floor(v + 0.5) if v >= 0.0 else math.ceil(v - 0.5)


# --------------------------------------------------------------------------
# imaging
# --------------------------------------------------------------------------
def gray8_to_unit(u8: np.ndarray) -> np.ndarray:
    """u8 luma -> [0,1] float64 by division by 255 (imaging.py:52-56)."""
    return np.asarray(u8, dtype=np.float64) / 255.0


def pyramid(img: np.ndarray, levels: int) -> list:
    """Blur+decimate chain (imaging.py:75-95), with the 2x2 floor check."""
    if levels < 1:
        raise ValueError("num_levels must be >= 1")
    h, w = img.shape
    for lvl in range(1, levels):
        w //= 2
        h //= 2
        if w < 2 or h < 2:
            raise ValueError(
                f"pyramid level {lvl} would be {w}x{h}; at least 2x2 required")
    out = [img]
    for _ in range(1, levels):
        out.append(halve(blur5(out[-1])))
    return out


def select_level(width: int, height: int) -> int:
    """Smallest L with max(W,H)/2^L <= 1280 (imaging.py:98-106)."""
    if width < 2 or height < 2:
        raise ValueError("frame must be at least 2x2")
    lvl = 0
    while float(max(width, height)) / (1 << lvl) > LEVEL_DIM_LIMIT:
        lvl += 1
    return lvl


def rof(img: np.ndarray, weight: float, iterations: int, step: float = 0.25):
    """Dual projected-gradient ROF (imaging.py:109-125)."""
    if weight <= 0:
        raise ValueError("weight must be positive")
    px = np.zeros_like(img)
    py = np.zeros_like(img)
    for _ in range(iterations):
        gx, gy = grad_fwd(div_bwd(px, py) - img / weight)
        den = 1.0 + step * np.hypot(gx, gy)
        px = (px + step * gx) / den
        py = (py + step * gy) / den
    return img - weight * div_bwd(px, py)


def structure_texture(img: np.ndarray, weight: float = 12.0,
                      blend: float = 0.05, iterations: int = 40):
    """Texture + blend*structure remapped to [0,1] (imaging.py:128-144)."""
    if not 0.0 <= blend <= 1.0:
        raise ValueError("blend must lie in [0, 1]")
    s = rof(img, weight, iterations)
    mix = (img - s) + blend * s
    mix = (mix + (1.0 - blend)) / (2.0 - blend)
    return np.clip(mix, 0.0, 1.0)


# --------------------------------------------------------------------------
# TV-L1 flow
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class FlowParams:
    """Solver parameters (optflow.py:36-66)."""
    data_weight: float = 0.15
    huber_epsilon: float = 0.01
    time_step: float = 0.25
    warps_per_level: int = 5
    iterations_per_warp: int = 50
    pyramid_scales: int | None = None


def auto_scales(width: int, height: int) -> int:
    """Deepest pyramid whose coarsest sides stay >= 16 (optflow.py:96-104)."""
    n, w, h = 1, width, height
    while min(w // 2, h // 2) >= COARSE_MIN:
        w, h, n = w // 2, h // 2, n + 1
    return n


def tvl1_level(i0, i1, u1, u2, prm: FlowParams):
    """Warps x iterations of the primal-dual solver on one scale
    (optflow.py:147-214)."""
    h, w = i0.shape
    yy, xx = np.meshgrid(np.arange(h, dtype=np.float64),
                         np.arange(w, dtype=np.float64), indexing="ij")
    lam, tau = prm.data_weight, prm.time_step
    sigma = 1.0 / (8.0 * tau)
    shrink = 1.0 / (1.0 + sigma * prm.huber_epsilon)
    tl = tau * lam
    ix, iy = central_grad(i1)
    for _ in range(prm.warps_per_level):
        mx = xx + u1
        my = yy + u2
        i1w = sample(i1, mx, my)
        gx = sample(ix, mx, my)
        gy = sample(iy, mx, my)
        g2 = gx * gx + gy * gy
        ok = g2 > 1e-12
        ig2 = np.where(ok, 1.0 / np.maximum(g2, 1e-12), 0.0)
        r0 = i1w - i0 - gx * u1 - gy * u2
        thr = tl * g2
        p11 = np.zeros_like(u1); p12 = np.zeros_like(u1)
        p21 = np.zeros_like(u1); p22 = np.zeros_like(u1)
        b1, b2 = u1, u2
        for _ in range(prm.iterations_per_warp):
            a1x, a1y = grad_fwd(b1)
            a2x, a2y = grad_fwd(b2)
            p11 = (p11 + sigma * a1x) * shrink
            p12 = (p12 + sigma * a1y) * shrink
            p21 = (p21 + sigma * a2x) * shrink
            p22 = (p22 + sigma * a2y) * shrink
            n1 = np.maximum(1.0, np.hypot(p11, p12))
            n2 = np.maximum(1.0, np.hypot(p21, p22))
            p11 = p11 / n1; p12 = p12 / n1
            p21 = p21 / n2; p22 = p22 / n2
            v1 = u1 + tau * div_bwd(p11, p12)
            v2 = u2 + tau * div_bwd(p21, p22)
            rho = r0 + gx * v1 + gy * v2
            lo = rho < -thr
            hi = rho > thr
            d = np.where(lo, tl, np.where(hi, -tl, -rho * ig2))
            d = np.where(ok | lo | hi, d, 0.0)
            n1u = v1 + d * gx
            n2u = v2 + d * gy
            b1 = 2.0 * n1u - u1
            b2 = 2.0 * n2u - u2
            u1, u2 = n1u, n2u
        u1 = median9(u1)
        u2 = median9(u2)
    return u1, u2


def compute_flow(prev: np.ndarray, curr: np.ndarray,
                 prm: FlowParams = FlowParams()):
    """Coarse-to-fine TV-L1 (optflow.py:217-253); returns (dx, dy)."""
    if prev.shape != curr.shape:
        raise ValueError(f"frame sizes differ: {prev.shape} vs {curr.shape}")
    h, w = prev.shape
    if w < 2 or h < 2:
        raise ValueError("frames must be at least 2x2")
    s = prm.pyramid_scales if prm.pyramid_scales is not None else auto_scales(w, h)
    pa = pyramid(prev, s)
    pb = pyramid(curr, s)
    u1 = np.zeros(pa[-1].shape)
    u2 = np.zeros_like(u1)
    for lvl in range(s - 1, -1, -1):
        i0 = pa[lvl] * INTENSITY
        i1 = pb[lvl] * INTENSITY
        if lvl != s - 1:
            hh, ww = i0.shape
            fx = ww / u1.shape[1]
            fy = hh / u1.shape[0]
            u1 = resample(u1, ww, hh) * fx
            u2 = resample(u2, ww, hh) * fy
        u1, u2 = tvl1_level(i0, i1, u1, u2, prm)
    return u1, u2


# --------------------------------------------------------------------------
# box mean with numpy's exact summation order (track.py:82-83)
# --------------------------------------------------------------------------
def _pairwise(vals) -> float:
    """numpy's pairwise_sum for a contiguous run (<8 sequential, <=128 eight
    lanes, else split at n/2 rounded down to a multiple of 8)."""
    n = len(vals)
    if n < 8:
        acc = 0.0
        for v in vals:
            acc += float(v)
        return acc
    if n <= 128:
        lane = [float(v) for v in vals[:8]]
        i = 8
        stop = n - (n % 8)
        while i < stop:
            for j in range(8):
                lane[j] += float(vals[i + j])
            i += 8
        acc = ((lane[0] + lane[1]) + (lane[2] + lane[3])) + \
              ((lane[4] + lane[5]) + (lane[6] + lane[7]))
        while i < n:
            acc += float(vals[i])
            i += 1
        return acc
    half = n // 2
    half -= half % 8
    return _pairwise(vals[:half]) + _pairwise(vals[half:])


def window_mean(plane: np.ndarray, top: int, bottom: int, left: int,
                right: int) -> float:
    """`plane[top:bottom, left:right].mean()` reproduced bit-exactly for
    numpy 2.3: a contiguous window is one pairwise run; otherwise the
    reduction iterator buffers floor(8192/width) whole rows at a time and
    adds each buffer's pairwise sum to a 0.0 accumulator."""
    hh, ww = bottom - top, right - left
    flat = plane[top:bottom, left:right].ravel()
    if hh == 1 or ww == plane.shape[1]:
        total = _pairwise(flat)
    else:
        chunk = (8192 // ww) * ww
        total = 0.0
        for i in range(0, flat.size, chunk):
            total += _pairwise(flat[i:i + chunk])
    return total / float(hh * ww)


# --------------------------------------------------------------------------
# tracks, matching, update
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Det:
    class_id: int
    label: str
    score: float
    box: tuple


@dataclass(frozen=True)
class Track:
    id: int
    class_id: int
    label: str
    box: tuple
    state: str = ACTIVE
    born_at: int = 0
    last_seen: int = 0
    score: float = 1.0
    lost_at: int | None = None


def predict(tracks, dx: np.ndarray, dy: np.ndarray, level: int, frame_wh):
    """Mean-flow box shift (track.py:56-87); None when support is empty."""
    s = float(2 ** level)
    fw, fh = frame_wh
    fh_l, fw_l = dx.shape
    res = []
    for t in tracks:
        if t.state != ACTIVE:
            raise ValueError(f"cannot predict lost object {t.id}")
        x, y, w, h = t.box
        l = max(int(rha(x / s)), 0)
        tp = max(int(rha(y / s)), 0)
        r = min(int(rha((x + w) / s)), fw_l)
        b = min(int(rha((y + h) / s)), fh_l)
        if r <= l or b <= tp:
            res.append(None)
            continue
        sx = window_mean(dx, tp, b, l, r) * s
        sy = window_mean(dy, tp, b, l, r) * s
        nx = min(max(x + sx, 0.0), max(float(fw) - w, 0.0))
        ny = min(max(y + sy, 0.0), max(float(fh) - h, 0.0))
        res.append((nx, ny, w, h))
    return res


def iou(a, b) -> float:
    """Continuous-area IoU of (x,y,w,h) boxes (assoc.py:30-41)."""
    ax, ay, aw, ah = a
    bx, by, bw, bh = b
    if aw <= 0 or ah <= 0 or bw <= 0 or bh <= 0:
        raise ValueError("boxes must have positive width and height")
    iw = max(0.0, min(ax + aw, bx + bw) - max(ax, bx))
    ih = max(0.0, min(ay + ah, by + bh) - max(ay, by))
    inter = iw * ih
    return inter / (aw * ah + bw * bh - inter)


def lsap_rows_le_cols(c: np.ndarray):
    """Shortest augmenting path LSAP, rows <= cols (assoc.py:44-81)."""
    m, n = c.shape
    u = np.zeros(m)
    v = np.zeros(n + 1)
    own = np.full(n + 1, -1, dtype=np.intp)
    for row in range(m):
        own[n] = row
        j0 = n
        best = np.full(n, np.inf)
        via = np.full(n, n, dtype=np.intp)
        seen = np.zeros(n + 1, dtype=bool)
        while True:
            seen[j0] = True
            r = own[j0]
            sl = c[r, :] - u[r] - v[:n]
            imp = ~seen[:n] & (sl < best)
            best[imp] = sl[imp]
            via[imp] = j0
            cand = np.where(seen[:n], np.inf, best)
            j1 = int(np.argmin(cand))
            delta = cand[j1]
            for j in np.flatnonzero(seen):
                u[own[j]] += delta
                v[j] -= delta
            best[~seen[:n]] -= delta
            j0 = j1
            if own[j0] == -1:
                break
        while j0 != n:
            jp = via[j0]
            own[j0] = own[jp]
            j0 = jp
    return [(int(own[j]), j) for j in range(n) if own[j] != -1]


def hungarian(cost, forbidden=None):
    """Min-cost assignment with transpose for tall matrices and removal of
    forbidden cells (assoc.py:84-106)."""
    c = np.asarray(cost, dtype=np.float64)
    if c.ndim != 2:
        raise ValueError("cost must be a 2-D matrix")
    if c.size == 0:
        return []
    if not np.all(np.isfinite(c)):
        raise ValueError("costs must be finite")
    if c.shape[0] <= c.shape[1]:
        pairs = lsap_rows_le_cols(c)
    else:
        pairs = [(i, j) for j, i in lsap_rows_le_cols(c.T)]
    pairs.sort()
    if forbidden is not None:
        pairs = [(i, j) for i, j in pairs if c[i, j] < forbidden]
    return pairs


def gate_cost(tracks, dets, gate: float = 0.3):
    """IoU score and gated cost matrices (assoc.py:119-126)."""
    m, n = len(tracks), len(dets)
    sc = np.zeros((m, n))
    cost = np.full((m, n), FORBIDDEN)
    for i, t in enumerate(tracks):
        for j, d in enumerate(dets):
            s = iou(t.box, d.box)
            sc[i, j] = s
            if s >= gate and t.class_id == d.class_id:
                cost[i, j] = 1.0 - s
    return sc, cost


def match(tracks, dets, gate: float = 0.3):
    """Returns (pairs[(i,j,iou)], unmatched_tracks, unmatched_dets)
    (assoc.py:109-135)."""
    m, n = len(tracks), len(dets)
    if m == 0 or n == 0:
        return (), tuple(range(m)), tuple(range(n))
    sc, cost = gate_cost(tracks, dets, gate)
    pairs = hungarian(cost, forbidden=FORBIDDEN)
    mi = {i for i, _ in pairs}
    mj = {j for _, j in pairs}
    return (tuple((i, j, float(sc[i, j])) for i, j in pairs),
            tuple(i for i in range(m) if i not in mi),
            tuple(j for j in range(n) if j not in mj))


def update(tracks, pairs, dets, t: int, blend: float = 1.0):
    """Lifecycle update (track.py:90-139)."""
    by_track = {}
    used = set()
    for i, j, _ in pairs:
        if not 0 <= i < len(tracks):
            raise IndexError(f"scene index {i} out of range")
        if not 0 <= j < len(dets):
            raise IndexError(f"detection index {j} out of range")
        by_track[i] = j
        used.add(j)
    nid = max((o.id for o in tracks), default=-1) + 1
    out = []
    for i, o in enumerate(tracks):
        if i in by_track:
            if o.state != ACTIVE:
                raise ValueError(f"lost object {o.id} appeared in the assignment")
            d = dets[by_track[i]]
            if blend >= 1.0:
                bx = d.box
            else:
                bx = tuple(blend * dv + (1.0 - blend) * ov
                           for dv, ov in zip(d.box, o.box))
            out.append(replace(o, box=tuple(float(v) for v in bx),
                               score=d.score, last_seen=t))
        elif o.state == ACTIVE:
            out.append(replace(o, state=LOST, lost_at=t))
        else:
            out.append(o)
    for j, d in enumerate(dets):
        if j in used:
            continue
        out.append(Track(id=nid, class_id=d.class_id, label=d.label,
                         box=tuple(float(v) for v in d.box), state=ACTIVE,
                         born_at=t, last_seen=t, score=d.score))
        nid += 1
    return out


# --------------------------------------------------------------------------
# per-frame step
# --------------------------------------------------------------------------
@dataclass
class StreamState:
    tracks: list = field(default_factory=list)
    prev_st: np.ndarray | None = None


def step(state: StreamState, luma_u8: np.ndarray, t: int, dets,
         prm: FlowParams = FlowParams(), gate: float = 0.3,
         min_score: float = 0.5):
    """Frame in, tracks out.  `dets is None` means no detector result for
    this frame (coast).  Mutates and returns `state`."""
    hh, ww = luma_u8.shape
    lvl = select_level(ww, hh)
    img = pyramid(gray8_to_unit(luma_u8), lvl + 1)[lvl]
    st = structure_texture(img)
    if dets is not None:
        dets = [d for d in dets if d.score >= min_score]
    if state.prev_st is None:
        if dets is not None:
            state.tracks = update([], (), dets, t)
    else:
        dx, dy = compute_flow(state.prev_st, st, prm)
        act = [i for i, o in enumerate(state.tracks) if o.state == ACTIVE]
        pred = predict([state.tracks[i] for i in act], dx, dy, lvl, (ww, hh))
        for i, p in zip(act, pred):
            if p is not None:
                state.tracks[i] = replace(state.tracks[i], box=p)
        if dets is not None:
            cand = [i for i, p in zip(act, pred) if p is not None]
            pairs, _, _ = match([state.tracks[i] for i in cand], dets, gate)
            full = tuple((cand[i], j, s) for i, j, s in pairs)
            state.tracks = update(state.tracks, full, dets, t)
    state.prev_st = st
    return state

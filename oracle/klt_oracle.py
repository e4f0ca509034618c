"""CPU oracle for the KLT / MedianFlow motion backend -- TEST INFRASTRUCTURE.

SURVEY.md section 8 f4: north_star describes pyramidal Lucas-Kanade on
per-track point grids with a forward-backward check and a median / scale
box update.  The reference (flowtrack) has no such code, so this oracle
*defines* the backend (parity is against this file, not the reference:
"parity unpinned" in the sense of SPEC), and the device implementation in
libomnitrack (k_klt.cu) must reproduce it bit for bit.  Floating-point order
is spelled out wherever it matters:

* window sums use the device order: lane k (0..31) accumulates window
  elements k, k+32, k+64, ... sequentially from 0.0, then the 32 partial
  sums are combined by an xor butterfly (offsets 16, 8, 4, 2, 1;
  s = s + partner) -- IEEE addition is commutative, so every lane ends with
  the same bits and so does this restatement;
* medians are lower medians of an exact sort (element (n-1)//2).

Algorithm (per box, frames at the tracker's processing level L):
1. a GxG grid: point (i, j) at (x/s + (i+0.5)*w/s/G, y/s + (j+0.5)*h/s/G),
   s = 2^L;
2. pyramidal LK (Bouguet) prev -> curr over KLT_LEVELS levels built with the
   same binomial pyramid as the flow path, window (2R+1)^2 sampled with one
   shared bilinear fraction per window (see `window`), central gradients of
   the source level, up to ITERS Gauss-Newton steps per level
   (stop when |eta| < EPS_STEP; the 2x2 solve multiplies by 1/det, divided
   once per level), a point is lost when the structure tensor determinant is
   < MIN_DET or it leaves the level;
3. the same tracking back curr -> prev; fb = |p_back - p|;
4. keep valid points with fb <= lower-median(fb of valid points);
5. shift = lower-median of kept dx, dy; scale = lower-median of
   |p'_a - p'_b| / |p_a - p_b| over kept pairs (a, a + K/2) in kept order,
   K = number kept (scale 1 when K < 2);
6. new box (frame pixels): centre moved by shift*s, size times scale,
   position clamped like track.predict (track.py:84-85); None when K == 0.
"""
from __future__ import annotations

import math

import numpy as np

from oracle import ftoracle as O

KLT_LEVELS = 3
R = 4                # window half size: 9x9 = 81 samples
ITERS = 10
EPS_STEP = 0.01      # px
MIN_DET = 1e-9


def lane_sum(vals) -> float:
    """Device reduction order (see module docstring)."""
    part = [0.0] * 32
    for k, v in enumerate(vals):
        part[k % 32] = part[k % 32] + float(v)
    for off in (16, 8, 4, 2, 1):
        part = [part[l] + part[l ^ off] for l in range(32)]
    return part[0]


def sample(img, x, y) -> float:
    """Clamped bilinear lookup (same formula as the flow path)."""
    return float(O.sample(img, np.array([x]), np.array([y]))[0])


_DX = np.array([e % (2 * R + 1) - R for e in range((2 * R + 1) ** 2)])
_DY = np.array([e // (2 * R + 1) - R for e in range((2 * R + 1) ** 2)])


def window(img: np.ndarray, qx: float, qy: float):
    """The (2R+1)^2 window samples around (qx, qy), element e at integer offset
    (e % (2R+1) - R, e // (2R+1) - R): the centre is clamped to the image,
    split into an integer base and a fraction shared by the whole window
    (standard KLT interpolation), and every sample is the bilinear blend of
    the four border-replicated neighbours of base + offset:
    top = a00*(1-fx) + a01*fx, bot = a10*(1-fx) + a11*fx,
    v = top*(1-fy) + bot*fy."""
    h, w = img.shape
    qx = qx if qx > 0.0 else 0.0       # comparison order of the device clamp
    qx = qx if qx < w - 1.0 else w - 1.0
    qy = qy if qy > 0.0 else 0.0
    qy = qy if qy < h - 1.0 else h - 1.0
    x0, y0 = math.floor(qx), math.floor(qy)
    fx, fy = qx - x0, qy - y0
    gx, gy = 1.0 - fx, 1.0 - fy
    c0 = np.clip(x0 + _DX, 0, w - 1)
    c1 = np.clip(x0 + _DX + 1, 0, w - 1)
    r0 = np.clip(y0 + _DY, 0, h - 1)
    r1 = np.clip(y0 + _DY + 1, 0, h - 1)
    top = img[r0, c0] * gx + img[r0, c1] * fx
    bot = img[r1, c0] * gx + img[r1, c1] * fx
    return (top * gy + bot * fy).tolist()


def lk_track(src_pyr, src_grad, dst_pyr, px: float, py: float):
    """Pyramidal LK of one point; returns (x, y, ok) at level 0 coordinates."""
    gx_, gy_ = 0.0, 0.0
    ok = True
    for lvl in range(KLT_LEVELS - 1, -1, -1):
        I, J = src_pyr[lvl], dst_pyr[lvl]
        Ix, Iy = src_grad[lvl]
        h, w = I.shape
        sc = float(1 << lvl)
        cx, cy = px / sc, py / sc
        if not (0.0 <= cx <= w - 1.0 and 0.0 <= cy <= h - 1.0):
            ok = False
            break
        ixs = window(Ix, cx, cy)
        iys = window(Iy, cx, cy)
        ivs = window(I, cx, cy)
        gxx = lane_sum([a * a for a in ixs])
        gxy = lane_sum([a * b for a, b in zip(ixs, iys)])
        gyy = lane_sum([b * b for b in iys])
        det = gxx * gyy - gxy * gxy
        if not det >= MIN_DET:
            ok = False
            break
        idet = 1.0 / det  # once per level; the steps multiply by it
        vx, vy = 0.0, 0.0
        for _ in range(ITERS):
            qx, qy = cx + gx_ + vx, cy + gy_ + vy
            jv = window(J, qx, qy)
            dI = [iv - jj for iv, jj in zip(ivs, jv)]
            bx = lane_sum([d * a for d, a in zip(dI, ixs)])
            by = lane_sum([d * b for d, b in zip(dI, iys)])
            ex = (gyy * bx - gxy * by) * idet
            ey = (gxx * by - gxy * bx) * idet
            vx = vx + ex
            vy = vy + ey
            if ex * ex + ey * ey < EPS_STEP * EPS_STEP:
                break
        if lvl > 0:
            gx_ = 2.0 * (gx_ + vx)
            gy_ = 2.0 * (gy_ + vy)
        else:
            gx_ = gx_ + vx
            gy_ = gy_ + vy
    qx, qy = px + gx_, py + gy_
    h0, w0 = dst_pyr[0].shape
    if ok and not (0.0 <= qx <= w0 - 1.0 and 0.0 <= qy <= h0 - 1.0):
        ok = False
    return qx, qy, ok


def klt_pyramid(img: np.ndarray):
    pyr = O.pyramid(img, KLT_LEVELS)
    grads = [O.central_grad(p) for p in pyr]
    return pyr, grads


def _hyp(a: float, b: float) -> float:
    """glibc hypot (numpy's), which the device restates exactly."""
    return float(np.hypot(a, b))


def lower_median(vals) -> float:
    s = sorted(vals)
    return s[(len(s) - 1) // 2]


def klt_predict(boxes, prev: np.ndarray, curr: np.ndarray, level: int, frame_wh,
                grid: int = 10):
    """One (x, y, w, h) or None per box; prev/curr are processing-level frames."""
    pp, pg = klt_pyramid(prev)
    cp, cg = klt_pyramid(curr)
    s = float(1 << level)
    fw, fh = frame_wh
    out = []
    for (x, y, w, h) in boxes:
        pts = []
        for j in range(grid):
            for i in range(grid):
                pts.append((x / s + (i + 0.5) * (w / s) / grid, y / s + (j + 0.5) * (h / s) / grid))
        fwd = [lk_track(pp, pg, cp, px, py) for px, py in pts]
        bwd = [lk_track(cp, cg, pp, qx, qy) if ok else (0.0, 0.0, False) for qx, qy, ok in fwd]
        valid, fb = [], []
        for k, ((px, py), (qx, qy, ok), (rx, ry, okb)) in enumerate(zip(pts, fwd, bwd)):
            if ok and okb:
                valid.append(k)
                fb.append(_hyp(rx - px, ry - py))
        if not valid:
            out.append(None)
            continue
        thr = lower_median(fb)
        kept = [k for k, e in zip(valid, fb) if e <= thr]
        dxs = [fwd[k][0] - pts[k][0] for k in kept]
        dys = [fwd[k][1] - pts[k][1] for k in kept]
        mdx, mdy = lower_median(dxs), lower_median(dys)
        K = len(kept)
        scale = 1.0
        if K >= 2:
            ratios = []
            for a in range(K - K // 2):
                b = a + K // 2
                ka, kb = kept[a], kept[b]
                d0 = _hyp(pts[kb][0] - pts[ka][0], pts[kb][1] - pts[ka][1])
                d1 = _hyp(fwd[kb][0] - fwd[ka][0], fwd[kb][1] - fwd[ka][1])
                if d0 > 0.0:
                    ratios.append(d1 / d0)
            if ratios:
                scale = lower_median(ratios)
        nw, nh = w * scale, h * scale
        cx = x + 0.5 * w + mdx * s
        cy = y + 0.5 * h + mdy * s
        nx = min(max(cx - 0.5 * nw, 0.0), max(float(fw) - nw, 0.0))
        ny = min(max(cy - 0.5 * nh, 0.0), max(float(fh) - nh, 0.0))
        out.append((nx, ny, nw, nh))
    return out


def step_klt(state, luma_u8, t: int, dets, grid: int = 10, gate: float = 0.3,
             min_score: float = 0.5):
    """ftoracle.step with the KLT backend in place of flow + mean-box
    predict: prediction runs on the processing-level frames (no
    structure-texture); matching and the lifecycle are the reference's.
    `state.prev_st` holds the previous processing-level frame."""
    from dataclasses import replace
    hh, ww = luma_u8.shape
    lvl = O.select_level(ww, hh)
    img = O.pyramid(O.gray8_to_unit(luma_u8), lvl + 1)[lvl]
    if dets is not None:
        dets = [d for d in dets if d.score >= min_score]
    if state.prev_st is None:
        if dets is not None:
            state.tracks = O.update([], (), dets, t)
    else:
        act = [i for i, o in enumerate(state.tracks) if o.state == O.ACTIVE]
        pred = klt_predict([state.tracks[i].box for i in act], state.prev_st, img, lvl,
                           (ww, hh), grid)
        for i, p in zip(act, pred):
            if p is not None:
                state.tracks[i] = replace(state.tracks[i], box=p)
        if dets is not None:
            cand = [i for i, p in zip(act, pred) if p is not None]
            pairs, _, _ = O.match([state.tracks[i] for i in cand], dets, gate)
            full = tuple((cand[i], j, s) for i, j, s in pairs)
            state.tracks = O.update(state.tracks, full, dets, t)
    state.prev_st = img
    return state

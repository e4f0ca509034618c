// KLT / MedianFlow motion backend (north_star items
// (2)-(3)): pyramidal Lucas-Kanade on a GxG point grid per box, one warp per
// point, window sums reduced with warp shuffles, forward-backward check,
// median displacement and scale ratio per box.  The reference has no such
// code; oracle/klt_oracle.py defines the algorithm and this file reproduces
// it bit for bit (same IEEE operation order, same reduction tree).
#include "ft_internal.cuh"
#include "ft_klt.cuh"

#include <cstdlib>

namespace ft {

namespace {

constexpr int kR = kKltR, kWin = (2 * kR + 1) * (2 * kR + 1);  // 81 window samples
constexpr int kPerLane = (kWin + 31) / 32;                      // 3

// lane-strided partial sum then xor butterfly (oracle: klt_oracle.lane_sum)
__device__ __forceinline__ double warp_sum(double part) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) part = part + __shfl_xor_sync(0xffffffffu, part, off);
  return part;
}

// Window sampling (klt_oracle.window): the centre is clamped to the image and
// split into an integer base and one bilinear fraction shared by the whole
// window; element e samples base + (e % 9 - 4, e / 9 - 4) with
// border-replicated neighbours.  Per-lane element offsets are precomputed.
struct WinPos {
  int x0, y0;
  double fx, fy, gx, gy;  // fraction and 1 - fraction
  bool inside;            // every tap of the window lies in the image
};

__device__ __forceinline__ WinPos win_pos(double qx, double qy, int w, int h) {
  WinPos p;
  qx = qx > 0.0 ? qx : 0.0;
  qx = qx < w - 1.0 ? qx : w - 1.0;
  qy = qy > 0.0 ? qy : 0.0;
  qy = qy < h - 1.0 ? qy : h - 1.0;
  p.x0 = (int)floor(qx);
  p.y0 = (int)floor(qy);
  p.fx = qx - (double)p.x0;
  p.fy = qy - (double)p.y0;
  p.gx = 1.0 - p.fx;
  p.gy = 1.0 - p.fy;
  p.inside = p.x0 - kR >= 0 && p.x0 + kR + 1 <= w - 1 && p.y0 - kR >= 0 && p.y0 + kR + 1 <= h - 1;
  return p;
}

__device__ __forceinline__ double win_sample(const double *__restrict__ img, int w, int h,
                                             const WinPos &p, int dx, int dy) {
  int c0 = p.x0 + dx, r0 = p.y0 + dy, c1 = c0 + 1, r1 = r0 + 1;
  if (!p.inside) {
    c0 = min(max(c0, 0), w - 1);
    c1 = min(max(c1, 0), w - 1);
    r0 = min(max(r0, 0), h - 1);
    r1 = min(max(r1, 0), h - 1);
  }
  const double *a = img + (int64_t)r0 * w, *b = img + (int64_t)r1 * w;
  const double top = a[c0] * p.gx + a[c1] * p.fx;
  const double bot = b[c0] * p.gx + b[c1] * p.fx;
  return top * p.gy + bot * p.fy;
}

// Two lane-strided partial sums reduced at once, bit-identical to two
// warp_sum butterflies: at offset 16 lanes < 16 keep the first sum and
// lanes >= 16 the second (each adds its partner's partial exactly as the
// butterfly does), the remaining offsets stay within a half, and the totals
// are read from lanes 0 and 16.
__device__ __forceinline__ void warp_sum2(double a, double b, double &sa, double &sb) {
  const bool lo = (threadIdx.x & 16) == 0;
  double v = (lo ? a : b) + __shfl_xor_sync(0xffffffffu, lo ? b : a, 16);
#pragma unroll
  for (int off = 8; off > 0; off >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, off);
  sa = __shfl_sync(0xffffffffu, v, 0);
  sb = __shfl_sync(0xffffffffu, v, 16);
}

// Pyramidal LK of one point from pyramid A to pyramid B (image `img`);
// identical on every lane of the warp.  Returns false when the point is lost.
__device__ bool lk_point(const KltPyr &A, const KltPyr &B, int img, double px, double py,
                         double &qx, double &qy) {
  const int lane = threadIdx.x & 31;
  double ga = 0.0, gb = 0.0;
  bool ok = true;
  for (int lvl = kKltLevels - 1; lvl >= 0; --lvl) {
    const int w = A.w[lvl], h = A.h[lvl];
    const int64_t o = (int64_t)img * A.stride + A.off[lvl];
    const double *I = A.lvl + o, *Ix = A.gx + o, *Iy = A.gy + o;
    const double *J = B.lvl + (int64_t)img * B.stride + B.off[lvl];
    const double sc = (double)(1 << lvl);
    const double cx = px / sc, cy = py / sc;
    if (!(0.0 <= cx && cx <= w - 1.0 && 0.0 <= cy && cy <= h - 1.0)) {
      ok = false;
      break;
    }
    double ix[kPerLane], iy[kPerLane], iv[kPerLane];
    int ox[kPerLane], oy[kPerLane];
    double pxx = 0.0, pxy = 0.0, pyy = 0.0;
    const WinPos pc = win_pos(cx, cy, w, h);
#pragma unroll
    for (int k = 0; k < kPerLane; ++k) {
      const int e = lane + 32 * k;
      ox[k] = e % (2 * kR + 1) - kR;
      oy[k] = e / (2 * kR + 1) - kR;
      ix[k] = iy[k] = iv[k] = 0.0;
      if (e < kWin) {
        ix[k] = win_sample(Ix, w, h, pc, ox[k], oy[k]);
        iy[k] = win_sample(Iy, w, h, pc, ox[k], oy[k]);
        iv[k] = win_sample(I, w, h, pc, ox[k], oy[k]);
        pxx = pxx + ix[k] * ix[k];
        pxy = pxy + ix[k] * iy[k];
        pyy = pyy + iy[k] * iy[k];
      }
    }
    double gxx, gxy;
    warp_sum2(pxx, pxy, gxx, gxy);
    const double gyy = warp_sum(pyy);
    const double det = gxx * gyy - gxy * gxy;
    if (!(det >= kKltMinDet)) {
      ok = false;
      break;
    }
    const double idet = 1.0 / det;  // once per level (klt_oracle.lk_track)
    double vx = 0.0, vy = 0.0;
    for (int it = 0; it < kKltIters; ++it) {
      const double qx_ = cx + ga + vx, qy_ = cy + gb + vy;
      const WinPos pq = win_pos(qx_, qy_, w, h);
      double bxp = 0.0, byp = 0.0;
#pragma unroll
      for (int k = 0; k < kPerLane; ++k) {
        const int e = lane + 32 * k;
        if (e < kWin) {
          const double jv = win_sample(J, w, h, pq, ox[k], oy[k]);
          const double dI = iv[k] - jv;
          bxp = bxp + dI * ix[k];
          byp = byp + dI * iy[k];
        }
      }
      double bx, by;
      warp_sum2(bxp, byp, bx, by);
      const double ex = (gyy * bx - gxy * by) * idet;
      const double ey = (gxx * by - gxy * bx) * idet;
      vx = vx + ex;
      vy = vy + ey;
      if (ex * ex + ey * ey < kKltEps * kKltEps) break;
    }
    if (lvl > 0) {
      ga = 2.0 * (ga + vx);
      gb = 2.0 * (gb + vy);
    } else {
      ga = ga + vx;
      gb = gb + vy;
    }
  }
  qx = px + ga;
  qy = py + gb;
  if (ok && !(0.0 <= qx && qx <= B.w[0] - 1.0 && 0.0 <= qy && qy <= B.h[0] - 1.0)) ok = false;
  return ok;
}

constexpr int kPtWarps = 8;

// one warp per (stream, box, point): forward LK, then backward LK from the
// forward result; writes the grid point, its forward position and the
// forward-backward error (-1 when lost either way)
template <int MINB>
__global__ void __launch_bounds__(32 * kPtWarps, MINB)
    k_klt_points(KltArgs a, const double *boxes, int64_t box_stride, const int32_t *n_boxes,
                 int n_boxes_const, double *pts, double *fwd, double *fb) {
  const int s = blockIdx.y;
  const int warp = threadIdx.x >> 5;
  const int item = blockIdx.x * kPtWarps + warp;
  const int G = a.grid, GG = G * G;
  const int nb = n_boxes ? n_boxes[s] : n_boxes_const;
  const int b = item / GG, k = item % GG;
  if (b >= nb) return;
  const double *box = boxes + ((int64_t)s * box_stride + b) * 4;
  const double sc = a.scale;
  const int i = k % G, j = k / G;
  // x/s + (i+0.5)*(w/s)/G  (oracle order)
  const double px = box[0] / sc + ((double)i + 0.5) * (box[2] / sc) / (double)G;
  const double py = box[1] / sc + ((double)j + 0.5) * (box[3] / sc) / (double)G;
  double qx, qy, rx, ry;
  bool ok = lk_point(a.prev, a.curr, s, px, py, qx, qy);
  if (ok) ok = lk_point(a.curr, a.prev, s, qx, qy, rx, ry);
  if ((threadIdx.x & 31) == 0) {
    const int64_t o = ((int64_t)s * box_stride + b) * a.max_pts + k;
    pts[2 * o] = px;
    pts[2 * o + 1] = py;
    fwd[2 * o] = qx;
    fwd[2 * o + 1] = qy;
    fb[o] = ok ? glibc_hypot(rx - px, ry - py) : -1.0;
  }
}

// warp bitonic sort of 128 doubles in shared memory (ascending)
__device__ void warp_sort128(double *v) {
  const int lane = threadIdx.x & 31;
  for (int size = 2; size <= 128; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int t = lane + 32 * q;  // 64 compare-exchange pairs, 2 per lane
        if (t < 64) {
          const int lo = 2 * stride * (t / stride) + (t % stride);
          const int hi = lo + stride;
          const bool up = ((lo & size) == 0);
          const double x = v[lo], y = v[hi];
          if ((x > y) == up) {
            v[lo] = y;
            v[hi] = x;
          }
        }
      }
      __syncwarp();
    }
  }
}

__device__ __forceinline__ double py_max2(double a, double b) { return b > a ? b : a; }
__device__ __forceinline__ double py_min2(double a, double b) { return b < a ? b : a; }

struct BoxScratch {
  double v[128];
  int kept[128];
};

// one warp per box: FB-median filter, median shift, pairwise scale ratio,
// new box (klt_oracle.klt_predict steps 4-6).  valid[b] = 0 for None.
__global__ void __launch_bounds__(32 * kPtWarps)
    k_klt_boxes(KltArgs a, const double *boxes, double *out_boxes, int64_t box_stride,
                const int32_t *n_boxes, int n_boxes_const, const double *pts, const double *fwd,
                const double *fb, unsigned char *valid, int frame_w, int frame_h) {
  __shared__ BoxScratch scr[kPtWarps];
  const int s = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b = blockIdx.x * kPtWarps + warp;
  const int nb = n_boxes ? n_boxes[s] : n_boxes_const;
  if (b >= nb) return;
  BoxScratch &S = scr[warp];
  const int GG = a.grid * a.grid;
  const int64_t base = ((int64_t)s * box_stride + b) * a.max_pts;
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  // ---- lower median of the valid FB errors
  int cnt = 0;
  for (int k = lane; k < 128; k += 32) {
    const double e = k < GG ? fb[base + k] : -1.0;
    S.v[k] = e >= 0.0 ? e : inf;
    cnt += e >= 0.0 ? 1 : 0;
  }
  const int nvalid = __reduce_add_sync(0xffffffffu, cnt);
  __syncwarp();
  const int64_t ob = ((int64_t)s * box_stride + b) * 4;
  if (nvalid == 0) {
    if (lane == 0) valid[(int64_t)s * box_stride + b] = 0;
    return;
  }
  warp_sort128(S.v);
  const double thr = S.v[(nvalid - 1) / 2];
  __syncwarp();
  // ---- kept points in point order (fb valid and <= thr)
  int K = 0;
  for (int k0 = 0; k0 < GG; k0 += 32) {
    const int k = k0 + lane;
    const double e = k < GG ? fb[base + k] : -1.0;
    const bool keep = k < GG && e >= 0.0 && e <= thr;
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (keep) S.kept[K + __popc(m & ((1u << lane) - 1u))] = k;
    K += __popc(m);
  }
  __syncwarp();
  // ---- lower medians of kept dx and dy
  double med[2];
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    for (int t = lane; t < 128; t += 32)
      S.v[t] = t < K ? fwd[2 * (base + S.kept[t]) + c] - pts[2 * (base + S.kept[t]) + c] : inf;
    __syncwarp();
    warp_sort128(S.v);
    med[c] = S.v[(K - 1) / 2];
    __syncwarp();
  }
  // ---- scale: lower median of |p'_a - p'_b| / |p_a - p_b|, b = a + K/2
  double scale = 1.0;
  if (K >= 2) {
    const int half = K / 2, npair = K - half;
    int nr = 0;
    for (int a0 = 0; a0 < npair; a0 += 32) {
      const int aa = a0 + lane;
      double r = 0.0;
      bool has = false;
      if (aa < npair) {
        const int64_t ka = base + S.kept[aa], kb = base + S.kept[aa + half];
        const double d0 = glibc_hypot(pts[2 * kb] - pts[2 * ka], pts[2 * kb + 1] - pts[2 * ka + 1]);
        const double d1 = glibc_hypot(fwd[2 * kb] - fwd[2 * ka], fwd[2 * kb + 1] - fwd[2 * ka + 1]);
        has = d0 > 0.0;
        if (has) r = d1 / d0;
      }
      const unsigned m = __ballot_sync(0xffffffffu, has);
      __syncwarp();
      if (has) S.v[nr + __popc(m & ((1u << lane) - 1u))] = r;
      nr += __popc(m);
    }
    __syncwarp();
    if (nr > 0) {
      for (int t = nr + lane; t < 128; t += 32) S.v[t] = inf;
      __syncwarp();
      warp_sort128(S.v);
      scale = S.v[(nr - 1) / 2];
    }
  }
  if (lane == 0) {
    const double *bx = boxes + ob;
    const double x = bx[0], y = bx[1], w = bx[2], h = bx[3];
    const double sc = a.scale;
    const double nw = w * scale, nh = h * scale;
    const double cx = x + 0.5 * w + med[0] * sc;
    const double cy = y + 0.5 * h + med[1] * sc;
    out_boxes[ob] = py_min2(py_max2(cx - 0.5 * nw, 0.0), py_max2((double)frame_w - nw, 0.0));
    out_boxes[ob + 1] = py_min2(py_max2(cy - 0.5 * nh, 0.0), py_max2((double)frame_h - nh, 0.0));
    out_boxes[ob + 2] = nw;
    out_boxes[ob + 3] = nh;
    valid[(int64_t)s * box_stride + b] = 1;
  }
}

}  // namespace

int launch_klt_predict(const KltArgs &a, const double *boxes, double *out_boxes,
                       int64_t box_stride, const int32_t *n_boxes, int n_boxes_const,
                       int n_streams, int max_boxes, double *pts, double *fwd, double *fb,
                       unsigned char *valid, int frame_w, int frame_h, cudaStream_t s) {
  if (a.grid < 1 || a.grid * a.grid > 128) return fail(FT_EINVAL, "klt grid must be 1..11");
  const int items = max_boxes * a.grid * a.grid;
  if (items == 0) return FT_OK;
  // 3 resident CTAs per SM requested from ptxas (register cap; 2 and 4
  // measured slower)
  const dim3 grid((items + kPtWarps - 1) / kPtWarps, n_streams);
  k_klt_points<3><<<grid, 32 * kPtWarps, 0, s>>>(a, boxes, box_stride, n_boxes, n_boxes_const, pts,
                                                 fwd, fb);
  k_klt_boxes<<<dim3((max_boxes + kPtWarps - 1) / kPtWarps, n_streams), 32 * kPtWarps, 0, s>>>(
      a, boxes, out_boxes, box_stride, n_boxes, n_boxes_const, pts, fwd, fb, valid, frame_w,
      frame_h);
  count_launch(2);
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

}  // namespace ft

// Dense coarse-to-fine TV-L1 optical flow (reference optflow.py:147-253).
//
// Per scale: central gradient of I1 (optflow.py:155); per warp a setup pass
// (bilinear gathers + linearised data-term constants, :158-176); the
// primal-dual iterations (:178-208) in a temporally blocked tile kernel; a
// 3x3 median of both components (:210-211).  Between scales a bilinear
// upsample scaled by the size ratio (:244-249).
//
// HBM layout (per batch of nb image pairs, all planes float64 row-major,
// pitch == level width, capacity `cap` elements per plane):
//   const planes  gx, gy, r0        [nb][cap]
//   gradient      ix, iy            [nb][cap]
//   state ping-pong st[2]           [8][nb][cap]  (u1 u2 b1 b2 p11 p12 p21 p22)
// where b = "u bar" (optflow.py:173-174, :205-206).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include <cooperative_groups.h>

#include "ft_internal.cuh"

namespace ft {

namespace cg = cooperative_groups;

namespace {

enum { U1 = 0, U2, B1, B2, P11, P12, P21, P22, NST };

struct StatePtrs {
  double *p[NST];
};

__device__ __forceinline__ double clip_lo_hi(double v, double lo, double hi) {
  v = v > lo ? v : lo;  // numpy clip: min(max(v, lo), hi)
  return v < hi ? v : hi;
}

// bilinear_sample (imageops.py:53-66) at one point, clamped to the border
__device__ __forceinline__ double bsample(const double *__restrict__ img, int w, int h, double x,
                                          double y) {
  x = clip_lo_hi(x, 0.0, w - 1.0);
  y = clip_lo_hi(y, 0.0, h - 1.0);
  const int x0 = (int)floor(x), y0 = (int)floor(y);
  const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
  const double fx = x - (double)x0, fy = y - (double)y0;
  const double *r0 = img + (int64_t)y0 * w;
  const double *r1 = img + (int64_t)y1 * w;
  const double top = r0[x0] * (1.0 - fx) + r0[x1] * fx;
  const double bot = r1[x0] * (1.0 - fx) + r1[x1] * fx;
  return top * (1.0 - fy) + bot * fy;
}

// np.gradient(i1) with unit spacing (optflow.py:155): central inside,
// one-sided at the borders.  (a-b)/2 == (a-b)*0.5 exactly.
__global__ void k_central_grad(const double *__restrict__ img, int w, int h, int64_t is,
                               double *__restrict__ gx, double *__restrict__ gy, int64_t gs) {
  img += blockIdx.z * is;
  gx += blockIdx.z * gs;
  gy += blockIdx.z * gs;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (r >= h || c >= w) return;
  const int64_t o = (int64_t)r * w + c;
  double vx, vy;
  if (c == 0)
    vx = img[o + 1] - img[o];
  else if (c == w - 1)
    vx = img[o] - img[o - 1];
  else
    vx = (img[o + 1] - img[o - 1]) * 0.5;
  if (r == 0)
    vy = img[o + w] - img[o];
  else if (r == h - 1)
    vy = img[o] - img[o - w];
  else
    vy = (img[o + w] - img[o - w]) * 0.5;
  gx[o] = vx;
  gy[o] = vy;
}

// resize_bilinear(u, w, h) * ratio for both components (optflow.py:244-249,
// imageops.py:69-75).  rx = wc/wf, ry = hc/hf (host-computed IEEE quotients),
// sx = wf/wc, sy = hf/hc.
__global__ void k_upsample(const double *__restrict__ cu1, const double *__restrict__ cu2,
                           int wc, int hc, double *__restrict__ fu1, double *__restrict__ fu2,
                           int wf, int hf, int64_t cap, double rx, double ry, double sx,
                           double sy) {
  cu1 += blockIdx.z * cap;
  cu2 += blockIdx.z * cap;
  fu1 += blockIdx.z * cap;
  fu2 += blockIdx.z * cap;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (r >= hf || c >= wf) return;
  const double x = ((double)c + 0.5) * rx - 0.5;
  const double y = ((double)r + 0.5) * ry - 0.5;
  const int64_t o = (int64_t)r * wf + c;
  fu1[o] = bsample(cu1, wc, hc, x, y) * sx;
  fu2[o] = bsample(cu2, wc, hc, x, y) * sy;
}

// Per-warp linearisation (optflow.py:158-167): gather I1, dI1/dx, dI1/dy at
// x+u; rho0 = I1w - I0 - gx*u1 - gy*u2.
__global__ void k_warp_setup(const double *__restrict__ i0, const double *__restrict__ i1,
                             int64_t ps, const double *__restrict__ ix,
                             const double *__restrict__ iy, const double *__restrict__ u1,
                             const double *__restrict__ u2, int w, int h, int64_t cap,
                             double *__restrict__ gx, double *__restrict__ gy,
                             double *__restrict__ r0) {
  i0 += blockIdx.z * ps;
  i1 += blockIdx.z * ps;
  const int64_t so = blockIdx.z * cap;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (r >= h || c >= w) return;
  const int64_t o = (int64_t)r * w + c;
  const double a = u1[so + o], b = u2[so + o];
  const double mx = (double)c + a, my = (double)r + b;
  const double v = bsample(i1, w, h, mx, my);
  const double g1 = bsample(ix + so, w, h, mx, my);
  const double g2 = bsample(iy + so, w, h, mx, my);
  gx[so + o] = g1;
  gy[so + o] = g2;
  r0[so + o] = v - i0[o] - g1 * a - g2 * b;
}

// 3x3 median with replicated border (imageops.py:78-84): exact 5th order
// statistic of 9 via a min/max selection network.
__device__ __forceinline__ void cswap(double &a, double &b) {
  const double lo = fmin(a, b), hi = fmax(a, b);
  a = lo;
  b = hi;
}

__device__ __forceinline__ double median9(double *v) {
  // Paeth / Devillard opt_med9 network (19 compare-swaps)
  cswap(v[1], v[2]); cswap(v[4], v[5]); cswap(v[7], v[8]);
  cswap(v[0], v[1]); cswap(v[3], v[4]); cswap(v[6], v[7]);
  cswap(v[1], v[2]); cswap(v[4], v[5]); cswap(v[7], v[8]);
  cswap(v[0], v[3]); cswap(v[5], v[8]); cswap(v[4], v[7]);
  cswap(v[3], v[6]); cswap(v[1], v[4]); cswap(v[2], v[5]);
  cswap(v[4], v[7]); cswap(v[4], v[2]); cswap(v[6], v[4]);
  cswap(v[4], v[2]);
  return v[4];
}

__device__ __forceinline__ double med3(double a, double b, double c) {
  return fmax(fmin(a, b), fmin(fmax(a, b), c));
}

// Two horizontally adjacent outputs per thread: the four 3-sample columns
// c-1..c+2 are sorted once and shared; median9 = med3(max of the column
// minima, med3 of the column medians, min of the column maxima), the same
// order statistic as the sort (exact selection).
__global__ void k_median(const double *__restrict__ a1, const double *__restrict__ a2,
                         double *__restrict__ o1, double *__restrict__ o2, int w, int h,
                         int64_t cap) {
  const int64_t so = blockIdx.z * cap;
  const int c = 2 * (blockIdx.x * blockDim.x + threadIdx.x);
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (r >= h || c >= w) return;
  const int64_t rr[3] = {(int64_t)max(r - 1, 0) * w, (int64_t)r * w, (int64_t)min(r + 1, h - 1) * w};
  int cc[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) cc[k] = min(max(c - 1 + k, 0), w - 1);
  const bool two = c + 1 < w;
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    const double *a = (f ? a2 : a1) + so;
    double lo[4], md[4], hi[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double x = a[rr[0] + cc[k]], y = a[rr[1] + cc[k]], z = a[rr[2] + cc[k]];
      cswap(x, y);
      cswap(y, z);
      cswap(x, y);
      lo[k] = x, md[k] = y, hi[k] = z;
    }
    double *o = (f ? o2 : o1) + so + (int64_t)r * w + c;
    o[0] = med3(fmax(fmax(lo[0], lo[1]), lo[2]), med3(md[0], md[1], md[2]),
                fmin(fmin(hi[0], hi[1]), hi[2]));
    if (two)
      o[1] = med3(fmax(fmax(lo[1], lo[2]), lo[3]), med3(md[1], md[2], md[3]),
                  fmin(fmin(hi[1], hi[2]), hi[3]));
  }
}

// Per-pixel terms of the TV-L1 objective (optflow.py:121-137): data term
// |I1(x+u) - I0| and, per component, huber(hypot(forward_gradient(u))).
// The reference sums these arrays with numpy; the caller does exactly that
// on the host copies, so the scalar is bit-identical too.
__global__ void k_energy_terms(const double *__restrict__ i0, const double *__restrict__ i1,
                               const double *__restrict__ u1, const double *__restrict__ u2,
                               int w, int h, double eps, double *__restrict__ data,
                               double *__restrict__ s1, double *__restrict__ s2) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (r >= h || c >= w) return;
  const int64_t o = (int64_t)r * w + c;
  const double v = bsample(i1, w, h, (double)c + u1[o], (double)r + u2[o]);
  data[o] = fabs(v - i0[o]);
  const double *comp[2] = {u1, u2};
  double *dst[2] = {s1, s2};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double *u = comp[k];
    const double gx = c < w - 1 ? u[o + 1] - u[o] : 0.0;
    const double gy = r < h - 1 ? u[o + w] - u[o] : 0.0;
    const double m = glibc_hypot(gx, gy);
    // _huber (optflow.py:121-124)
    dst[k][o] = eps <= 0.0 ? m : (m <= eps ? m * m / (2.0 * eps) : m - eps / 2.0);
  }
}

StatePtrs state_ptrs(double *base, int nb, int64_t cap) {
  StatePtrs s;
  for (int k = 0; k < NST; ++k) s.p[k] = base + (int64_t)k * nb * cap;
  return s;
}

// ------------------------------------------------------------------------
// Primal-dual iterations, temporally blocked (optflow.py:178-208).
//
// A CTA owns a TW x TH tile of the level that overlaps its neighbours by
// `halo` pixels on every side that is not an image border.  One iteration's
// dependency radius is 1 in each direction (dual step reads u-bar at x+1 and
// y+1; primal step reads p at x-1 and y-1), so after `iters <= halo`
// iterations the inner (TW-2*halo) x (TH-2*halo) region is exact and is
// written back.  A tile that covers the whole level needs no halo and runs a
// whole warp's iterations in one launch.
//
// Shared memory holds the fields read at a neighbour (b1 b2 p11 p12 p21 p22)
// in [TH+2][TW+2] planes with a one-element apron, so every neighbour read
// is an immediate offset from the thread's base address.  Each field is
// updated in place: the dual step reads only its own p, the primal step only
// its own u-bar, so two barriers per iteration suffice.  Pointwise fields
// (u, the gathered gradient, rho0, the threshold, 1/|grad|^2 derived once per
// launch) live in registers of the owning thread: thread (tx, ty) owns
// columns tx + 32*cx (cx < TW/32) and rows ty + BY*k (k < PY).
// ------------------------------------------------------------------------
struct PDArgs {
  StatePtrs in, out;
  const double *gx, *gy, *r0;
  int w, h;
  int64_t cap;
  int halo, iters, first, nb;
  int pow2;  // sigma and tau are powers of two (exact fused multiply-adds)
  int cone;  // compute only the rows feeding the written interior (FT_PD_CONE)
  int cq;    // CTA-wide projection queue (FT_PD_CQ)
  int async_ld;  // exchange planes loaded with cp.async (FT_PD_ASYNC)
  // k_pd_tile half-step schedule: the launch runs `nhalf` alternating dual (D)
  // / primal (P) half-steps, starting with D when `first` (u-bar = u, p = 0)
  // and with P otherwise; it ends after a D (state u, p) unless `last` (ends
  // after a P, writes u only).  rows_lo/hi[j]: rows half-step j must compute
  // (shrinking cone; cone_rows == 0 -> all rows).
  int nhalf, last, cone_rows;
  signed char rows_lo[16], rows_hi[16];
  double tau, lam, sigma, shrink;  // shrink = 1/(1+sigma*eps)
};

// per-pixel border flags (global position, fixed for the launch)
enum : unsigned { FL_R = 1, FL_D = 2, FL_L = 4, FL_LASTC = 8, FL_U = 16, FL_LASTR = 32, FL_OK = 64 };

// Exchange planes hold the fields read at a neighbour as three interleaved
// double2 planes -- (b1,b2), (p11,p21), (p12,p22) -- the pairs that are always
// read together, so each neighbour access is one 128-bit shared load.  sxi()
// maps field f (0..5 = b1 b2 p11 p12 p21 p22) of element id to its double
// index.
__device__ __forceinline__ int sxi(int f, int id, int PL) {
  const int pair = f == 0 || f == 1 ? 0 : (f == 2 || f == 4 ? 1 : 2);
  const int comp = f == 1 || f == 4 || f == 5 ? 1 : 0;
  return 2 * (pair * PL + id) + comp;
}

template <int TW, int BY, int PY>
struct PDGeom {
  static constexpr int NX = TW / 32, TH = BY * PY, NP = NX * PY;
  static constexpr int SP = TW + 2, SR = TH + 2, PLANE = SP * SR;
  // 6 exchange planes + per-warp projection queue (2*NP pairs per lane)
  static constexpr size_t smem = 6 * PLANE * sizeof(double) + BY * 2 * NP * 32 * 16;
};

// `iters` primal-dual iterations over a tile held in shared memory (the six
// exchange planes with apron) and registers (pointwise fields); `xch` runs
// after each half step's shared-memory writes (a block barrier in the tiled
// kernel, the DSMEM edge exchange in the cluster kernel).
// a*b + c.  With P2 the product is exact (b or a is a power of two: sigma
// and tau for the default time_step 0.25, the literal 2.0), so one fused
// multiply-add rounds exactly like the reference's separate multiply and
// add; otherwise the two IEEE operations are kept (-fmad=false).
template <bool P2>
__device__ __forceinline__ double madx(double a, double b, double c) {
  return P2 ? fma(a, b, c) : a * b + c;
}

// IN: the tile holds no image-border pixel (all border rules are "interior":
// the reference's zero gradients / one-sided divergences never apply), so the
// per-pixel flag selects fold away.
template <int TW, int BY, int PY, bool P2, bool IN, typename X>
__device__ __forceinline__ void pd_iterate(int iters, double *sm, int base, int tx,
                                           const unsigned *fl, double *u1, double *u2,
                                           const double *gx, const double *gy, const double *r0,
                                           const double *thr, const double *ig2, double tau,
                                           double tl, double sigma, double shrink, double2 *queue,
                                           X &xch, int ty = 0, int cone = -1) {
  using G = PDGeom<TW, BY, PY>;
  constexpr int NX = G::NX, NP = G::NP, SP = G::SP, PL = G::PLANE, TH = G::TH;
  double2 *const sB = reinterpret_cast<double2 *>(sm), *const sPX = sB + PL, *const sPY = sPX + PL;
  const unsigned lt_mask = (1u << tx) - 1u;
  for (int it = 0; it < iters; ++it) {
    double p11[NP], p12[NP], p21[NP], p22[NP];
    // Shrinking cone (cone = halo - iters >= 0, tiles with a halo): only the
    // rows that feed the written interior [halo, TH-halo) are computed.
    // Iteration it needs p on rows [cone+it, TH-1-cone-it) and u on
    // [cone+it+1, TH-1-cone-it); a row is one warp, so the skip is
    // warp-uniform.  Values outside the cone are never read by rows inside.
    bool dual_row[NP], primal_row[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int lr = ty + BY * (q / NX);
      dual_row[q] = cone < 0 || (lr >= cone + it && lr < TH - 1 - cone - it);
      primal_row[q] = cone < 0 || (lr >= cone + it + 1 && lr < TH - 1 - cone - it);
    }
    // ---- dual ascent with Huber prox (:180-185); the apron makes the
    // neighbour loads safe, the border flags select the reference's zeros
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      if (!dual_row[q]) {
        p11[q] = p12[q] = p21[q] = p22[q] = 0.0;  // not projected, not stored
        continue;
      }
      const int id = base + (q / NX) * BY * SP + 32 * (q % NX);
      const double2 cb = sB[id], rb = sB[id + 1], db = sB[id + SP];
      const double2 opx = sPX[id], opy = sPY[id];
      const double c1 = cb.x, c2 = cb.y, r1 = rb.x, r2 = rb.y, d1 = db.x, d2 = db.y;
      const bool R = IN || (fl[q] & FL_R), D = IN || (fl[q] & FL_D);
      const double a1x = R ? r1 - c1 : 0.0;
      const double a1y = D ? d1 - c1 : 0.0;
      const double a2x = R ? r2 - c2 : 0.0;
      const double a2y = D ? d2 - c2 : 0.0;
      p11[q] = madx<P2>(sigma, a1x, opx.x) * shrink;
      p12[q] = madx<P2>(sigma, a1y, opy.x) * shrink;
      p21[q] = madx<P2>(sigma, a2x, opx.y) * shrink;
      p22[q] = madx<P2>(sigma, a2y, opy.y) * shrink;
    }
    // ---- unit-ball projection n = max(1, hypot(.)); p /= n (:186-191).
    // When |q|^2 is clearly below 1 the norm is exactly 1 and p/1 == p, so
    // only the few saturated pairs need hypot + two divisions.  They are
    // compacted into a per-warp queue (ballot + popc) and processed by all
    // 32 lanes together, instead of up to 2*NP divergent passes per warp.
    {
      unsigned need = 0;
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        // screening test only (not reference arithmetic): fused is fine
        if (fma(p11[q], p11[q], p12[q] * p12[q]) > 0.999999) need |= 1u << (2 * q);
        if (fma(p21[q], p21[q], p22[q] * p22[q]) > 0.999999) need |= 1u << (2 * q + 1);
      }
      int off[2 * NP];
      int total = 0;
      if (__any_sync(0xffffffffu, need != 0u)) {  // most warps skip the queue
#pragma unroll
        for (int j = 0; j < 2 * NP; ++j) {
          const unsigned m = __ballot_sync(0xffffffffu, (need >> j) & 1u);
          off[j] = total + __popc(m & lt_mask);
          total += __popc(m);
        }
      }
      if (total) {  // warp-uniform
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          if (need & (1u << (2 * q))) queue[off[2 * q]] = make_double2(p11[q], p12[q]);
          if (need & (1u << (2 * q + 1))) queue[off[2 * q + 1]] = make_double2(p21[q], p22[q]);
        }
        __syncwarp();
        for (int t = tx; t < total; t += 32) {
          const double2 v = queue[t];
          const double n = np_max(1.0, glibc_hypot(v.x, v.y));
          queue[t] = make_double2(v.x / n, v.y / n);
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          if (need & (1u << (2 * q))) {
            const double2 v = queue[off[2 * q]];
            p11[q] = v.x;
            p12[q] = v.y;
          }
          if (need & (1u << (2 * q + 1))) {
            const double2 v = queue[off[2 * q + 1]];
            p21[q] = v.x;
            p22[q] = v.y;
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      if (!dual_row[q]) continue;
      const int id = base + (q / NX) * BY * SP + 32 * (q % NX);
      sPX[id] = make_double2(p11[q], p21[q]);  // in place: only the owner reads p here
      sPY[id] = make_double2(p12[q], p22[q]);
    }
    xch.after_dual();
    // ---- primal descent + TV-L1 shrinkage (:194-208)
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      if (!primal_row[q]) continue;
      const int id = base + (q / NX) * BY * SP + 32 * (q % NX);
      const unsigned f = fl[q];
      // divergence (imageops.py:41-50): dx + dy with border rules
      const double2 lp = sPX[id - 1], up = sPY[id - SP];
      const double l11 = lp.x, l21 = lp.y, u12 = up.x, u22 = up.y;
      const bool L = IN || (f & FL_L), LC = !IN && (f & FL_LASTC);
      const bool U = IN || (f & FL_U), LR = !IN && (f & FL_LASTR);
      const double dx1 = L ? (LC ? -l11 : p11[q] - l11) : p11[q];
      const double dx2 = L ? (LC ? -l21 : p21[q] - l21) : p21[q];
      const double dy1 = U ? (LR ? -u12 : p12[q] - u12) : p12[q];
      const double dy2 = U ? (LR ? -u22 : p22[q] - u22) : p22[q];
      const double v1 = madx<P2>(tau, dx1 + dy1, u1[q]);
      const double v2 = madx<P2>(tau, dx2 + dy2, u2[q]);
      const double rho = r0[q] + gx[q] * v1 + gy[q] * v2;
      const bool lo = rho < -thr[q];
      const bool hi = rho > thr[q];
      double d = lo ? tl : (hi ? -tl : -rho * ig2[q]);
      d = (ig2[q] != 0.0 || lo || hi) ? d : 0.0;  // ig2 != 0 <=> |grad|^2 > 1e-12
      const double n1 = v1 + d * gx[q];
      const double n2 = v2 + d * gy[q];
      // in place: no other thread reads u-bar in this phase
      sB[id] = make_double2(madx<true>(2.0, n1, -u1[q]), madx<true>(2.0, n2, -u2[q]));
      u1[q] = n1;
      u2[q] = n2;
    }
    xch.after_primal();
  }
}

// Half-step schedule of k_pd_tile with a CTA-wide projection queue.
//
// The launch boundary sits after a dual step, where the state is (u, p):
// u-bar is recomputed by the primal step that opens the next launch, so a
// launch reads 9 planes and writes 6 instead of 11 / 8.
//
// Dual half-step: the unprojected p is stored in place, the saturated pairs
// of the whole CTA (~9 % at C2) are appended to one shared index list, and
// after a barrier the first ceil(n/32) warps project them in place (instead
// of every warp running the hypot + division code for its own ~4 pairs with
// most lanes idle).  Primal half-step: reads its p from shared memory.
// Same arithmetic in the same order as the reference iteration.
// CL: the CTA is one of a 2x1 thread-block cluster covering a 64-column
// region; the seam column is exchanged through distributed shared memory
// after every half-step (see k_pd_tile).
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::
                   : "memory");
}

template <int TW, int BY, int PY, bool P2, bool IN, bool MID, bool CL = false>
__device__ __forceinline__ void pd_halfsteps_cq(const PDArgs &a, double *sm, int base, int tx,
                                                int ty, const unsigned *fl, double *u1,
                                                double *u2, const double *gx, const double *gy,
                                                const double *r0, const double *thr,
                                                const double *ig2, double tl, int *qidx,
                                                int *ctr) {
  using G = PDGeom<TW, BY, PY>;
  constexpr int NX = G::NX, NP = G::NP, SP = G::SP, PL = G::PLANE, TH = G::TH;
  constexpr int NT = 32 * BY;
  const double tau = a.tau, sigma = a.sigma, shrink = a.shrink;
  double2 *const sB = reinterpret_cast<double2 *>(sm), *const sPX = sB + PL, *const sPY = sPX + PL;
  double *const dPX = reinterpret_cast<double *>(sPX), *const dPY = reinterpret_cast<double *>(sPY);
  const unsigned lt_mask = (1u << tx) - 1u;
  const int tid = ty * 32 + tx;
  int nd = 0;  // dual half-steps done (queue counter parity)
  auto half = [&](const bool dual, const int lo, const int hi) {
    bool row_on[NP];
    bool all = true;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int lr = ty + BY * (q / NX);
      row_on[q] = lr >= lo && lr < hi;
      all = all && row_on[q];
    }
    if (dual) {
      // ---- dual ascent with Huber prox (:180-185), unprojected p stored in place
      unsigned need = 0;
      // (the common all-rows-active case runs branch-free so the compiler can
      // interleave the pixels' dependency chains)
      auto dual_px = [&](const int q) {
        const int id = base + (q / NX) * BY * SP + 32 * (q % NX);
        const double2 cb = sB[id], rb = sB[id + 1], db = sB[id + SP];
        const double2 opx = sPX[id], opy = sPY[id];
        const bool R = IN || (fl[q] & FL_R), D = IN || (fl[q] & FL_D);
        const double a1x = R ? rb.x - cb.x : 0.0;
        const double a1y = D ? db.x - cb.x : 0.0;
        const double a2x = R ? rb.y - cb.y : 0.0;
        const double a2y = D ? db.y - cb.y : 0.0;
        const double p11 = madx<P2>(sigma, a1x, opx.x) * shrink;
        const double p12 = madx<P2>(sigma, a1y, opy.x) * shrink;
        const double p21 = madx<P2>(sigma, a2x, opx.y) * shrink;
        const double p22 = madx<P2>(sigma, a2y, opy.y) * shrink;
        sPX[id] = make_double2(p11, p21);
        sPY[id] = make_double2(p12, p22);
        // screening test only (not reference arithmetic): fused is fine
        if (fma(p11, p11, p12 * p12) > 0.999999) need |= 1u << (2 * q);
        if (fma(p21, p21, p22 * p22) > 0.999999) need |= 1u << (2 * q + 1);
#ifdef FT_PD_DEBUG_NOPROJ
        need = 0;  // timing study only: skip the projection (breaks parity)
#endif
      };
      if (all) {
#pragma unroll
        for (int q = 0; q < NP; ++q) dual_px(q);
      } else {
#pragma unroll
        for (int q = 0; q < NP; ++q)
          if (row_on[q]) dual_px(q);
      }
      // ---- append saturated pairs: one shared atomic per warp
      int off[2 * NP];
      int total = 0;
      if (__any_sync(0xffffffffu, need != 0u)) {
#pragma unroll
        for (int k = 0; k < 2 * NP; ++k) {
          const unsigned m = __ballot_sync(0xffffffffu, (need >> k) & 1u);
          off[k] = total + __popc(m & lt_mask);
          total += __popc(m);
        }
        int wbase = 0;
        if (tx == 0) wbase = atomicAdd(&ctr[nd & 1], total);
        wbase = __shfl_sync(0xffffffffu, wbase, 0);
#pragma unroll
        for (int k = 0; k < 2 * NP; ++k) {
          const int q = k >> 1;
          const int id = base + (q / NX) * BY * SP + 32 * (q % NX);
          if ((need >> k) & 1u) qidx[wbase + off[k]] = 2 * id + (k & 1);
        }
      }
      __syncthreads();
      // ---- unit-ball projection n = max(1, hypot(.)); p /= n (:186-191)
      const int n = ctr[nd & 1];
      if (tid == 0) ctr[(nd + 1) & 1] = 0;  // next dual's list (unused until then)
      for (int e = tid; e < n; e += NT) {
        const int k = qidx[e];
        const double pa = dPX[k], pb = dPY[k];
        const double nn = np_max(1.0, glibc_hypot(pa, pb));
        dPX[k] = pa / nn;
        dPY[k] = pb / nn;
      }
      ++nd;
    } else {
      // ---- primal descent + TV-L1 shrinkage (:194-208), u-bar stored in place
      auto primal_px = [&](const int q) {
        const int id = base + (q / NX) * BY * SP + 32 * (q % NX);
        const unsigned f = fl[q];
        const double2 mpx = sPX[id], mpy = sPY[id];
        const double p11 = mpx.x, p21 = mpx.y, p12 = mpy.x, p22 = mpy.y;
        const double2 lp = sPX[id - 1], up = sPY[id - SP];
        const double l11 = lp.x, l21 = lp.y, u12 = up.x, u22 = up.y;
        const bool L = IN || (f & FL_L), LC = !IN && (f & FL_LASTC);
        const bool U = IN || (f & FL_U), LR = !IN && (f & FL_LASTR);
        const double dx1 = L ? (LC ? -l11 : p11 - l11) : p11;
        const double dx2 = L ? (LC ? -l21 : p21 - l21) : p21;
        const double dy1 = U ? (LR ? -u12 : p12 - u12) : p12;
        const double dy2 = U ? (LR ? -u22 : p22 - u22) : p22;
        const double v1 = madx<P2>(tau, dx1 + dy1, u1[q]);
        const double v2 = madx<P2>(tau, dx2 + dy2, u2[q]);
        const double rho = r0[q] + gx[q] * v1 + gy[q] * v2;
        const bool lo_ = rho < -thr[q];
        const bool hi_ = rho > thr[q];
        double d = lo_ ? tl : (hi_ ? -tl : -rho * ig2[q]);
        d = (ig2[q] != 0.0 || lo_ || hi_) ? d : 0.0;  // ig2 != 0 <=> |grad|^2 > 1e-12
        const double n1 = v1 + d * gx[q];
        const double n2 = v2 + d * gy[q];
        sB[id] = make_double2(madx<true>(2.0, n1, -u1[q]), madx<true>(2.0, n2, -u2[q]));
        u1[q] = n1;
        u2[q] = n2;
      };
      if (all) {
#pragma unroll
        for (int q = 0; q < NP; ++q) primal_px(q);
      } else {
#pragma unroll
        for (int q = 0; q < NP; ++q)
          if (row_on[q]) primal_px(q);
      }
    }
    if (CL) {
      // seam exchange: after a primal step the right CTA's column 0 u-bar
      // goes to the left CTA's right apron; after a dual step (projection
      // done: block barrier first) the left CTA's column 31 (p11, p21) goes
      // to the right CTA's left apron.  The cluster barrier publishes them.
      static_assert(!CL || TW == 32, "seam exchange assumes 32-column tiles");
      cg::cluster_group cl = cg::this_cluster();
      const unsigned rank = cl.block_rank();
      if (dual) __syncthreads();
      if (dual ? (rank == 0 && tx == 31) : (rank == 1 && tx == 0)) {
        double2 *const plane = dual ? sPX : sB;
        double2 *const remote = cl.map_shared_rank(plane, rank ^ 1u);
#pragma unroll
        for (int q = 0; q < NP; ++q) {
          const int id = base + (q / NX) * BY * SP + 32 * (q % NX);
          remote[id + (dual ? -31 : 31) + (dual ? -1 : 1)] = plane[id];
        }
      }
      cluster_sync_all();
    } else {
      __syncthreads();
    }
  };
  if (MID) {
    // middle launch (P D)x4 of a 32-row tile with halo 4: the cone rows of
    // halfstep_schedule in closed form -- P_i: [1+i, 32-i), D_i: [1+i, 31-i)
    static_assert(!MID || TH == 32, "closed-form cone is for 32-row tiles");
    for (int i = 0; i < 4; ++i) {
      half(false, 1 + i, TH - i);
      half(true, 1 + i, TH - 1 - i);
    }
  } else {
    for (int j = 0; j < a.nhalf; ++j) {
      const bool dual = ((j & 1) == 0) == (a.first != 0);
      half(dual, a.cone_rows ? a.rows_lo[j] : 0, a.cone_rows ? a.rows_hi[j] : TH);
    }
  }
}

// global -> shared copies without register staging (LDGSTS)
__device__ __forceinline__ void cp_async8(double *dst, const double *src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 8 : 0;  // src-size 0: zero-fill the 8 bytes
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

struct BlockBarrier {
  __device__ __forceinline__ void after_dual() { __syncthreads(); }
  __device__ __forceinline__ void after_primal() { __syncthreads(); }
};


template <int TW, int BY, int PY, int MINB, bool MID = false, bool CL = false>
__global__ void __launch_bounds__(32 * BY, MINB) k_pd_tile(const PDArgs a) {
  using G = PDGeom<TW, BY, PY>;
  constexpr int NX = G::NX, TH = G::TH, NP = G::NP, SP = G::SP, PL = G::PLANE;
  extern __shared__ __align__(16) double sm[];

  const int W = a.w, H = a.h;
  const int step_x = TW - 2 * a.halo, step_y = TH - 2 * a.halo;
  // CL: 2x1 cluster over a (2 TW)-column region with the halo on its outer
  // sides only; rank 0 is the left tile, rank 1 the right one
  const int rk = CL ? (int)(blockIdx.x & 1) : 0;
  const int ox = CL ? (int)(blockIdx.x >> 1) * (2 * TW - 2 * a.halo) - a.halo + TW * rk
                    : (int)blockIdx.x * step_x - a.halo;
  const int oy = blockIdx.y * step_y - a.halo;
  const int64_t so = blockIdx.z * a.cap;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * 32 + tx;
  const int base = (ty + 1) * SP + tx + 1;  // apron offset (+1,+1)

  // zero the apron ring once (read only by halo pixels, keeps them finite)
  for (int k = tid; k < 2 * SP + 2 * TH; k += 32 * BY) {
    int idx;
    if (k < SP) idx = k;
    else if (k < 2 * SP) idx = (TH + 1) * SP + (k - SP);
    else if (k < 2 * SP + TH) idx = (k - 2 * SP + 1) * SP;
    else idx = (k - 2 * SP - TH + 1) * SP + SP - 1;
#pragma unroll
    for (int f = 0; f < 6; ++f) sm[sxi(f, idx, PL)] = 0.0;
  }
  if (CL) {
    // seam apron before the first half-step (later ones are pushed by the
    // neighbour): the right tile's first primal step reads (p11, p21) at
    // column ox-1; the left tile's first dual step (first launch) reads
    // u-bar = u at column ox+TW
    __syncthreads();  // after the apron zeroing
    const bool need = rk == 1 ? (!a.first && tx == 0) : (a.first && tx == 31);
    if (need) {
      const int gc = rk == 1 ? ox - 1 : ox + TW;
#pragma unroll
      for (int k = 0; k < PY; ++k) {
        const int lr = ty + BY * k, gr = oy + lr;
        const bool in = gc >= 0 && gc < W && gr >= 0 && gr < H;
        const int64_t o = so + (int64_t)gr * W + gc;
        const int idx = (lr + 1) * SP + (rk == 1 ? 0 : SP - 1);
        const int f0 = rk == 1 ? 2 : 0, f1 = rk == 1 ? 4 : 1;  // (p11, p21) / (b1, b2)
        const double *s0 = rk == 1 ? a.in.p[P11] : a.in.p[U1];
        const double *s1 = rk == 1 ? a.in.p[P21] : a.in.p[U2];
        sm[sxi(f0, idx, PL)] = in ? s0[o] : 0.0;
        sm[sxi(f1, idx, PL)] = in ? s1[o] : 0.0;
      }
    }
  }

  const double tl = a.tau * a.lam;
  double u1[NP], u2[NP], gx[NP], gy[NP], r0[NP], thr[NP], ig2[NP];
  unsigned fl[NP];

#pragma unroll
  for (int k = 0; k < PY; ++k) {
#pragma unroll
    for (int cx = 0; cx < NX; ++cx) {
      const int q = k * NX + cx;
      const int gc = ox + tx + 32 * cx, gr = oy + ty + BY * k;
      const bool in = gc >= 0 && gc < W && gr >= 0 && gr < H;
      const int64_t o = so + (int64_t)gr * W + gc;
      const int id = base + k * BY * SP + 32 * cx;
      // p planes go straight to shared memory (cp.async, zero-filled outside
      // the image): no registers held, all copies in flight at once.  u-bar
      // is not part of the state between launches: the launch opens with a
      // primal half-step that writes it (first launch: u-bar = u, p = 0).
      if (!a.first) {
#pragma unroll
        for (int f = 2; f < 6; ++f)
          cp_async8(&sm[sxi(f, id, PL)], in ? a.in.p[B1 + f] + o : a.in.p[B1 + f], in);
      }
      double vu1 = 0, vu2 = 0, vgx = 0, vgy = 0, vr0 = 0;
      if (in) {
        vu1 = a.in.p[U1][o];
        vu2 = a.in.p[U2][o];
        vgx = a.gx[o];
        vgy = a.gy[o];
        vr0 = a.r0[o];
      }
      u1[q] = vu1;
      u2[q] = vu2;
      gx[q] = vgx;
      gy[q] = vgy;
      r0[q] = vr0;
      const double g2 = vgx * vgx + vgy * vgy;  // optflow.py:163
      const bool ok = g2 > 1e-12;
      ig2[q] = ok ? 1.0 / (g2 > 1e-12 ? g2 : 1e-12) : 0.0;
      thr[q] = tl * g2;  // tau*lam*grad_sq (optflow.py:176)
      fl[q] = (gc < W - 1 ? FL_R : 0u) | (gr < H - 1 ? FL_D : 0u) | (gc > 0 ? FL_L : 0u) |
              (gc == W - 1 ? FL_LASTC : 0u) | (gr > 0 ? FL_U : 0u) | (gr == H - 1 ? FL_LASTR : 0u) |
              (ok ? FL_OK : 0u);
      if (a.first) {  // ub = u, p = 0 at the start of a warp (optflow.py:169-174)
        sm[sxi(0, id, PL)] = vu1;
        sm[sxi(1, id, PL)] = vu2;
#pragma unroll
        for (int f = 2; f < 6; ++f) sm[sxi(f, id, PL)] = 0.0;
      }
    }
  }
  if (!a.first) cp_async_wait_all();
  if (tid < 2) reinterpret_cast<int *>(sm + 6 * PL)[2 * NP * 32 * BY + tid] = 0;  // queue counters
  __syncthreads();

  // tile free of image-border pixels (uniform per CTA): flag-free fast path
  const bool interior = ox >= 1 && oy >= 1 && ox + TW <= W - 1 && oy + TH <= H - 1;
  {
    int *const qidx = reinterpret_cast<int *>(sm + 6 * PL);
    int *const ctr = qidx + 2 * NP * 32 * BY;
#define FT_PD_CALL(P2_, IN_)                                                                 \
  pd_halfsteps_cq<TW, BY, PY, P2_, IN_, MID, CL>(a, sm, base, tx, ty, fl, u1, u2, gx, gy, r0, thr, ig2, \
                                        tl, qidx, ctr)
    if (a.pow2) {
      if (interior) FT_PD_CALL(true, true); else FT_PD_CALL(true, false);
    } else {
      if (interior) FT_PD_CALL(false, true); else FT_PD_CALL(false, false);
    }
#undef FT_PD_CALL
  }

  // ---- write back the exact interior: u, and p unless this is the warp's
  // last launch (the next warp starts from p = 0)
  const int lo_x = (CL && rk == 1) ? 0 : a.halo, hi_x = (CL && rk == 0) ? TW : TW - a.halo;
  const int lo_y = a.halo, hi_y = TH - a.halo;
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const int k = q / NX, cx = q % NX;
    const int lc = tx + 32 * cx, lr = ty + BY * k;
    const int gc = ox + lc, gr = oy + lr;
    if (gc < 0 || gc >= W || gr < 0 || gr >= H) continue;
    if (lc < lo_x || lc >= hi_x || lr < lo_y || lr >= hi_y) continue;
    const int id = base + k * BY * SP + 32 * cx;
    const int64_t o = so + (int64_t)gr * W + gc;
    a.out.p[U1][o] = u1[q];
    a.out.p[U2][o] = u2[q];
    if (!a.last) {
#pragma unroll
      for (int f = 2; f < 6; ++f) a.out.p[B1 + f][o] = sm[sxi(f, id, PL)];
    }
  }
}

#include "pd_sweep.cuh"

// ------------------------------------------------------------------------
// Register-strip variant.  Tile = 32 columns x (BY*PY) rows; lane = column,
// warp w owns rows [w*PY, w*PY+PY) as a vertical strip held entirely in
// registers (u, u-bar, p, gathered gradient, rho0, threshold, 1/|grad|^2).
// x-neighbours come from warp shuffles (u-bar at x+1 in the dual step, p at
// x-1 in the primal step); y-neighbours are in the same thread except at the
// strip ends, where one row per warp is exchanged through shared memory
// (each warp publishes its first-row u-bar for the warp above and its
// last-row p for the warp below).  Lanes / warps at the tile edge read their
// own values instead of a neighbour's: those pixels are halo (or image
// border, where the reference does not read the neighbour), exactly as in
// k_pd_tile.  Same arithmetic, same operation order, bit-identical results.
// ------------------------------------------------------------------------
template <int BY, int PY, int MINB>
__global__ void __launch_bounds__(32 * BY, MINB) k_pd_strip(const PDArgs a) {
  constexpr int TH = BY * PY;
  __shared__ double s_b1[BY][32], s_b2[BY][32];    // first-row u-bar of each warp
  __shared__ double s_p12[BY][32], s_p22[BY][32];  // last-row p of each warp
  const int W = a.w, H = a.h;
  const int step_x = 32 - 2 * a.halo, step_y = TH - 2 * a.halo;
  const int ox = blockIdx.x * step_x - a.halo;
  const int oy = blockIdx.y * step_y - a.halo;
  const int64_t so = blockIdx.z * a.cap;
  const int lane = threadIdx.x, w = threadIdx.y;
  const int gc = ox + lane;
  const int gr0 = oy + w * PY;
  const bool cin = gc >= 0 && gc < W;
  const bool fR = gc < W - 1, fL = gc > 0, fLastC = gc == W - 1;
  const int wd = w < BY - 1 ? w + 1 : w;  // warp below / above (self at tile edge)
  const int wu = w > 0 ? w - 1 : w;

  const double tl = a.tau * a.lam;
  double u1[PY], u2[PY], b1[PY], b2[PY], p11[PY], p12[PY], p21[PY], p22[PY];
  double gx[PY], gy[PY], r0[PY], thr[PY], ig2[PY];
#pragma unroll
  for (int k = 0; k < PY; ++k) {
    const int gr = gr0 + k;
    const bool in = cin && gr >= 0 && gr < H;
    const int64_t o = so + (int64_t)gr * W + gc;
    double vu1 = 0, vu2 = 0, vb1 = 0, vb2 = 0, q11 = 0, q12 = 0, q21 = 0, q22 = 0;
    double vgx = 0, vgy = 0, vr0 = 0;
    if (in) {
      vu1 = a.in.p[U1][o];
      vu2 = a.in.p[U2][o];
      if (a.first) {
        vb1 = vu1;  // ub = u, p = 0 at the start of a warp (optflow.py:169-174)
        vb2 = vu2;
      } else {
        vb1 = a.in.p[B1][o];
        vb2 = a.in.p[B2][o];
        q11 = a.in.p[P11][o];
        q12 = a.in.p[P12][o];
        q21 = a.in.p[P21][o];
        q22 = a.in.p[P22][o];
      }
      vgx = a.gx[o];
      vgy = a.gy[o];
      vr0 = a.r0[o];
    }
    u1[k] = vu1;
    u2[k] = vu2;
    b1[k] = vb1;
    b2[k] = vb2;
    p11[k] = q11;
    p12[k] = q12;
    p21[k] = q21;
    p22[k] = q22;
    gx[k] = vgx;
    gy[k] = vgy;
    r0[k] = vr0;
    const double g2 = vgx * vgx + vgy * vgy;  // optflow.py:163
    ig2[k] = g2 > 1e-12 ? 1.0 / g2 : 0.0;     // == 1/max(g2,1e-12) where safe
    thr[k] = tl * g2;                          // optflow.py:176
  }
  s_b1[w][lane] = b1[0];
  s_b2[w][lane] = b2[0];
  __syncthreads();

  for (int it = 0; it < a.iters; ++it) {
    // ---- dual ascent with Huber prox and unit-ball projection (:180-191)
    const double db1 = s_b1[wd][lane], db2 = s_b2[wd][lane];  // row below the strip
#pragma unroll
    for (int k = 0; k < PY; ++k) {
      const int gr = gr0 + k;
      const double r1 = __shfl_down_sync(0xffffffffu, b1[k], 1);
      const double r2 = __shfl_down_sync(0xffffffffu, b2[k], 1);
      const double d1 = k < PY - 1 ? b1[k + 1] : db1;
      const double d2 = k < PY - 1 ? b2[k + 1] : db2;
      const bool fD = gr < H - 1;
      const double a1x = fR ? r1 - b1[k] : 0.0;
      const double a1y = fD ? d1 - b1[k] : 0.0;
      const double a2x = fR ? r2 - b2[k] : 0.0;
      const double a2y = fD ? d2 - b2[k] : 0.0;
      double q11 = (p11[k] + a.sigma * a1x) * a.shrink;
      double q12 = (p12[k] + a.sigma * a1y) * a.shrink;
      double q21 = (p21[k] + a.sigma * a2x) * a.shrink;
      double q22 = (p22[k] + a.sigma * a2y) * a.shrink;
      if (q11 * q11 + q12 * q12 > 0.999999) {
        const double n1 = np_max(1.0, glibc_hypot(q11, q12));
        q11 = q11 / n1;
        q12 = q12 / n1;
      }
      if (q21 * q21 + q22 * q22 > 0.999999) {
        const double n2 = np_max(1.0, glibc_hypot(q21, q22));
        q21 = q21 / n2;
        q22 = q22 / n2;
      }
      p11[k] = q11;
      p12[k] = q12;
      p21[k] = q21;
      p22[k] = q22;
    }
    s_p12[w][lane] = p12[PY - 1];
    s_p22[w][lane] = p22[PY - 1];
    __syncthreads();
    // ---- primal descent + TV-L1 shrinkage (:194-208)
    const double up12 = s_p12[wu][lane], up22 = s_p22[wu][lane];  // row above the strip
#pragma unroll
    for (int k = 0; k < PY; ++k) {
      const int gr = gr0 + k;
      const double l11 = __shfl_up_sync(0xffffffffu, p11[k], 1);
      const double l21 = __shfl_up_sync(0xffffffffu, p21[k], 1);
      const double a12 = k > 0 ? p12[k - 1] : up12;
      const double a22 = k > 0 ? p22[k - 1] : up22;
      // divergence (imageops.py:41-50): dx + dy with border rules
      const double dx1 = !fL ? p11[k] : (fLastC ? -l11 : p11[k] - l11);
      const double dx2 = !fL ? p21[k] : (fLastC ? -l21 : p21[k] - l21);
      const double dy1 = gr <= 0 ? p12[k] : (gr == H - 1 ? -a12 : p12[k] - a12);
      const double dy2 = gr <= 0 ? p22[k] : (gr == H - 1 ? -a22 : p22[k] - a22);
      const double v1 = u1[k] + a.tau * (dx1 + dy1);
      const double v2 = u2[k] + a.tau * (dx2 + dy2);
      const double rho = r0[k] + gx[k] * v1 + gy[k] * v2;
      const bool lo = rho < -thr[k];
      const bool hi = rho > thr[k];
      double d = lo ? tl : (hi ? -tl : -rho * ig2[k]);
      // ig2 == 0 exactly when |grad|^2 <= 1e-12 (the reference's ~safe)
      d = (ig2[k] != 0.0 || lo || hi) ? d : 0.0;
      const double n1 = v1 + d * gx[k];
      const double n2 = v2 + d * gy[k];
      b1[k] = 2.0 * n1 - u1[k];
      b2[k] = 2.0 * n2 - u2[k];
      u1[k] = n1;
      u2[k] = n2;
    }
    s_b1[w][lane] = b1[0];
    s_b2[w][lane] = b2[0];
    __syncthreads();
  }

  // ---- write back the exact interior
  if (!cin || lane < a.halo || lane >= 32 - a.halo) return;
#pragma unroll
  for (int k = 0; k < PY; ++k) {
    const int lr = w * PY + k, gr = gr0 + k;
    if (gr < 0 || gr >= H || lr < a.halo || lr >= TH - a.halo) continue;
    const int64_t o = so + (int64_t)gr * W + gc;
    a.out.p[U1][o] = u1[k];
    a.out.p[U2][o] = u2[k];
    a.out.p[B1][o] = b1[k];
    a.out.p[B2][o] = b2[k];
    a.out.p[P11][o] = p11[k];
    a.out.p[P12][o] = p12[k];
    a.out.p[P21][o] = p21[k];
    a.out.p[P22][o] = p22[k];
  }
}

// ------------------------------------------------------------------------
// Cluster-resident coarse level.  A thread-block cluster of CX x CY CTAs
// (64x32 tile each, <= 16 CTAs, 1 per SM) holds an entire pyramid level on
// chip and runs the whole _solve_level (optflow.py:147-214) in ONE launch:
// bilinear upsample of the coarser flow (:244-249), then per warp the
// linearisation (:158-176), all primal-dual iterations and the 3x3 median
// (:210-211).  Tiles do not overlap: after every half step each CTA copies
// its neighbours' edge rows/columns of the just-written field into its apron
// through distributed shared memory (cluster.sync() + map_shared_rank), so
// no halo is recomputed and no state leaves the chip until the level ends.
// ------------------------------------------------------------------------
struct LevelArgs {
  const double *i0, *i1;  // x255 pyramid level of image 0; per-image stride ps
  int64_t ps;
  const double *ix, *iy;    // gradient of i1, [nb][cap]
  const double *uc1, *uc2;  // coarser flow [nb][cap], null at the coarsest level
  int wc, hc;
  double rx, ry, sx, sy;  // wc/w, hc/h, w/wc, h/hc
  double *uo1, *uo2;      // this level's flow out [nb][cap]
  int w, h;
  int64_t cap;
  int warps, iters;
  double tau, lam, sigma, shrink;
};

constexpr int kCTW = 64, kCBY = 16, kCPY = 2;  // 64 x 32 tile, 512 threads
using CGeom = PDGeom<kCTW, kCBY, kCPY>;

struct ClusterExchange {
  double *sm;
  int tid, bx, by, cx, cy;
  // neighbour ranks (x fastest) or -1 outside the cluster
  __device__ __forceinline__ int rank(int x, int y) const {
    return (x < 0 || y < 0 || x >= cx || y >= cy) ? -1 : x + y * cx;
  }
  // copy `count` doubles at local offsets dst[k] <- neighbour's src[k]
  __device__ __forceinline__ void pull(int nrank, int plane, int dst, int src, int dstride,
                                       int sstride, int count, int t0) {
    if (nrank < 0) return;
    cg::cluster_group cl = cg::this_cluster();
    const double *theirs = cl.map_shared_rank(sm, nrank);
    const int k = tid - t0;  // field `plane` = b1 b2 p11 p12 p21 p22 index
    if (k >= 0 && k < count)
      sm[sxi(plane, dst + k * dstride, CGeom::PLANE)] =
          theirs[sxi(plane, src + k * sstride, CGeom::PLANE)];
  }
  // p after the dual step: left apron column <- left neighbour's last column
  // (p11, p21); top apron row <- upper neighbour's last row (p12, p22)
  __device__ void after_dual() {
    cg::this_cluster().sync();
    constexpr int SP = CGeom::SP, TW = kCTW, TH = CGeom::TH;
    const int l = rank(bx - 1, by), u = rank(bx, by - 1);
    pull(l, 2, SP, SP + TW, SP, SP, TH, 0);               // p11 col
    pull(l, 4, SP, SP + TW, SP, SP, TH, TH);              // p21 col
    pull(u, 3, 1, TH * SP + 1, 1, 1, TW, 2 * TH);         // p12 row
    pull(u, 5, 1, TH * SP + 1, 1, 1, TW, 2 * TH + TW);    // p22 row
    __syncthreads();
  }
  // u-bar after the primal step: right apron column <- right neighbour's
  // first column; bottom apron row <- lower neighbour's first row
  __device__ void after_primal() {
    cg::this_cluster().sync();
    constexpr int SP = CGeom::SP, TW = kCTW, TH = CGeom::TH;
    const int r = rank(bx + 1, by), d = rank(bx, by + 1);
    pull(r, 0, SP + TW + 1, SP + 1, SP, SP, TH, 0);               // b1 col
    pull(r, 1, SP + TW + 1, SP + 1, SP, SP, TH, TH);              // b2 col
    pull(d, 0, (TH + 1) * SP + 1, SP + 1, 1, 1, TW, 2 * TH);      // b1 row
    pull(d, 1, (TH + 1) * SP + 1, SP + 1, 1, 1, TW, 2 * TH + TW); // b2 row
    __syncthreads();
  }
};

__global__ void __launch_bounds__(32 * kCBY, 1) k_level_cluster(const LevelArgs a) {
  constexpr int NX = CGeom::NX, TH = CGeom::TH, NP = CGeom::NP, SP = CGeom::SP;
  constexpr int PL = CGeom::PLANE, TW = kCTW, BY = kCBY;
  extern __shared__ __align__(16) double sm[];
  const int W = a.w, H = a.h;
  const int ox = blockIdx.x * TW, oy = blockIdx.y * TH;
  const int64_t so = blockIdx.z * a.cap;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int base = (ty + 1) * SP + tx + 1;
  ClusterExchange xch{sm, tid, (int)blockIdx.x, (int)blockIdx.y, (int)gridDim.x, (int)gridDim.y};
  double2 *const queue = reinterpret_cast<double2 *>(sm + 6 * PL) + ty * (2 * NP * 32);
  const double *i0 = a.i0 + blockIdx.z * a.ps, *i1 = a.i1 + blockIdx.z * a.ps;

  for (int k = tid; k < 6 * PL; k += 32 * BY) sm[k] = 0.0;  // aprons start finite (all planes)
  __syncthreads();

  // ---- initial flow: zero at the coarsest level, else upsampled (:244-249)
  double u1[NP], u2[NP];
  unsigned fl[NP];
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const int gc = ox + tx + 32 * (q % NX), gr = oy + ty + BY * (q / NX);
    u1[q] = 0.0;
    u2[q] = 0.0;
    if (a.uc1 && gc < W && gr < H) {
      const double x = ((double)gc + 0.5) * a.rx - 0.5;
      const double y = ((double)gr + 0.5) * a.ry - 0.5;
      u1[q] = bsample(a.uc1 + so, a.wc, a.hc, x, y) * a.sx;
      u2[q] = bsample(a.uc2 + so, a.wc, a.hc, x, y) * a.sy;
    }
    fl[q] = (gc < W - 1 ? FL_R : 0u) | (gr < H - 1 ? FL_D : 0u) | (gc > 0 ? FL_L : 0u) |
            (gc == W - 1 ? FL_LASTC : 0u) | (gr > 0 ? FL_U : 0u) | (gr == H - 1 ? FL_LASTR : 0u);
  }

  const double tl = a.tau * a.lam;
  for (int wp = 0; wp < a.warps; ++wp) {
    // ---- linearise at the current flow (:158-176); ub = u, p = 0
    double gx[NP], gy[NP], r0[NP], thr[NP], ig2[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int gc = ox + tx + 32 * (q % NX), gr = oy + ty + BY * (q / NX);
      double vgx = 0.0, vgy = 0.0, vr0 = 0.0;
      if (gc < W && gr < H) {
        const double mx = (double)gc + u1[q], my = (double)gr + u2[q];
        const double v = bsample(i1, W, H, mx, my);
        vgx = bsample(a.ix + so, W, H, mx, my);
        vgy = bsample(a.iy + so, W, H, mx, my);
        vr0 = v - i0[(int64_t)gr * W + gc] - vgx * u1[q] - vgy * u2[q];
      }
      gx[q] = vgx;
      gy[q] = vgy;
      r0[q] = vr0;
      const double g2 = vgx * vgx + vgy * vgy;
      const bool ok = g2 > 1e-12;
      ig2[q] = ok ? 1.0 / (g2 > 1e-12 ? g2 : 1e-12) : 0.0;
      thr[q] = tl * g2;
      fl[q] = (fl[q] & ~(unsigned)FL_OK) | (ok ? FL_OK : 0u);
      const int id = base + (q / NX) * BY * SP + 32 * (q % NX);
      sm[sxi(0, id, PL)] = u1[q];
      sm[sxi(1, id, PL)] = u2[q];
#pragma unroll
      for (int f = 2; f < 6; ++f) sm[sxi(f, id, PL)] = 0.0;
    }
    xch.after_primal();  // publish u-bar edges before the first dual step

    pd_iterate<kCTW, kCBY, kCPY, false, false>(a.iters, sm, base, tx, fl, u1, u2, gx, gy, r0, thr, ig2, a.tau,
                                 tl, a.sigma, a.shrink, queue, xch);

    // ---- 3x3 median of u1, u2 with replicated borders (:210-211).  The p
    // planes are free now (no neighbour reads them after the last exchange).
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int id = base + (q / NX) * BY * SP + 32 * (q % NX);
      sm[sxi(2, id, PL)] = u1[q];
      sm[sxi(3, id, PL)] = u2[q];
    }
    cg::this_cluster().sync();
    {  // apron ring incl. corners from the 8 neighbours
      cg::cluster_group cl = cg::this_cluster();
      for (int k = tid; k < 2 * (2 * TW + 2 * TH + 4); k += 32 * BY) {
        const int plane = 2 + (k & 1);
        const int e = k >> 1;
        int lr, lc;  // apron cell in local coordinates (-1..TH, -1..TW)
        if (e < TW) { lr = -1; lc = e; }
        else if (e < 2 * TW) { lr = TH; lc = e - TW; }
        else if (e < 2 * TW + TH) { lr = e - 2 * TW; lc = -1; }
        else if (e < 2 * TW + 2 * TH) { lr = e - 2 * TW - TH; lc = TW; }
        else { const int c = e - 2 * TW - 2 * TH; lr = (c & 2) ? TH : -1; lc = (c & 1) ? TW : -1; }
        const int nx = lc < 0 ? -1 : (lc >= TW ? 1 : 0), ny = lr < 0 ? -1 : (lr >= TH ? 1 : 0);
        const int nr = xch.rank(xch.bx + nx, xch.by + ny);
        if (nr < 0) continue;
        const int sr = lr - ny * TH, sc = lc - nx * TW;  // cell in the neighbour's frame
        sm[sxi(plane, (lr + 1) * SP + lc + 1, PL)] =
            cl.map_shared_rank(sm, nr)[sxi(plane, (sr + 1) * SP + sc + 1, PL)];
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int gc = ox + tx + 32 * (q % NX), gr = oy + ty + BY * (q / NX);
      if (gc >= W || gr >= H) continue;
      double v1[9], v2[9];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int rr = min(max(gr - 1 + i, 0), H - 1) - oy;
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const int cc = min(max(gc - 1 + j, 0), W - 1) - ox;
          v1[i * 3 + j] = sm[sxi(2, (rr + 1) * SP + cc + 1, PL)];
          v2[i * 3 + j] = sm[sxi(3, (rr + 1) * SP + cc + 1, PL)];
        }
      }
      u1[q] = median9(v1);
      u2[q] = median9(v2);
    }
    cg::this_cluster().sync();  // neighbours are done reading our u planes
  }

#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const int gc = ox + tx + 32 * (q % NX), gr = oy + ty + BY * (q / NX);
    if (gc >= W || gr >= H) continue;
    a.uo1[so + (int64_t)gr * W + gc] = u1[q];
    a.uo2[so + (int64_t)gr * W + gc] = u2[q];
  }
}

// ------------------------------------------------------------------------
// Persistent, software-pipelined variant of k_pd_tile.  The launch cost of
// the tiled kernel is (load+store, HBM-bound) + K x (iteration, issue-bound)
// with almost no overlap between the two (tools/pd_cost_model.sh).  Here a
// grid of one CTA per SM walks the tiles; while a CTA iterates on tile t its
// threads' cp.async copies (LDGSTS, zero-fill outside the image) are already
// streaming tile t+1 into a shared-memory staging buffer, and the interior of
// tile t is written back with plain stores that drain during the next tile's
// compute.  Every thread stages exactly the pixels it owns, so the hand-off
// needs only its own cp.async.wait_group.
// ------------------------------------------------------------------------
constexpr int kNStage = 11;  // u1 u2 b1 b2 p11 p12 p21 p22 gx gy rho0

template <int TW, int BY, int PY>
struct PersistGeom {
  using G = PDGeom<TW, BY, PY>;
  static constexpr int TPX = TW * G::TH;  // pixels per tile
  // exchange planes (no projection queue) + staging
  static constexpr size_t smem = 6 * G::PLANE * sizeof(double) + kNStage * TPX * sizeof(double) +
                                 BY * 2 * G::NP * 32 * 16;
};


template <int TW, int BY, int PY>
__global__ void __launch_bounds__(32 * BY, 1) k_pd_persist(const PDArgs a) {
  using G = PDGeom<TW, BY, PY>;
  using PG = PersistGeom<TW, BY, PY>;
  constexpr int NX = G::NX, TH = G::TH, NP = G::NP, SP = G::SP, PL = G::PLANE, TPX = PG::TPX;
  extern __shared__ __align__(16) double sm[];
  double *const stage = sm + 6 * PL;
  double2 *const queue =
      reinterpret_cast<double2 *>(stage + kNStage * TPX) + threadIdx.y * (2 * NP * 32);
  const int W = a.w, H = a.h;
  const int step_x = TW - 2 * a.halo, step_y = TH - 2 * a.halo;
  const int ntx = a.halo ? (W + step_x - 1) / step_x : 1;
  const int nty = a.halo ? (H + step_y - 1) / step_y : 1;
  const int ntiles = ntx * nty * a.nb;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  const int base = (ty + 1) * SP + tx + 1;
  const int nload = a.first ? 5 : kNStage;  // first launch of a warp: u, gx, gy, rho0
  const double tl = a.tau * a.lam;

  for (int k = tid; k < 6 * PL; k += 32 * BY) sm[k] = 0.0;  // apron stays zero

  auto tile_origin = [&](int t, int &ox, int &oy, int64_t &so) {
    const int bz = t / (ntx * nty), r = t % (ntx * nty);
    ox = (r % ntx) * step_x - a.halo;
    oy = (r / ntx) * step_y - a.halo;
    so = (int64_t)bz * a.cap;
  };
  // stage the pixels this thread owns; plane order: U1 U2 (B1 B2 P11..P22) gx gy r0
  auto issue_loads = [&](int t) {
    int ox, oy;
    int64_t so;
    tile_origin(t, ox, oy, so);
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int lc = tx + 32 * (q % NX), lr = ty + BY * (q / NX);
      const int gc = ox + lc, gr = oy + lr;
      const bool in = gc >= 0 && gc < W && gr >= 0 && gr < H;
      const int64_t o = in ? so + (int64_t)gr * W + gc : 0;
      const int li = lr * TW + lc;
      cp_async8(stage + 0 * TPX + li, a.in.p[U1] + o, in);
      cp_async8(stage + 1 * TPX + li, a.in.p[U2] + o, in);
      if (!a.first) {
#pragma unroll
        for (int f = B1; f <= P22; ++f) cp_async8(stage + f * TPX + li, a.in.p[f] + o, in);
      }
      cp_async8(stage + 8 * TPX + li, a.gx + o, in);
      cp_async8(stage + 9 * TPX + li, a.gy + o, in);
      cp_async8(stage + 10 * TPX + li, a.r0 + o, in);
    }
    cp_async_commit();
  };
  (void)nload;

  int t = blockIdx.x;
  if (t < ntiles) issue_loads(t);
  for (; t < ntiles; t += gridDim.x) {
    int ox, oy;
    int64_t so;
    tile_origin(t, ox, oy, so);
    cp_async_wait_all();  // this thread's staged pixels of tile t have landed
    double u1[NP], u2[NP], gx[NP], gy[NP], r0[NP], thr[NP], ig2[NP];
    unsigned fl[NP];
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int lc = tx + 32 * (q % NX), lr = ty + BY * (q / NX);
      const int gc = ox + lc, gr = oy + lr;
      const int li = lr * TW + lc;
      u1[q] = stage[0 * TPX + li];
      u2[q] = stage[1 * TPX + li];
      gx[q] = stage[8 * TPX + li];
      gy[q] = stage[9 * TPX + li];
      r0[q] = stage[10 * TPX + li];
      const double g2 = gx[q] * gx[q] + gy[q] * gy[q];  // optflow.py:163
      const bool ok = g2 > 1e-12;
      ig2[q] = ok ? 1.0 / (g2 > 1e-12 ? g2 : 1e-12) : 0.0;
      thr[q] = tl * g2;
      fl[q] = (gc < W - 1 ? FL_R : 0u) | (gr < H - 1 ? FL_D : 0u) | (gc > 0 ? FL_L : 0u) |
              (gc == W - 1 ? FL_LASTC : 0u) | (gr > 0 ? FL_U : 0u) |
              (gr == H - 1 ? FL_LASTR : 0u) | (ok ? FL_OK : 0u);
      const int id = base + (q / NX) * BY * SP + 32 * (q % NX);
      if (a.first) {
        sm[sxi(0, id, PL)] = u1[q];  // ub = u, p = 0 (optflow.py:169-174)
        sm[sxi(1, id, PL)] = u2[q];
#pragma unroll
        for (int f = 2; f < 6; ++f) sm[sxi(f, id, PL)] = 0.0;
      } else {
#pragma unroll
        for (int f = 0; f < 6; ++f) sm[sxi(f, id, PL)] = stage[(2 + f) * TPX + li];
      }
    }
    __syncthreads();  // exchange planes hold tile t (and tile t-1 is finished)
    if (t + (int)gridDim.x < ntiles) issue_loads(t + gridDim.x);  // overlaps the compute

    BlockBarrier bar;
    if (a.pow2)
      pd_iterate<TW, BY, PY, true, false>(a.iters, sm, base, tx, fl, u1, u2, gx, gy, r0, thr,
                                          ig2, a.tau, tl, a.sigma, a.shrink, queue, bar);
    else
      pd_iterate<TW, BY, PY, false, false>(a.iters, sm, base, tx, fl, u1, u2, gx, gy, r0, thr,
                                           ig2, a.tau, tl, a.sigma, a.shrink, queue, bar);

    // ---- write back the exact interior (drains during the next tile)
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int lc = tx + 32 * (q % NX), lr = ty + BY * (q / NX);
      const int gc = ox + lc, gr = oy + lr;
      if (gc < 0 || gc >= W || gr < 0 || gr >= H) continue;
      if (lc < a.halo || lc >= TW - a.halo || lr < a.halo || lr >= TH - a.halo) continue;
      const int id = base + (q / NX) * BY * SP + 32 * (q % NX);
      const int64_t o = so + (int64_t)gr * W + gc;
      a.out.p[U1][o] = u1[q];
      a.out.p[U2][o] = u2[q];
#pragma unroll
      for (int f = 0; f < 6; ++f) a.out.p[B1 + f][o] = sm[sxi(f, id, PL)];
    }
  }
}

int env_int(const char *name, int dflt) {
  const char *v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

// Launch configurations (tile width x height, threads, min CTAs/SM).
struct PDConfig {
  int idx, tw, th, by;
  void (*fn)(PDArgs);
  size_t smem;
  bool persistent = false;
  size_t smem_cq = 0;  // k_pd_tile with the CTA-wide queue (PDArgs::cq)
  bool tile = false;    // k_pd_tile: half-step schedule (PDArgs::nhalf)
  void (*fn_mid)(PDArgs) = nullptr;  // k_pd_tile<..., MID>: middle (P D)x4 launches, halo 4
  void (*fn_cl)(PDArgs) = nullptr;   // 2x1 cluster variants (FT_PD_CL=1)
  void (*fn_mid_cl)(PDArgs) = nullptr;
};

template <int TW, int BY, int PY>
PDConfig make_persist_cfg(int idx) {
  using G = PDGeom<TW, BY, PY>;
  return PDConfig{idx, TW, G::TH, BY, &k_pd_persist<TW, BY, PY>, PersistGeom<TW, BY, PY>::smem,
                  true};
}

template <int BY, int PY, int MINB>
PDConfig make_strip_cfg(int idx) {
  return PDConfig{idx, 32, BY * PY, BY, &k_pd_strip<BY, PY, MINB>, 0};
}

template <int TW, int BY, int PY, int MINB>
PDConfig make_cfg(int idx) {
  using G = PDGeom<TW, BY, PY>;
  PDConfig c{idx, TW, G::TH, BY, &k_pd_tile<TW, BY, PY, MINB>, G::smem};
  c.smem_cq = 6 * G::PLANE * sizeof(double) + (2 * G::NP * 32 * BY + 2) * sizeof(int);
  c.tile = true;
  if (G::TH == 32) c.fn_mid = &k_pd_tile<TW, BY, PY, MINB, G::TH == 32>;
  if (TW == 32 && G::TH == 32 && BY == 16) {
    c.fn_cl = &k_pd_tile<TW, BY, PY, MINB, false, TW == 32 && BY == 16>;
    c.fn_mid_cl = &k_pd_tile<TW, BY, PY, MINB, G::TH == 32, TW == 32 && BY == 16>;
  }
  return c;
}

// index: 0 = 32x32/256thr, 1 = 32x32/512thr, 2 = 64x32/512thr, 3 = 64x32/256thr
inline PDConfig pd_config(int i) {
  switch (i) {
    case 1: return make_cfg<32, 16, 2, 2>(1);
    case 2: return make_cfg<64, 16, 2, 2>(2);
    case 3: return make_cfg<64, 8, 4, 1>(3);
    // register strips: 32 x (BY*PY) tiles
    case 4: return make_strip_cfg<8, 4, 1>(4);
    case 5: return make_strip_cfg<8, 3, 2>(5);
    case 6: return make_strip_cfg<16, 3, 1>(6);
    case 7: return make_strip_cfg<16, 2, 1>(7);
    case 8: return make_strip_cfg<8, 2, 2>(8);
    case 9: return make_strip_cfg<16, 4, 1>(9);
    case 10: return make_cfg<32, 16, 2, 1>(10);
    case 11: return make_cfg<32, 32, 1, 1>(11);
    case 12: return make_persist_cfg<32, 16, 2>(12);
    case 13: return make_persist_cfg<32, 8, 4>(13);
    default: return make_cfg<32, 8, 4, 2>(0);
  }
}

int pd_launch(const PDConfig &c, const PDArgs &a, int nb, cudaStream_t s) {
  static bool attr_done[32] = {};
  if (!attr_done[c.idx]) {
    FT_CUDA_TRY(cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)c.smem));
    attr_done[c.idx] = true;
  }
  const int step_x = c.tw - 2 * a.halo, step_y = c.th - 2 * a.halo;
  const dim3 grid(a.halo ? (a.w + step_x - 1) / step_x : 1, a.halo ? (a.h + step_y - 1) / step_y : 1,
                  nb);
  if (c.persistent) {  // one CTA per SM walking all tiles
    static int sms = 0;
    if (!sms) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (sms <= 0) sms = kSMs;
    }
    const int ntiles = grid.x * grid.y * grid.z;
    c.fn<<<ntiles < sms ? ntiles : sms, dim3(32, c.by), c.smem, s>>>(a);
    count_launch();
    return FT_OK;
  }
  // the CTA-wide projection queue needs 4 B per pair instead of the per-warp
  // 16 B: smaller carve-out, larger L1
  const size_t smem = c.tile ? c.smem_cq : c.smem;
  const bool mid = c.fn_mid && !a.first && !a.last && a.nhalf == 8 && a.halo == 4 && a.cone_rows &&
                   c.th == 32 && env_int("FT_PD_MID", 1);
  if (mid && !attr_done[16 + c.idx]) {
    FT_CUDA_TRY(cudaFuncSetAttribute(c.fn_mid, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)c.smem));
    attr_done[16 + c.idx] = true;
  }
  if (c.fn_cl && a.halo > 0 && env_int("FT_PD_CL", 0)) {
    void (*fn)(PDArgs) = mid ? c.fn_mid_cl : c.fn_cl;
    static void (*cl_attr[4])(PDArgs) = {};
    const int ck = (mid ? 1 : 0);
    if (cl_attr[ck] != fn) {
      FT_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem));
      cl_attr[ck] = fn;
    }
    const int rx = 2 * c.tw - 2 * a.halo;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * ((a.w + rx - 1) / rx), grid.y, grid.z);
    cfg.blockDim = dim3(32, c.by);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    FT_CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, a));
    count_launch();
    return FT_OK;
  }
  (mid ? c.fn_mid : c.fn)<<<grid, dim3(32, c.by), smem, s>>>(a);
  count_launch();
  return FT_OK;
}


// k_pd_sweep launches: `nh` half-steps, starting with a dual step when
// `first` (the warp's first launch).  pow2 time steps only (the default);
// other tau use k_pd_tile.
constexpr int kSweepSlots = 4;  // input ring rows (prefetch distance 1 row)
constexpr int kSweepMinB = 8;   // resident warps per SM

using SweepFn = void (*)(SweepArgs);

int sweep_launch(const PDArgs &pa, int nh, bool first, int nb, cudaStream_t s) {
  SweepFn fn = nullptr;
  size_t smem = 0;
#define FT_SWEEP_CASE(NH_, FD_)                                                  \
  case (FD_ ? 0 : 16) + NH_:                                                     \
    if (cols == 2 && NH_ <= 4) {                                                 \
      fn = &k_pd_sweep<NH_, FD_, true, kSweepSlots, 6, (NH_ <= 4 ? 2 : 1)>;     \
      smem = SweepGeom<NH_, kSweepSlots, (NH_ <= 4 ? 2 : 1)>::smem_per_warp;    \
    } else {                                                                     \
      fn = &k_pd_sweep<NH_, FD_, true, kSweepSlots, (NH_ <= 4 ? 16 : kSweepMinB), 1>; \
      smem = SweepGeom<NH_, kSweepSlots, 1>::smem_per_warp;                      \
      cols = 1;                                                                  \
    }                                                                            \
    break;
  int cols = env_int("FT_SWEEP_COLS", 2);
  switch ((first ? 0 : 16) + nh) {
    FT_SWEEP_CASE(2, true)
    FT_SWEEP_CASE(3, true)
    FT_SWEEP_CASE(4, true)
    FT_SWEEP_CASE(6, true)
    FT_SWEEP_CASE(7, true)
    FT_SWEEP_CASE(1, false)
    FT_SWEEP_CASE(3, false)
    FT_SWEEP_CASE(4, false)
    FT_SWEEP_CASE(5, false)
    FT_SWEEP_CASE(7, false)
    FT_SWEEP_CASE(8, false)
    default: return fail(FT_EINVAL, "k_pd_sweep: unsupported half-step count");
  }
#undef FT_SWEEP_CASE
  static SweepFn attr_done[64] = {};
  const int key = (first ? 0 : 16) + nh + (cols == 2 ? 32 : 0);
  if (attr_done[key] != fn) {
    FT_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
    attr_done[key] = fn;
  }
  SweepArgs a;
  a.in = pa.in;
  a.out = pa.out;
  a.gx = pa.gx;
  a.gy = pa.gy;
  a.r0 = pa.r0;
  a.w = pa.w;
  a.h = pa.h;
  a.cap = pa.cap;
  a.seg = std::max(1, env_int("FT_SWEEP_SEG", 64));
  const int khalo = cols == 1 ? (nh + 1) / 2 : ((nh + 1) / 2 + 1) / 2 * 2;
  const int strip = 32 * cols - 2 * khalo;  // interior columns per warp
  a.nstrips = (pa.w + strip - 1) / strip;
  sweep_cone(first, nh, a.cA, a.cB);
  a.tau = pa.tau;
  a.tl = pa.tau * pa.lam;
  a.sigma = pa.sigma;
  a.shrink = pa.shrink;
  const dim3 grid(a.nstrips, (pa.h + a.seg - 1) / a.seg, nb);
  fn<<<grid, dim3(32, 1), smem, s>>>(a);
  count_launch();
  return FT_OK;
}

// tile configuration + halo used for a level of w x h
struct PDPlan {
  PDConfig cfg;
  int halo;
};


PDPlan pd_plan(int w, int h) {
  // coarse levels that fit one tile run resident (no halo, all iterations)
  for (int i : {0, 2}) {
    PDConfig c = pd_config(i);
    if (w <= c.tw && h <= c.th) return PDPlan{c, 0};
  }
  // defaults from the sweep on B200 (profiles/README.md): 32x32 tile,
  // 512 threads, halo 4
  return PDPlan{pd_config(env_int("FT_PD_CFG", 1)), env_int("FT_PD_HALO", 4)};
}

// tau = 2^k (then sigma = 1/(8 tau) = 2^(-k-3) too): products by them are exact
inline int pow2_params(double tau) {
  int e = 0;
  return tau > 0.0 && std::frexp(tau, &e) == 0.5 ? 1 : 0;
}

bool use_sweep(const PDPlan &plan, double tau) {
  return plan.cfg.tile && plan.halo == 4 && pow2_params(tau) && env_int("FT_PD_SWEEP", 0) != 0;
}

inline dim3 grid2d(int w, int h, int nb) { return dim3((w + 31) / 32, (h + 7) / 8, nb); }

const char *const kLevelNames[8] = {"flow level 0", "flow level 1", "flow level 2",
                                    "flow level 3", "flow level 4", "flow level 5",
                                    "flow level 6", "flow level 7+"};

cudaLaunchConfig_t level_cluster_cfg(int w, int h, int nb, cudaStream_t s,
                                     cudaLaunchAttribute *attr) {
  const int cx = (w + kCTW - 1) / kCTW, cy = (h + CGeom::TH - 1) / CGeom::TH;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cx, cy, nb);
  cfg.blockDim = dim3(32, kCBY, 1);
  cfg.dynamicSmemBytes = CGeom::smem;
  cfg.stream = s;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cx;
  attr[0].val.clusterDim.y = cy;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cfg;
}

int level_cluster_setup() {
  static int done = 0;
  if (done) return FT_OK;
  FT_CUDA_TRY(cudaFuncSetAttribute(k_level_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed,
                                   1));
  FT_CUDA_TRY(cudaFuncSetAttribute(k_level_cluster, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)CGeom::smem));
  done = 1;
  return FT_OK;
}

// Can level w x h run as one cluster (<= 16 CTAs, schedulable)?  Opt-in with
// FT_CLUSTER=1: on B200 the per-iteration latency of one 64x32 CTA makes it
// slower than the tiled kernels (profiles/r01_launches_cluster.md); FT_CLUSTER=0
// disables the path (tiled kernels for every level).
bool cluster_level_ok(int w, int h) {
  if (!env_int("FT_CLUSTER", 0)) return false;
  const int cx = (w + kCTW - 1) / kCTW, cy = (h + CGeom::TH - 1) / CGeom::TH;
  if (cx * cy > 16) return false;
  static int cache[17][17];  // 0 unknown, 1 yes, 2 no
  int &c = cache[cx][cy];
  if (c == 0) {
    c = 2;
    if (level_cluster_setup() == FT_OK) {
      cudaLaunchAttribute attr[1];
      cudaLaunchConfig_t cfg = level_cluster_cfg(w, h, 1, nullptr, attr);
      int n = 0;
      if (cudaOccupancyMaxActiveClusters(&n, k_level_cluster, &cfg) == cudaSuccess && n > 0) c = 1;
      cudaGetLastError();
    }
  }
  return c == 1;
}

int launch_level_cluster(const LevelArgs &a, int nb, cudaStream_t s) {
  FT_TRY(level_cluster_setup());
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t cfg = level_cluster_cfg(a.w, a.h, nb, s, attr);
  FT_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_level_cluster, a));
  count_launch();
  return FT_OK;
}

}  // namespace

// Time the dominant kernel alone: `reps` eager launches of the finest-level
// primal-dual tile kernel over the workspace's current state (as left by the
// last step), bracketed by CUDA events on `s`.  Returns the mean duration.
// Half-step schedule of one k_pd_tile launch (PDArgs::nhalf / first / last)
// and its shrinking cone: the rows each half-step must compute, propagated
// backwards from the written interior [halo, th-halo).  A dual step at row r
// reads u-bar at r, r+1 and its own p; a primal step reads p at r, r-1.
// Returns false if the schedule needs rows outside the tile (too many
// half-steps for the halo).
bool halfstep_schedule(PDArgs &a, bool first, int nhalf, bool last, int halo, int th) {
  a.first = first;
  a.nhalf = nhalf;
  a.last = last;
  a.cone_rows = 0;
  if (halo == 0) return true;  // the tile is the whole level: every row is needed
  if (nhalf > 16) return false;
  const int kNone = 1 << 20;
  int ulo = halo, uhi = th - halo;                             // u needed after step j
  int plo = last ? kNone : halo, phi = last ? -kNone : th - halo;  // p needed
  int blo = kNone, bhi = -kNone;                               // u-bar needed
  for (int j = nhalf - 1; j >= 0; --j) {
    const bool dual = ((j & 1) == 0) == first;
    int lo, hi;
    if (dual) {
      lo = plo;
      hi = phi;
      if (lo < hi) blo = std::min(blo, lo), bhi = std::max(bhi, hi + 1);
    } else {
      lo = std::min(ulo, blo);
      hi = std::max(uhi, bhi);
      plo = std::min(plo, lo - 1);
      phi = std::max(phi, hi);
      ulo = lo, uhi = hi;
      blo = kNone, bhi = -kNone;
    }
    if (lo >= hi) lo = hi = 0;
    if (lo < 0 || hi > th) return false;
    a.rows_lo[j] = (signed char)lo;
    a.rows_hi[j] = (signed char)hi;
  }
  if ((plo < phi && (plo < 0 || phi > th)) || ulo < 0 || uhi > th) return false;
  if (first && blo < bhi && (blo < 0 || bhi > th)) return false;  // u-bar = u on [0, th)
  a.cone_rows = 1;
  return true;
}

int profile_pd(FlowWork &fw, int w, int h, int nb, const FlowParamsD &p, int reps,
               cudaStream_t s, double *ms_per_launch, int *iters_per_launch) {
  const PDPlan plan = pd_plan(w, h);
  const int halo = plan.halo;
  // FT_PD_PROFILE_ITERS overrides the iterations per launch (cost model:
  // load/store overhead vs per-iteration cost)
  const int hs = use_sweep(plan, p.tau) ? std::max(1, std::min(4, env_int("FT_SWEEP_ITERS", 2)))
                                        : halo;
  const int iters = env_int("FT_PD_PROFILE_ITERS", hs ? std::min(hs, p.iters) : p.iters);
  PDArgs a;
  a.gx = fw.gx;
  a.gy = fw.gy;
  a.r0 = fw.r0;
  a.w = w;
  a.h = h;
  a.cap = fw.cap;
  a.halo = halo;
  a.iters = iters;
  a.first = 0;
  a.nb = nb;
  a.pow2 = pow2_params(p.tau);
  a.cone = env_int("FT_PD_CONE", 1);
  a.cq = env_int("FT_PD_CQ", 1);
  a.async_ld = env_int("FT_PD_ASYNC", 1);
  if (plan.cfg.tile) {  // a middle launch: `iters` primal + dual pairs
    if (!halfstep_schedule(a, false, 2 * iters, false, halo, plan.cfg.th))
      return fail(FT_EINVAL, "FT_PD_PROFILE_ITERS exceeds the halo");
    if (!a.cone) a.cone_rows = 0;
  }
  a.tau = p.tau;
  a.lam = p.lam;
  a.sigma = 1.0 / (8.0 * p.tau);
  a.shrink = 1.0 / (1.0 + a.sigma * p.eps);
  cudaEvent_t e0, e1;
  FT_CUDA_TRY(cudaEventCreate(&e0));
  FT_CUDA_TRY(cudaEventCreate(&e1));
  int cur = 0;
  // one untimed launch to warm the instruction cache
  for (int r = -1; r < reps; ++r) {
    if (r == 0) FT_CUDA_TRY(cudaEventRecord(e0, s));
    a.in = state_ptrs(fw.st[cur], fw.nb, fw.cap);
    a.out = state_ptrs(fw.st[1 - cur], fw.nb, fw.cap);
    if (use_sweep(plan, p.tau)) FT_TRY(sweep_launch(a, 2 * iters, false, nb, s));
    else FT_TRY(pd_launch(plan.cfg, a, nb, s));
    cur = 1 - cur;
  }
  FT_CUDA_TRY(cudaEventRecord(e1, s));
  FT_CUDA_TRY(cudaEventSynchronize(e1));
  float ms = 0.f;
  FT_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  FT_CUDA_TRY(cudaGetLastError());
  *ms_per_launch = reps > 0 ? ms / reps : 0.0;
  *iters_per_launch = iters;
  return FT_OK;
}

int flow_work_alloc(FlowWork &fw, int nb, int64_t cap) {
  flow_work_free(fw);
  fw.nb = nb;
  fw.cap = cap;
  const size_t plane = (size_t)nb * cap * sizeof(double);
  double *all = nullptr;
  // gx gy r0 ix iy + 2 x 8 state planes
  cudaError_t e = cudaMalloc(&all, plane * (5 + 2 * NST));
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(flow workspace)");
  const int64_t pe = (int64_t)nb * cap;
  fw.gx = all;
  fw.gy = all + pe;
  fw.r0 = all + 2 * pe;
  fw.ix = all + 3 * pe;
  fw.iy = all + 4 * pe;
  fw.st[0] = all + 5 * pe;
  fw.st[1] = all + (5 + NST) * pe;
  return FT_OK;
}

void flow_work_free(FlowWork &fw) {
  if (fw.gx) cudaFree(fw.gx);
  fw = FlowWork();
}

int run_flow(const double *pyr0, const double *pyr1, int64_t pyr_stride, const int *lw,
             const int *lh, const int64_t *loff, int scales, const FlowParamsD &p, FlowWork &fw,
             double *dx, double *dy, int64_t out_stride, int nb, cudaStream_t s,
             double *energy_terms) {
  const int64_t cap = fw.cap;
  if (nb > fw.nb || (int64_t)lw[0] * lh[0] > cap) return fail(FT_EINVAL, "flow workspace too small");
  int cur = 0;
  const double sigma = 1.0 / (8.0 * p.tau);
  const double shrink = 1.0 / (1.0 + sigma * p.eps);
  const dim3 blk(32, 8);


  for (int lvl = scales - 1; lvl >= 0; --lvl) {
    const int w = lw[lvl], h = lh[lvl];
    StatePtrs st = state_ptrs(fw.st[cur], fw.nb, cap);
    if (cluster_level_ok(w, h)) {  // whole level on chip, one launch
      const double *i0 = pyr0 + loff[lvl];
      const double *i1 = pyr1 + loff[lvl];
      k_central_grad<<<grid2d(w, h, nb), blk, 0, s>>>(i1, w, h, pyr_stride, fw.ix, fw.iy, cap);
      count_launch();
      LevelArgs la;
      la.i0 = i0;
      la.i1 = i1;
      la.ps = pyr_stride;
      la.ix = fw.ix;
      la.iy = fw.iy;
      const bool coarsest = lvl == scales - 1;
      la.uc1 = coarsest ? nullptr : st.p[U1];
      la.uc2 = coarsest ? nullptr : st.p[U2];
      la.wc = coarsest ? 0 : lw[lvl + 1];
      la.hc = coarsest ? 0 : lh[lvl + 1];
      la.rx = coarsest ? 0.0 : (double)la.wc / (double)w;
      la.ry = coarsest ? 0.0 : (double)la.hc / (double)h;
      la.sx = coarsest ? 0.0 : (double)w / (double)la.wc;
      la.sy = coarsest ? 0.0 : (double)h / (double)la.hc;
      cur = 1 - cur;
      StatePtrs out = state_ptrs(fw.st[cur], fw.nb, cap);
      la.uo1 = out.p[U1];
      la.uo2 = out.p[U2];
      la.w = w;
      la.h = h;
      la.cap = cap;
      la.warps = p.warps;
      la.iters = p.iters;
      la.tau = p.tau;
      la.lam = p.lam;
      la.sigma = sigma;
      la.shrink = shrink;
      FT_TRY(launch_level_cluster(la, nb, s));
      phase_mark(kLevelNames[lvl < 8 ? lvl : 7]);
      continue;
    }
    if (lvl == scales - 1) {
      for (int b = 0; b < nb; ++b) {
        FT_CUDA_TRY(cudaMemsetAsync(st.p[U1] + b * cap, 0, (size_t)w * h * 8, s));
        FT_CUDA_TRY(cudaMemsetAsync(st.p[U2] + b * cap, 0, (size_t)w * h * 8, s));
      }
    } else {
      const int wc = lw[lvl + 1], hc = lh[lvl + 1];
      StatePtrs cs = state_ptrs(fw.st[cur], fw.nb, cap);
      cur = 1 - cur;
      st = state_ptrs(fw.st[cur], fw.nb, cap);
      k_upsample<<<grid2d(w, h, nb), blk, 0, s>>>(
          cs.p[U1], cs.p[U2], wc, hc, st.p[U1], st.p[U2], w, h, cap, (double)wc / (double)w,
          (double)hc / (double)h, (double)w / (double)wc, (double)h / (double)hc);
      count_launch();
    }
    const double *i0 = pyr0 + loff[lvl];
    const double *i1 = pyr1 + loff[lvl];
    k_central_grad<<<grid2d(w, h, nb), blk, 0, s>>>(i1, w, h, pyr_stride, fw.ix, fw.iy, cap);
    count_launch();

    const PDPlan plan = pd_plan(w, h);
    const bool resident = plan.halo == 0;
    const int halo = plan.halo;
    // barrier-free row sweep (k_pd_sweep) for tiled levels: same launch
    // schedule (<= 8 half-steps per launch), power-of-two time steps
    const bool sweep = use_sweep(plan, p.tau);
    // iterations per launch: the tile halo, or FT_SWEEP_ITERS (<= 4) for the sweep
    const int hs = sweep ? std::max(1, std::min(4, env_int("FT_SWEEP_ITERS", 2))) : halo;
    // Stream groups (FT_PD_GROUP, finest level): a group of streams runs all
    // of its warps before the next group starts, so the group's state planes
    // (~63 MB per SD stream incl. ping-pong) can stay resident in the 126 MB
    // L2 across the PD launches instead of streaming through HBM.
    const int grp = lvl == 0 ? std::max(1, std::min(nb, env_int("FT_PD_GROUP", nb))) : nb;
    const int cur0 = cur;
    PdSpan *span = lvl == 0 && !resident ? g_pd_span : nullptr;
    if (span) span->spans = span->launches = 0, span->pixel_iters = 0;
    for (int g0 = 0; g0 < nb; g0 += grp) {
      const int gn = std::min(grp, nb - g0);
      cur = cur0;
      auto sp = [&](int which) {
        StatePtrs r = state_ptrs(fw.st[which], fw.nb, cap);
        for (int k = 0; k < NST; ++k) r.p[k] += (int64_t)g0 * cap;
        return r;
      };
      const int64_t go = (int64_t)g0 * cap;
      const double *gi0 = i0 + (int64_t)g0 * pyr_stride, *gi1 = i1 + (int64_t)g0 * pyr_stride;
      for (int wp = 0; wp < p.warps; ++wp) {
        st = sp(cur);
        k_warp_setup<<<grid2d(w, h, gn), blk, 0, s>>>(gi0, gi1, pyr_stride, fw.ix + go, fw.iy + go,
                                                       st.p[U1], st.p[U2], w, h, cap, fw.gx + go,
                                                       fw.gy + go, fw.r0 + go);
        count_launch();
        const int si = span && span->spans < PdSpan::kMaxSpans ? span->spans : -1;
        if (si >= 0)
          FT_CUDA_TRY(cudaEventRecordWithFlags(span->ev[2 * si], s, cudaEventRecordExternal));
        // k_pd_tile: 2*iters half-steps D P D P ... split into launches that
        // end after a dual step (state u, p) -- the first of at most 2*halo-1
        // half-steps (starts with D), then 2*halo (P..D), and the rest (odd,
        // P..P) in the last launch.  Other kernels: `halo` whole iterations.
        const int total = plan.cfg.tile ? 2 * p.iters : p.iters;
        int done = 0;
        while (done < total) {
          int n;
          if (!plan.cfg.tile) n = resident ? p.iters : std::min(halo, p.iters - done);
          else if (resident) n = total;
          else if (done == 0) n = std::min(2 * hs - 1, total);
          else n = total - done <= 2 * hs ? total - done : 2 * hs;
          PDArgs a;
          a.in = sp(cur);
          a.out = sp(1 - cur);
          a.gx = fw.gx + go;
          a.gy = fw.gy + go;
          a.r0 = fw.r0 + go;
          a.w = w;
          a.h = h;
          a.cap = cap;
          a.halo = halo;
          a.iters = n;
          a.first = done == 0;
          a.nb = gn;
          a.pow2 = pow2_params(p.tau);
          a.cone = env_int("FT_PD_CONE", 1);
          a.cq = env_int("FT_PD_CQ", 1);
          a.async_ld = env_int("FT_PD_ASYNC", 1);
          if (plan.cfg.tile) {
            if (!halfstep_schedule(a, done == 0, n, done + n == total, halo, plan.cfg.th))
              return fail(FT_EINVAL, "primal-dual schedule exceeds the tile halo");
            if (!a.cone) a.cone_rows = 0;
          }
          a.tau = p.tau;
          a.lam = p.lam;
          a.sigma = sigma;
          a.shrink = shrink;
          if (sweep) FT_TRY(sweep_launch(a, n, done == 0, gn, s));
          else FT_TRY(pd_launch(plan.cfg, a, gn, s));
          cur = 1 - cur;
          done += n;
          if (si >= 0) ++span->launches;
        }
        if (si >= 0) {
          FT_CUDA_TRY(cudaEventRecordWithFlags(span->ev[2 * si + 1], s, cudaEventRecordExternal));
          span->spans = si + 1;
          span->pixel_iters += (int64_t)w * h * gn * p.iters;
        }
        StatePtrs in = sp(cur);
        StatePtrs out = sp(1 - cur);
        k_median<<<grid2d((w + 1) / 2, h, gn), blk, 0, s>>>(in.p[U1], in.p[U2], out.p[U1],
                                                            out.p[U2], w, h, cap);
        count_launch();
        cur = 1 - cur;
        if (energy_terms && lvl == 0 && nb == 1) {  // energy_trace (optflow.py:212-213)
          const int64_t n0 = (int64_t)w * h;
          StatePtrs now = sp(cur);
          double *tb = energy_terms + (int64_t)wp * 3 * n0;
          FT_TRY(launch_energy_terms(i0, i1, now.p[U1], now.p[U2], w, h, p.eps, tb, tb + n0,
                                     tb + 2 * n0, s));
        }
      }
    }
    phase_mark(kLevelNames[lvl < 8 ? lvl : 7]);
  }
  StatePtrs st = state_ptrs(fw.st[cur], fw.nb, cap);
  const int64_t n0 = (int64_t)lw[0] * lh[0];
  for (int b = 0; b < nb; ++b) {
    FT_CUDA_TRY(cudaMemcpyAsync(dx + b * out_stride, st.p[U1] + b * cap, n0 * 8,
                                cudaMemcpyDeviceToDevice, s));
    FT_CUDA_TRY(cudaMemcpyAsync(dy + b * out_stride, st.p[U2] + b * cap, n0 * 8,
                                cudaMemcpyDeviceToDevice, s));
  }
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

}  // namespace ft

namespace ft {
int launch_energy_terms(const double *i0, const double *i1, const double *u1, const double *u2,
                        int w, int h, double eps, double *data, double *s1, double *s2,
                        cudaStream_t s) {
  k_energy_terms<<<dim3((w + 31) / 32, (h + 7) / 8), dim3(32, 8), 0, s>>>(i0, i1, u1, u2, w, h, eps,
                                                                       data, s1, s2);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}
}  // namespace ft

namespace ft {
int launch_central_grad(const double *img, int w, int h, int64_t is, double *gx, double *gy,
                        int64_t gs, int nb, cudaStream_t s) {
  k_central_grad<<<grid2d(w, h, nb), dim3(32, 8), 0, s>>>(img, w, h, is, gx, gy, gs);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}
}  // namespace ft

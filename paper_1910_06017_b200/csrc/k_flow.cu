// Dense coarse-to-fine TV-L1 optical flow (reference optflow.py:147-253).
//
// Per scale: central gradient of I1 (optflow.py:155); per warp a setup pass
// (bilinear gathers + linearised data-term constants, :158-176); the
// primal-dual iterations (:178-208) in a temporally blocked tile kernel; a
// 3x3 median of both components (:210-211).  Between scales a bilinear
// upsample scaled by the size ratio (:244-249).
//
// HBM layout (per batch of nb image pairs, capacity `cap` pixels per stream
// and plane, pitch == level width).  Fields used together are interleaved
// as double2 so the tile kernel moves whole tiles with TMA box copies:
//   U  (u1, u2)       state ping-pong st[2] = [U | PX | PY][nb][cap] double2
//   PX (p11, p21)     (u-bar is recomputed at the start of every launch and
//   PY (p12, p22)      never leaves the chip)
//   G  (gx, gy)       warp constants          [nb][cap] double2
//   RT (rho0, 1/|grad|^2 or 0)                [nb][cap] double2
//   IX (dI1/dx, dI1/dy) level gradient        [nb][cap] double2
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "ft_internal.cuh"

namespace ft {

namespace {

struct StatePtrs {
  double2 *u, *px, *py;
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

// the same sample of both components of an interleaved double2 plane (each
// component in exactly bsample's operation order)
__device__ __forceinline__ double2 bsample2(const double2 *__restrict__ img, int w, int h,
                                            double x, double y) {
  x = clip_lo_hi(x, 0.0, w - 1.0);
  y = clip_lo_hi(y, 0.0, h - 1.0);
  const int x0 = (int)floor(x), y0 = (int)floor(y);
  const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
  const double fx = x - (double)x0, fy = y - (double)y0;
  const double2 *r0 = img + (int64_t)y0 * w;
  const double2 *r1 = img + (int64_t)y1 * w;
  const double2 a = r0[x0], b = r0[x1], c = r1[x0], d = r1[x1];
  const double tx = a.x * (1.0 - fx) + b.x * fx, ty = a.y * (1.0 - fx) + b.y * fx;
  const double bx = c.x * (1.0 - fx) + d.x * fx, by = c.y * (1.0 - fx) + d.y * fx;
  return make_double2(tx * (1.0 - fy) + bx * fy, ty * (1.0 - fy) + by * fy);
}

// np.gradient(i1) with unit spacing (optflow.py:155): central inside,
// one-sided at the borders.  (a-b)/2 == (a-b)*0.5 exactly.
__device__ __forceinline__ double2 central_grad_at(const double *__restrict__ img, int w, int h,
                                                   int c, int r) {
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
  return make_double2(vx, vy);
}

// separate gx / gy planes (the KLT backend's pyramids)
__global__ void k_central_grad(const double *__restrict__ img, int w, int h, int64_t is,
                               double *__restrict__ gx, double *__restrict__ gy, int64_t gs) {
  img += blockIdx.z * is;
  gx += blockIdx.z * gs;
  gy += blockIdx.z * gs;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (r >= h || c >= w) return;
  const double2 g = central_grad_at(img, w, h, c, r);
  const int64_t o = (int64_t)r * w + c;
  gx[o] = g.x;
  gy[o] = g.y;
}

// interleaved IX plane (the flow's warp setup gathers both with one sample)
__global__ void k_central_grad2(const double *__restrict__ img, int w, int h, int64_t is,
                                double2 *__restrict__ ix, int64_t cap) {
  img += blockIdx.z * is;
  ix += blockIdx.z * cap;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (r >= h || c >= w) return;
  ix[(int64_t)r * w + c] = central_grad_at(img, w, h, c, r);
}

// resize_bilinear(u, w, h) * ratio for both components (optflow.py:244-249,
// imageops.py:69-75).  rx = wc/wf, ry = hc/hf (host-computed IEEE quotients),
// sx = wf/wc, sy = hf/hc.
__global__ void k_upsample(const double2 *__restrict__ cu, int wc, int hc,
                           double2 *__restrict__ fu, int wf, int hf, int64_t cap, double rx,
                           double ry, double sx, double sy) {
  cu += blockIdx.z * cap;
  fu += blockIdx.z * cap;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (r >= hf || c >= wf) return;
  const double x = ((double)c + 0.5) * rx - 0.5;
  const double y = ((double)r + 0.5) * ry - 0.5;
  const double2 v = bsample2(cu, wc, hc, x, y);
  fu[(int64_t)r * wf + c] = make_double2(v.x * sx, v.y * sy);
}

// Per-warp linearisation (optflow.py:158-176): gather I1, dI1/dx, dI1/dy at
// x+u; rho0 = I1w - I0 - gx*u1 - gy*u2 and 1/|grad|^2 (0 where |grad|^2 <=
// 1e-12).  The threshold tau*lam*|grad|^2 is rederived from (gx, gy) by the
// tile kernel's prologue (a multiply instead of a plane).
__global__ void k_warp_setup(const double *__restrict__ i0, const double *__restrict__ i1,
                             int64_t ps, const double2 *__restrict__ ix,
                             const double2 *__restrict__ u, int w, int h, int64_t cap,
                             double2 *__restrict__ g, double2 *__restrict__ rt) {
  i0 += blockIdx.z * ps;
  i1 += blockIdx.z * ps;
  const int64_t so = blockIdx.z * cap;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (r >= h || c >= w) return;
  const int64_t o = (int64_t)r * w + c;
  const double2 uu = u[so + o];
  const double mx = (double)c + uu.x, my = (double)r + uu.y;
  const double v = bsample(i1, w, h, mx, my);
  const double2 gg = bsample2(ix + so, w, h, mx, my);
  g[so + o] = gg;
  const double g2 = gg.x * gg.x + gg.y * gg.y;  // optflow.py:163
  // 1/|grad|^2 once per warp here, not in every launch's prologue
  // (optflow.py:164-165: g2 > 1e-12 <=> max(g2, 1e-12) == g2)
  rt[so + o] = make_double2(v - i0[o] - gg.x * uu.x - gg.y * uu.y, recip_if(g2 > 1e-12, g2));
}

// 3x3 median with replicated border (imageops.py:78-84): exact 5th order
// statistic of 9 via a min/max selection network.  One comparison per
// compare-swap (the fields are finite: MotionField / compute_flow reject
// NaN, optflow.py:85-86); a tie between -0.0 and +0.0 may return either
// zero, as numpy's introselect may (np.median's partition is not
// order-stable).
__device__ __forceinline__ void cswap(double &a, double &b) {
  const bool sw = b < a;
  const double lo = sw ? b : a, hi = sw ? a : b;
  a = lo;
  b = hi;
}

__device__ __forceinline__ double med3(double a, double b, double c) {
  cswap(a, b);                 // a <= b
  const double m = c < b ? c : b;  // min(max(a, b), c)
  return m < a ? a : m;        // max(min(a, b), min(max(a, b), c))
}

__device__ __forceinline__ double max3(double a, double b, double c) {
  const double m = b < a ? a : b;
  return c < m ? m : c;
}

__device__ __forceinline__ double min3(double a, double b, double c) {
  const double m = b < a ? b : a;
  return c < m ? c : m;
}

// Two horizontally adjacent outputs per thread: the four 3-sample columns
// c-1..c+2 are sorted once and shared; median9 = med3(max of the column
// minima, med3 of the column medians, min of the column maxima), the same
// order statistic as the sort (exact selection).  Both components of U.
__global__ void k_median(const double2 *__restrict__ in, double2 *__restrict__ out, int w, int h,
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
  const double2 *a = in + so;
  double lo[2][4], md[2][4], hi[2][4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double2 x = a[rr[0] + cc[k]], y = a[rr[1] + cc[k]], z = a[rr[2] + cc[k]];
    double x0 = x.x, y0 = y.x, z0 = z.x, x1 = x.y, y1 = y.y, z1 = z.y;
    cswap(x0, y0);
    cswap(y0, z0);
    cswap(x0, y0);
    cswap(x1, y1);
    cswap(y1, z1);
    cswap(x1, y1);
    lo[0][k] = x0, md[0][k] = y0, hi[0][k] = z0;
    lo[1][k] = x1, md[1][k] = y1, hi[1][k] = z1;
  }
  double m[2][2];
#pragma unroll
  for (int f = 0; f < 2; ++f) {
    m[f][0] = med3(max3(lo[f][0], lo[f][1], lo[f][2]), med3(md[f][0], md[f][1], md[f][2]),
                   min3(hi[f][0], hi[f][1], hi[f][2]));
    m[f][1] = med3(max3(lo[f][1], lo[f][2], lo[f][3]), med3(md[f][1], md[f][2], md[f][3]),
                   min3(hi[f][1], hi[f][2], hi[f][3]));
  }
  double2 *o = out + so + (int64_t)r * w + c;
  o[0] = make_double2(m[0][0], m[1][0]);
  if (two) o[1] = make_double2(m[0][1], m[1][1]);
}

// Per-pixel terms of the TV-L1 objective (optflow.py:121-137): data term
// |I1(x+u) - I0| and, per component, huber(hypot(forward_gradient(u))).
// The reference sums these arrays with numpy; the caller does exactly that
// on the host copies, so the scalar is bit-identical too.  u1/u2 element
// stride us: 1 for separate planes, 2 for an interleaved U plane.
__global__ void k_energy_terms(const double *__restrict__ i0, const double *__restrict__ i1,
                               const double *__restrict__ u1, const double *__restrict__ u2,
                               int us, int w, int h, double eps, double *__restrict__ data,
                               double *__restrict__ s1, double *__restrict__ s2) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (r >= h || c >= w) return;
  const int64_t o = (int64_t)r * w + c;
  const double v = bsample(i1, w, h, (double)c + u1[us * o], (double)r + u2[us * o]);
  data[o] = fabs(v - i0[o]);
  const double *comp[2] = {u1, u2};
  double *dst[2] = {s1, s2};
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double *u = comp[k];
    const double gx = c < w - 1 ? u[us * (o + 1)] - u[us * o] : 0.0;
    const double gy = r < h - 1 ? u[us * (o + w)] - u[us * o] : 0.0;
    const double m = glibc_hypot(gx, gy);
    // _huber (optflow.py:121-124)
    dst[k][o] = eps <= 0.0 ? m : (m <= eps ? m * m / (2.0 * eps) : m - eps / 2.0);
  }
}

// the finest level's U -> the caller's dx / dy planes
__global__ void k_split(const double2 *__restrict__ u, int64_t n, int64_t cap,
                        double *__restrict__ dx, double *__restrict__ dy, int64_t os) {
  u += blockIdx.z * cap;
  dx += blockIdx.z * os;
  dy += blockIdx.z * os;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double2 v = u[i];
    dx[i] = v.x;
    dy[i] = v.y;
  }
}

StatePtrs state_ptrs(double2 *base, int nb, int64_t cap) {
  return StatePtrs{base, base + (int64_t)nb * cap, base + 2 * (int64_t)nb * cap};
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
// its own u-bar.  Pointwise fields
// (u, the gathered gradient, the threshold derived once per launch) live in
// registers of the owning thread, (rho0, 1/|grad|^2) in the shared RT
// staging box: thread (tx, ty) owns
// columns tx + 32*cx (cx < TW/32) and rows PY*ty + k (k < PY).
// ------------------------------------------------------------------------
struct alignas(64) PDArgs {
  // TMA descriptors (3-D: interleaved row, y, image of the batch), built per
  // launch: the tile plus its one-element apron of U / PX / PY, the tile's
  // G / RT, and the written interior of U / PX / PY.  Boxes that stick out
  // of the image are zero-filled on load and clipped on store.
  CUtensorMap in_u, in_px, in_py;
  CUtensorMap in_g, in_rt;
  CUtensorMap out_u, out_px, out_py;
  int w, h;
  int halo, first, nb;
  int pow2;  // sigma and tau are powers of two (exact fused multiply-adds)
  // k_pd_tile half-step schedule: the launch runs `nhalf` alternating dual (D)
  // / primal (P) half-steps, starting with D when `first` (u-bar = u, p = 0)
  // and with P otherwise; it ends after a D (state u, p) unless `last` (ends
  // after a P, writes u only).  rows_lo/hi[j]: rows half-step j must compute
  // (shrinking cone; cone_rows == 0 -> all rows).
  int nhalf, last, cone_rows;
  signed char rows_lo[16], rows_hi[16];
  double tau, lam, sigma, shrink;  // shrink = 1/(1+sigma*eps)
  int prefetch_stride;  // CTAs resident at once: the L2 prefetch target is bid + this (0: off)
};

// per-pixel border flags (global position, fixed for the launch)
enum : unsigned { FL_R = 1, FL_D = 2, FL_L = 4, FL_LASTC = 8, FL_U = 16, FL_LASTR = 32 };

// Exchange planes hold the fields read at a neighbour as three interleaved
// double2 planes -- (b1,b2), (p11,p21), (p12,p22) -- the pairs that are always
// read together, so each neighbour access is one 128-bit shared load.

template <int TW, int BY, int PY>
struct PDGeom {
  static constexpr int NX = TW / 32, TH = BY * PY, NP = NX * PY;
  static constexpr int SP = TW + 2, SR = TH + 2;
  // plane stride in double2, rounded to 128 bytes (TMA destinations)
  static constexpr int PLANE = (SP * SR + 7) / 8 * 8;
  // shared memory: 3 exchange planes | staging (in: G and RT boxes of the
  // tile; out: the U / PX / PY interior boxes) | CTA projection queue (one
  // int per pair, 2*NP pairs per thread, two counters) | mbarrier
  static constexpr size_t kPlanes = (size_t)3 * PLANE * 16;
  static constexpr size_t kStage = (size_t)2 * TW * TH * 16;
  static constexpr size_t kQueue = ((size_t)(2 * NP * 32 * BY + 2) * 4 + 15) / 16 * 16;
  static constexpr size_t smem = kPlanes + kStage + kQueue + 16;
  // thread (tx, ty) owns PY adjacent rows row(ty, k), k < PY: a pixel's
  // lower neighbour for the dual step and upper neighbour for the primal
  // step are then mostly values the thread has already loaded (one shared
  // load fewer per pixel pair and half-step than rows ty + BY*k: +3 %)
  static __device__ __forceinline__ int row(int ty, int k) { return PY * ty + k; }
  static constexpr int roff(int k) { return k * SP; }
};

// ---- TMA / mbarrier primitives (PTX)
__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "FT_MBAR_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra FT_MBAR_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// box at pixel (x, y) of image z of a plane_map (x counts double2 pixels)
__device__ __forceinline__ void tma_load(void *dst, const CUtensorMap *m, int x, int y, int z,
                                         uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(2 * x), "r"(y), "r"(z), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tma_store(const CUtensorMap *m, int x, int y, int z,
                                          const void *src) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
          reinterpret_cast<uint64_t>(m)),
      "r"(2 * x), "r"(y), "r"(z), "r"(smem_u32(src))
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_l2(const CUtensorMap *m, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(2 * x), "r"(y), "r"(z)
               : "memory");
}
__device__ __forceinline__ void tma_store_commit_wait() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// generic-proxy shared-memory writes -> visible to the async (TMA) proxy
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// a*b + c.  With P2 the product is exact (b or a is a power of two: sigma
// and tau for the default time_step 0.25, the literal 2.0), so one fused
// multiply-add rounds exactly like the reference's separate multiply and
// add; otherwise the two IEEE operations are kept (-fmad=false).
template <bool P2>
__device__ __forceinline__ double madx(double a, double b, double c) {
  return P2 ? fma(a, b, c) : a * b + c;
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
// launch schedules with compile-time half-step order (k_pd_tile MODE)
enum : int { kSchedGeneric = 0, kSchedMid = 1, kSchedFirst = 2, kSchedLast = 3 };

template <int TW, int BY, int PY, bool P2, bool IN, int MODE>
__device__ __forceinline__ void pd_halfsteps_cq(const PDArgs &a, double *sm, int base, int tx,
                                                int ty, const unsigned *fl, double *u1,
                                                double *u2, const double *gx, const double *gy,
                                                const double2 *rt, const double *thr_, double tl,
                                                int *qidx, int *ctr) {
  using G = PDGeom<TW, BY, PY>;
  constexpr int NX = G::NX, NP = G::NP, SP = G::SP, PL = G::PLANE, TH = G::TH;
  constexpr int NT = 32 * BY;
  const double tau = a.tau, sigma = a.sigma, shrink = a.shrink;
  double2 *const sB = reinterpret_cast<double2 *>(sm), *const sPX = sB + PL, *const sPY = sPX + PL;
  double *const dPX = reinterpret_cast<double *>(sPX), *const dPY = reinterpret_cast<double *>(sPY);
  const unsigned lt_mask = (1u << tx) - 1u;
  const int tid = ty * 32 + tx;
  int nd = 0;  // dual half-steps done (queue counter parity)
  // The own p as the primal step read it (after the projection) is the next
  // dual step's input, unchanged in between: in MID launches (where every
  // dual row is a row of the primal step just before it) the thread's first
  // pixel keeps it in registers instead of reloading it -- one pixel only:
  // both spill at the 64-register cap (+1.4 % vs 0.6 % for px alone, -0.1 %
  // for three of the four double2)
  constexpr int KEEPP = (MODE == kSchedMid) ? 1 : 0;
  double2 kpx[NP], kpy[NP];  // set by every MID primal step before its dual reads them
#pragma unroll
  for (int q = 0; q < NP; ++q) kpx[q] = kpy[q] = make_double2(0.0, 0.0);
  auto half = [&](const bool dual, const int lo, const int hi) {
    bool row_on[NP];
    bool all = true;
#pragma unroll
    for (int q = 0; q < NP; ++q) {
      const int lr = G::row(ty, q / NX);
      row_on[q] = lr >= lo && lr < hi;
      all = all && row_on[q];
    }
    if (dual) {
      // ---- dual ascent with Huber prox (:180-185), unprojected p stored in place
      unsigned need = 0;
      // (the common all-rows-active case runs branch-free so the compiler can
      // interleave the pixels' dependency chains)
      auto dual_px = [&](const int q) {
        const int id = base + G::roff(q / NX) + 32 * (q % NX);
        const double2 cb = sB[id], rb = sB[id + 1], db = sB[id + SP];
        const bool kp = q < KEEPP;
        const double2 opx = kp ? kpx[q] : sPX[id], opy = kp ? kpy[q] : sPY[id];
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
#pragma unroll
      for (int k = 0; k < 2 * NP; ++k) {
        const unsigned m = __ballot_sync(0xffffffffu, (need >> k) & 1u);
        off[k] = total + __popc(m & lt_mask);
        total += __popc(m);
      }
      if (total) {  // warp-uniform
        int wbase = 0;
        if (tx == 0) wbase = atomicAdd(&ctr[nd & 1], total);
        wbase = __shfl_sync(0xffffffffu, wbase, 0);
#pragma unroll
        for (int k = 0; k < 2 * NP; ++k) {
          const int q = k >> 1;
          const int id = base + G::roff(q / NX) + 32 * (q % NX);
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
        // (one shared reciprocal, div_by_recip, spills here: 1.616 -> 1.644 ms)
        dPX[k] = div_pos(pa, nn);  // nn >= 1
        dPY[k] = div_pos(pb, nn);
      }
      ++nd;
    } else {
      // ---- primal descent + TV-L1 shrinkage (:194-208), u-bar stored in place
      auto primal_px = [&](const int q) {
        const int id = base + G::roff(q / NX) + 32 * (q % NX);
        const unsigned f = fl[q];
        const double2 mpx = sPX[id], mpy = sPY[id];
        if (q < KEEPP) {
          kpx[q] = mpx;
          kpy[q] = mpy;
        }
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
        // (rho0, 1/|grad|^2) stay in the shared G/RT staging of the prologue
        const double2 rq = rt[G::row(ty, q / NX) * TW + tx + 32 * (q % NX)];
        const double rho = rq.x + gx[q] * v1 + gy[q] * v2;
        const double thr = thr_[q], ig = rq.y;
        const bool lo_ = rho < -thr;
        const bool hi_ = rho > thr;
        double d = lo_ ? tl : (hi_ ? -tl : -rho * ig);
        d = (ig != 0.0 || lo_ || hi_) ? d : 0.0;  // ig != 0 <=> |grad|^2 > 1e-12
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
    __syncthreads();
  };
  if (MODE == kSchedMid) {
    // middle launch (P D)x4 of a 32-row tile with halo 4: the cone rows of
    // halfstep_schedule in closed form -- P_i: [1+i, 32-i), D_i: [1+i, 31-i)
    static_assert(MODE != kSchedMid || TH == 32, "closed-form cone is for 32-row tiles");
    // fully unrolled: the pixel state alternates between register sets
    // instead of being moved back every iteration, and no spills remain
    // (+0.4 %; unrolling by 2 was slower)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      half(false, 1 + i, TH - i);
      half(true, 1 + i, TH - 1 - i);
    }
  } else if (MODE == kSchedFirst) {
    // a warp's first launch: D P D P D P D, cone rows from the schedule
#pragma unroll
    for (int j = 0; j < 7; ++j) half((j & 1) == 0, a.rows_lo[j], a.rows_hi[j]);
  } else if (MODE == kSchedLast) {
    // a warp's last launch: P D P D P
#pragma unroll
    for (int j = 0; j < 5; ++j) half((j & 1) == 1, a.rows_lo[j], a.rows_hi[j]);
  } else {
    for (int j = 0; j < a.nhalf; ++j) {
      const bool dual = ((j & 1) == 0) == (a.first != 0);
      half(dual, a.cone_rows ? a.rows_lo[j] : 0, a.cone_rows ? a.rows_hi[j] : TH);
    }
  }
}

// Tile movement is TMA: one elected thread issues box copies of the tile
// (+ apron) of U / PX / PY and of the tile's G / RT straight into shared
// memory, completing on an mbarrier, and stores the written interior of U /
// PX / PY with TMA box stores from a shared staging area.  Out-of-image
// elements are zero-filled on load (the reference's zeros outside the
// image never reach an interior pixel) and clipped on store.
template <int TW, int BY, int PY, int MINB, int MODE = kSchedGeneric>
__global__ void __launch_bounds__(32 * BY, MINB) k_pd_tile(const __grid_constant__ PDArgs a) {
  using G = PDGeom<TW, BY, PY>;
  constexpr int NX = G::NX, TH = G::TH, NP = G::NP, SP = G::SP, SR = G::SR, PL = G::PLANE;
  extern __shared__ __align__(128) unsigned char smraw[];
  double *const sm = reinterpret_cast<double *>(smraw);
  double2 *const sB = reinterpret_cast<double2 *>(smraw);
  double2 *const stage = reinterpret_cast<double2 *>(smraw + G::kPlanes);
  int *const qidx = reinterpret_cast<int *>(smraw + G::kPlanes + G::kStage);
  int *const ctr = qidx + 2 * NP * 32 * BY;
  uint64_t *const bar = reinterpret_cast<uint64_t *>(smraw + G::kPlanes + G::kStage + G::kQueue);

  const int W = a.w, H = a.h;
  const int step_x = TW - 2 * a.halo, step_y = TH - 2 * a.halo;
  const int ox = (int)blockIdx.x * step_x - a.halo;
  const int oy = blockIdx.y * step_y - a.halo;
  const int bz = blockIdx.z;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int tid = ty * 32 + tx;
  const int base = (G::row(ty, 0) + 1) * SP + tx + 1;  // apron offset (+1,+1)

  // ---- prologue: U (-> u-bar plane: u-bar = u), p, G, RT by TMA
  if (tid == 0) mbar_init(bar, 1);
  __syncthreads();
  if (tid == 0) {
    const unsigned box = SP * SR * 16, own = TW * TH * 16;
    mbar_expect_tx(bar, box * (a.first ? 1 : 3) + 2 * own);
    tma_load(sB, &a.in_u, ox - 1, oy - 1, bz, bar);
    if (!a.first) {
      tma_load(sB + PL, &a.in_px, ox - 1, oy - 1, bz, bar);
      tma_load(sB + 2 * PL, &a.in_py, ox - 1, oy - 1, bz, bar);
    }
    tma_load(stage, &a.in_g, ox, oy, bz, bar);
    tma_load(stage + TW * TH, &a.in_rt, ox, oy, bz, bar);
  }
  if (a.first) {  // p = 0 at the start of a warp (optflow.py:169-172)
    for (int k = tid; k < SP * SR; k += 32 * BY) {
      sB[PL + k] = make_double2(0.0, 0.0);
      sB[2 * PL + k] = make_double2(0.0, 0.0);
    }
  }
  if (tid < 2) ctr[tid] = 0;
  if (tid == 32 && a.prefetch_stride) {
    // the tile that will take this CTA's slot next (linear order, one full
    // wave later): pull its boxes into L2 while this tile computes
    const int nx = gridDim.x, ny = gridDim.y;
    const int nxt = (int)(blockIdx.x + nx * (blockIdx.y + ny * blockIdx.z)) + a.prefetch_stride;
    if (nxt < nx * ny * (int)gridDim.z) {
      const int px = nxt % nx, py = (nxt / nx) % ny, pz = nxt / (nx * ny);
      const int qx = px * step_x - a.halo, qy = py * step_y - a.halo;
      tma_prefetch_l2(&a.in_u, qx - 1, qy - 1, pz);
      if (!a.first) {
        tma_prefetch_l2(&a.in_px, qx - 1, qy - 1, pz);
        tma_prefetch_l2(&a.in_py, qx - 1, qy - 1, pz);
      }
      tma_prefetch_l2(&a.in_g, qx, qy, pz);
      tma_prefetch_l2(&a.in_rt, qx, qy, pz);
    }
  }
  if (ty == 0) mbar_wait(bar, 0);  // one warp polls; the others sleep in the barrier
  __syncthreads();
  mbar_wait(bar, 0);  // completed phase: returns at once, orders the TMA data

  const double tl = a.tau * a.lam;
  double u1[NP], u2[NP], gx[NP], gy[NP], thr_[NP];
  unsigned fl[NP];
#pragma unroll
  for (int k = 0; k < PY; ++k) {
#pragma unroll
    for (int cx = 0; cx < NX; ++cx) {
      const int q = k * NX + cx;
      const int lc = tx + 32 * cx, lr = G::row(ty, k);
      const int gc = ox + lc, gr = oy + lr;
      const double2 u = sB[base + G::roff(k) + 32 * cx];
      const double2 g = stage[lr * TW + lc];
      u1[q] = u.x;
      u2[q] = u.y;
      gx[q] = g.x;
      gy[q] = g.y;
      const double g2 = g.x * g.x + g.y * g.y;  // optflow.py:163-165
      thr_[q] = tl * g2;  // thresh = tau * lam * grad_sq (optflow.py:176)
      fl[q] = (gc < W - 1 ? FL_R : 0u) | (gr < H - 1 ? FL_D : 0u) | (gc > 0 ? FL_L : 0u) |
              (gc == W - 1 ? FL_LASTC : 0u) | (gr > 0 ? FL_U : 0u) | (gr == H - 1 ? FL_LASTR : 0u);
    }
  }
  __syncthreads();

  // tile free of image-border pixels (uniform per CTA): flag-free fast path
  const bool interior = ox >= 1 && oy >= 1 && ox + TW <= W - 1 && oy + TH <= H - 1;
  {
#define FT_PD_CALL(P2_, IN_)                                                                 \
  pd_halfsteps_cq<TW, BY, PY, P2_, IN_, MODE>(a, sm, base, tx, ty, fl, u1, u2, gx, gy, \
                                             stage + TW * TH, thr_, tl, qidx, ctr)
    if (a.pow2) {
      if (interior) FT_PD_CALL(true, true); else FT_PD_CALL(true, false);
    } else {
      if (interior) FT_PD_CALL(false, true); else FT_PD_CALL(false, false);
    }
#undef FT_PD_CALL
  }

  // ---- epilogue: the exact interior of u, and of p unless this is the
  // warp's last launch (the next warp starts from p = 0), staged densely and
  // stored by TMA (the G / RT staging is dead by now)
  const int hl = a.halo, iw = TW - 2 * hl, ih = TH - 2 * hl;
  double2 *const ou = stage, *const opx = stage + iw * ih, *const opy = stage + 2 * iw * ih;
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    const int k = q / NX, cx = q % NX;
    const int lc = tx + 32 * cx, lr = G::row(ty, k);
    if (lc < hl || lc >= TW - hl || lr < hl || lr >= TH - hl) continue;
    const int e = (lr - hl) * iw + (lc - hl);
    ou[e] = make_double2(u1[q], u2[q]);
    if (!a.last) {
      const int id = base + G::roff(k) + 32 * cx;
      opx[e] = sB[PL + id];
      opy[e] = sB[2 * PL + id];
    }
  }
  fence_proxy_async();
  __syncthreads();
  if (tid == 0) {
    tma_store(&a.out_u, ox + hl, oy + hl, bz, ou);
    if (!a.last) {
      tma_store(&a.out_px, ox + hl, oy + hl, bz, opx);
      tma_store(&a.out_py, ox + hl, oy + hl, bz, opy);
    }
    tma_store_commit_wait();
  }
}

// Launch configurations (tile width x height, threads, min CTAs/SM).
struct PDConfig {
  int tw, th, by;
  void (*fn)(PDArgs);
  void (*fn_mid)(PDArgs);    // k_pd_tile<..., kSchedMid>: middle (P D)x4 launches, halo 4
  void (*fn_first)(PDArgs);  // kSchedFirst: a warp's first launch (7 half-steps)
  void (*fn_last)(PDArgs);   // kSchedLast: a warp's last launch (5 half-steps)
  size_t smem;             // exchange planes, TMA staging, projection queue, mbarrier
};

template <int TW, int BY, int PY, int MINB>
PDConfig make_cfg() {
  using G = PDGeom<TW, BY, PY>;
  constexpr bool t32 = G::TH == 32 && TW == 32 && BY == 16;  // the tiled configuration
  return PDConfig{TW, G::TH, BY, &k_pd_tile<TW, BY, PY, MINB>,
                  G::TH == 32 ? &k_pd_tile<TW, BY, PY, MINB, kSchedMid> : nullptr,
                  t32 ? &k_pd_tile<TW, BY, PY, MINB, t32 ? kSchedFirst : kSchedGeneric> : nullptr,
                  t32 ? &k_pd_tile<TW, BY, PY, MINB, t32 ? kSchedLast : kSchedGeneric> : nullptr,
                  G::smem};
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no
// link-time dependency on libcuda)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) !=
            cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}

// 3-D map over nb interleaved double2 planes of w x h (stream stride cap
// pixels), viewed as rows of 2w doubles so a box row is one contiguous run
// of 2*bw doubles (a 16-byte innermost box dimension starves the TMA unit):
// dims (2w, h, image), box (2*bw, bh, 1)
int plane_map(CUtensorMap *m, const double2 *base, int w, int h, int nb, int64_t cap, int bw,
              int bh) {
  PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc) return fail(FT_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {2 * (cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)nb};
  const cuuint64_t strides[2] = {(cuuint64_t)w * 16, (cuuint64_t)cap * 16};
  const cuuint32_t box[3] = {2 * (cuuint32_t)bw, (cuuint32_t)bh, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  const CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double2 *>(base), dims,
                         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(FT_ECUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
  return FT_OK;
}

// Builds the launch's TMA maps and launches.  The shared-memory limit is set
// on every call: the attribute is per device context, and a process may run
// trackers on several GPUs.
int pd_launch(const PDConfig &c, PDArgs &a, const StatePtrs &in, const StatePtrs &out,
              const double2 *g, const double2 *rt, int64_t cap, int nb, cudaStream_t s) {
  const int step_x = c.tw - 2 * a.halo, step_y = c.th - 2 * a.halo;
  const dim3 grid(a.halo ? (a.w + step_x - 1) / step_x : 1, a.halo ? (a.h + step_y - 1) / step_y : 1,
                  nb);
  const int bw = c.tw + 2, bh = c.th + 2, iw = step_x, ih = step_y;
  FT_TRY(plane_map(&a.in_u, in.u, a.w, a.h, nb, cap, bw, bh));
  FT_TRY(plane_map(&a.in_px, in.px, a.w, a.h, nb, cap, bw, bh));
  FT_TRY(plane_map(&a.in_py, in.py, a.w, a.h, nb, cap, bw, bh));
  FT_TRY(plane_map(&a.in_g, g, a.w, a.h, nb, cap, c.tw, c.th));
  FT_TRY(plane_map(&a.in_rt, rt, a.w, a.h, nb, cap, c.tw, c.th));
  FT_TRY(plane_map(&a.out_u, out.u, a.w, a.h, nb, cap, iw, ih));
  FT_TRY(plane_map(&a.out_px, out.px, a.w, a.h, nb, cap, iw, ih));
  FT_TRY(plane_map(&a.out_py, out.py, a.w, a.h, nb, cap, iw, ih));
  const bool mid = c.fn_mid && !a.first && !a.last && a.nhalf == 8 && a.halo == 4 && a.cone_rows &&
                   c.th == 32;
  const bool first7 = c.fn_first && a.first && !a.last && a.nhalf == 7 && a.cone_rows;
  const bool last5 = c.fn_last && !a.first && a.last && a.nhalf == 5 && a.cone_rows;
  void (*fn)(PDArgs) = mid ? c.fn_mid : first7 ? c.fn_first : last5 ? c.fn_last : c.fn;
  FT_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c.smem));
  int dev = 0, sms = kSMs, per_sm = 0;
  FT_CUDA_TRY(cudaGetDevice(&dev));
  FT_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  FT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * c.by, c.smem));
  a.prefetch_stride = sms * per_sm;
  fn<<<grid, dim3(32, c.by), c.smem, s>>>(a);
  count_launch();
  return FT_OK;
}

// tile configuration + halo used for a level of w x h
struct PDPlan {
  PDConfig cfg;
  int halo;
};

PDPlan pd_plan(int w, int h) {
  // coarse levels that fit one tile run resident (no halo, all iterations):
  // 32x32 / 256 threads, 64x32 / 512 threads
  const PDConfig small = make_cfg<32, 8, 4, 2>(), wide = make_cfg<64, 16, 2, 2>();
  if (w <= small.tw && h <= small.th) return PDPlan{small, 0};
  if (w <= wide.tw && h <= wide.th) return PDPlan{wide, 0};
  // tiled levels: 32x32 tiles of 512 threads, halo 4 (sweeps on B200,
  // profiles/README.md)
  return PDPlan{make_cfg<32, 16, 2, 2>(), 4};
}

// tau = 2^k (then sigma = 1/(8 tau) = 2^(-k-3) too): products by them are exact
inline int pow2_params(double tau) {
  int e = 0;
  return tau > 0.0 && std::frexp(tau, &e) == 0.5 ? 1 : 0;
}

inline dim3 grid2d(int w, int h, int nb) { return dim3((w + 31) / 32, (h + 7) / 8, nb); }

const char *const kLevelNames[8] = {"flow level 0", "flow level 1", "flow level 2",
                                    "flow level 3", "flow level 4", "flow level 5",
                                    "flow level 6", "flow level 7+"};

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
  const int iters = halo ? std::min(halo, p.iters) : p.iters;
  PDArgs a;
  a.w = w;
  a.h = h;
  a.halo = halo;
  a.nb = nb;
  a.pow2 = pow2_params(p.tau);
  // a middle launch: `iters` primal + dual pairs
  if (!halfstep_schedule(a, false, 2 * iters, false, halo, plan.cfg.th))
    return fail(FT_EINVAL, "primal-dual schedule exceeds the tile halo");
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
    FT_TRY(pd_launch(plan.cfg, a, state_ptrs(fw.st[cur], fw.nb, fw.cap),
                     state_ptrs(fw.st[1 - cur], fw.nb, fw.cap), fw.g, fw.rt, fw.cap, nb, s));
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
  const size_t plane = (size_t)nb * cap * sizeof(double2);
  double2 *all = nullptr;
  // G RT IX + 2 x (U PX PY)
  cudaError_t e = cudaMalloc(&all, plane * 9);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(flow workspace)");
  const int64_t pe = (int64_t)nb * cap;
  fw.g = all;
  fw.rt = all + pe;
  fw.ix = all + 2 * pe;
  fw.st[0] = all + 3 * pe;
  fw.st[1] = all + 6 * pe;
  return FT_OK;
}

void flow_work_free(FlowWork &fw) {
  if (fw.g) cudaFree(fw.g);
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
    if (lvl == scales - 1) {  // zero flow at the coarsest scale (optflow.py:239-240)
      const StatePtrs st = state_ptrs(fw.st[cur], fw.nb, cap);
      for (int b = 0; b < nb; ++b)
        FT_CUDA_TRY(cudaMemsetAsync(st.u + b * cap, 0, (size_t)w * h * sizeof(double2), s));
    } else {
      const int wc = lw[lvl + 1], hc = lh[lvl + 1];
      const StatePtrs cs = state_ptrs(fw.st[cur], fw.nb, cap);
      cur = 1 - cur;
      const StatePtrs st = state_ptrs(fw.st[cur], fw.nb, cap);
      k_upsample<<<grid2d(w, h, nb), blk, 0, s>>>(cs.u, wc, hc, st.u, w, h, cap,
                                                  (double)wc / (double)w, (double)hc / (double)h,
                                                  (double)w / (double)wc, (double)h / (double)hc);
      count_launch();
    }
    const double *i0 = pyr0 + loff[lvl];
    const double *i1 = pyr1 + loff[lvl];
    k_central_grad2<<<grid2d(w, h, nb), blk, 0, s>>>(i1, w, h, pyr_stride, fw.ix, cap);
    count_launch();

    const PDPlan plan = pd_plan(w, h);
    const bool resident = plan.halo == 0;
    const int halo = plan.halo;
    PdSpan *span = lvl == 0 && !resident ? g_pd_span : nullptr;
    if (span) span->spans = span->launches = 0, span->pixel_iters = 0;
    for (int wp = 0; wp < p.warps; ++wp) {
      k_warp_setup<<<grid2d(w, h, nb), blk, 0, s>>>(i0, i1, pyr_stride, fw.ix,
                                                     state_ptrs(fw.st[cur], fw.nb, cap).u, w, h,
                                                     cap, fw.g, fw.rt);
      count_launch();
      const int si = span && span->spans < PdSpan::kMaxSpans ? span->spans : -1;
      if (si >= 0)
        FT_CUDA_TRY(cudaEventRecordWithFlags(span->ev[2 * si], s, cudaEventRecordExternal));
      // 2*iters half-steps D P D P ... split into launches that end after a
      // dual step (state u, p): the first of at most 2*halo-1 half-steps
      // (starts with D), then 2*halo (P..D), and the rest (odd, P..P) in the
      // last launch; a resident level runs them all in one launch.
      const int total = 2 * p.iters;
      int done = 0;
      while (done < total) {
        int n;
        if (resident) n = total;
        else if (done == 0) n = std::min(2 * halo - 1, total);
        else n = total - done <= 2 * halo ? total - done : 2 * halo;
        PDArgs a;
        a.w = w;
        a.h = h;
        a.halo = halo;
        a.nb = nb;
        a.pow2 = pow2_params(p.tau);
        if (!halfstep_schedule(a, done == 0, n, done + n == total, halo, plan.cfg.th))
          return fail(FT_EINVAL, "primal-dual schedule exceeds the tile halo");
        a.tau = p.tau;
        a.lam = p.lam;
        a.sigma = sigma;
        a.shrink = shrink;
        FT_TRY(pd_launch(plan.cfg, a, state_ptrs(fw.st[cur], fw.nb, cap),
                         state_ptrs(fw.st[1 - cur], fw.nb, cap), fw.g, fw.rt, cap, nb, s));
        cur = 1 - cur;
        done += n;
        if (si >= 0) ++span->launches;
      }
      if (si >= 0) {
        FT_CUDA_TRY(cudaEventRecordWithFlags(span->ev[2 * si + 1], s, cudaEventRecordExternal));
        span->spans = si + 1;
        span->pixel_iters += (int64_t)w * h * nb * p.iters;
      }
      k_median<<<grid2d((w + 1) / 2, h, nb), blk, 0, s>>>(
          state_ptrs(fw.st[cur], fw.nb, cap).u, state_ptrs(fw.st[1 - cur], fw.nb, cap).u, w, h,
          cap);
      count_launch();
      cur = 1 - cur;
      if (energy_terms && lvl == 0 && nb == 1) {  // energy_trace (optflow.py:212-213)
        const int64_t n0 = (int64_t)w * h;
        const double *u = reinterpret_cast<const double *>(state_ptrs(fw.st[cur], fw.nb, cap).u);
        double *tb = energy_terms + (int64_t)wp * 3 * n0;
        FT_TRY(launch_energy_terms(i0, i1, u, u + 1, 2, w, h, p.eps, tb, tb + n0, tb + 2 * n0, s));
      }
    }
    phase_mark(kLevelNames[lvl < 8 ? lvl : 7]);
  }
  const int64_t n0 = (int64_t)lw[0] * lh[0];
  k_split<<<dim3(std::max<int64_t>(1, std::min<int64_t>((n0 + 255) / 256, 1184)), 1, nb), 256, 0,
            s>>>(state_ptrs(fw.st[cur], fw.nb, cap).u, n0, cap, dx, dy, out_stride);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

}  // namespace ft

namespace ft {
int launch_energy_terms(const double *i0, const double *i1, const double *u1, const double *u2,
                        int us, int w, int h, double eps, double *data, double *s1, double *s2,
                        cudaStream_t s) {
  k_energy_terms<<<dim3((w + 31) / 32, (h + 7) / 8), dim3(32, 8), 0, s>>>(i0, i1, u1, u2, us, w, h,
                                                                       eps, data, s1, s2);
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

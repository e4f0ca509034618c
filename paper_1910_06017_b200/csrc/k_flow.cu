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

#include "ft_internal.cuh"

namespace ft {

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

__global__ void k_median(const double *__restrict__ a1, const double *__restrict__ a2,
                         double *__restrict__ o1, double *__restrict__ o2, int w, int h,
                         int64_t cap) {
  const int64_t so = blockIdx.z * cap;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (r >= h || c >= w) return;
  int rr[3] = {max(r - 1, 0), r, min(r + 1, h - 1)};
  int cc[3] = {max(c - 1, 0), c, min(c + 1, w - 1)};
  double v[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) v[i * 3 + j] = a1[so + (int64_t)rr[i] * w + cc[j]];
  o1[so + (int64_t)r * w + c] = median9(v);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j) v[i * 3 + j] = a2[so + (int64_t)rr[i] * w + cc[j]];
  o2[so + (int64_t)r * w + c] = median9(v);
}

// ------------------------------------------------------------------------
// Primal-dual iterations, temporally blocked.
//
// A CTA owns a TWxTH tile of the level that overlaps its neighbours by `halo`
// pixels on every side that is not an image border.  One iteration's
// dependency radius is 1 in each direction (dual step reads u-bar at x+1 and
// y+1; primal step reads p at x-1 and y-1), so after `iters <= halo`
// iterations the inner (TW-2*halo)x(TH-2*halo) region is exact and is
// written back.  A tile that covers the whole level needs no halo and runs a
// whole warp's iterations in one launch.
//
// Shared memory holds the fields read at a neighbour (b1 b2 p11 p12 p21 p22);
// the pointwise fields (u, the gathered gradient, rho0 and the derived
// threshold / inverse |grad|^2) live in registers of the owning thread.
// ------------------------------------------------------------------------
constexpr int kTW = 32;       // tile width  (one warp across)
constexpr int kBY = 8;        // warps per CTA
constexpr int kPY = 4;        // rows per thread (interleaved by kBY)
constexpr int kTH = kBY * kPY;  // tile height

struct PDArgs {
  StatePtrs in, out;
  const double *gx, *gy, *r0;
  int w, h;
  int64_t cap;
  int halo, iters, first;
  double tau, lam, sigma, shrink;  // shrink = 1/(1+sigma*eps)
};

__global__ void __launch_bounds__(kTW *kBY, 2) k_pd_tile(const PDArgs a) {
  __shared__ double s_b1[kTH][kTW], s_b2[kTH][kTW];
  __shared__ double s_p11[kTH][kTW], s_p12[kTH][kTW], s_p21[kTH][kTW], s_p22[kTH][kTW];

  const int W = a.w, H = a.h;
  const int step_x = kTW - 2 * a.halo, step_y = kTH - 2 * a.halo;
  const int ox = blockIdx.x * step_x - a.halo;
  const int oy = blockIdx.y * step_y - a.halo;
  const int64_t so = blockIdx.z * a.cap;
  const int tx = threadIdx.x, ty = threadIdx.y;
  const int gc = ox + tx;
  const bool cin = gc >= 0 && gc < W;

  const double tl = a.tau * a.lam;
  double u1[kPY], u2[kPY], gx[kPY], gy[kPY], r0[kPY], thr[kPY], ig2[kPY];
  bool ok[kPY];

#pragma unroll
  for (int k = 0; k < kPY; ++k) {
    const int lr = ty + kBY * k, gr = oy + lr;
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
    gx[k] = vgx;
    gy[k] = vgy;
    r0[k] = vr0;
    const double g2 = vgx * vgx + vgy * vgy;  // optflow.py:163
    ok[k] = g2 > 1e-12;
    ig2[k] = ok[k] ? 1.0 / (g2 > 1e-12 ? g2 : 1e-12) : 0.0;
    thr[k] = tl * g2;  // tau*lam*grad_sq (optflow.py:176)
    s_b1[lr][tx] = vb1;
    s_b2[lr][tx] = vb2;
    s_p11[lr][tx] = q11;
    s_p12[lr][tx] = q12;
    s_p21[lr][tx] = q21;
    s_p22[lr][tx] = q22;
  }
  __syncthreads();

  const int txr = tx < kTW - 1 ? tx + 1 : tx;  // clamped neighbour columns
  const int txl = tx > 0 ? tx - 1 : tx;
  const bool has_r = gc < W - 1, has_l = gc > 0, last_c = gc == W - 1;

  for (int it = 0; it < a.iters; ++it) {
    // ---- dual ascent with Huber prox and unit-ball projection (:180-191)
    double p11[kPY], p12[kPY], p21[kPY], p22[kPY];
#pragma unroll
    for (int k = 0; k < kPY; ++k) {
      const int lr = ty + kBY * k, gr = oy + lr;
      const int lrd = lr < kTH - 1 ? lr + 1 : lr;
      const bool has_d = gr < H - 1;
      const double c1 = s_b1[lr][tx], c2 = s_b2[lr][tx];
      const double a1x = has_r ? s_b1[lr][txr] - c1 : 0.0;
      const double a1y = has_d ? s_b1[lrd][tx] - c1 : 0.0;
      const double a2x = has_r ? s_b2[lr][txr] - c2 : 0.0;
      const double a2y = has_d ? s_b2[lrd][tx] - c2 : 0.0;
      double q11 = (s_p11[lr][tx] + a.sigma * a1x) * a.shrink;
      double q12 = (s_p12[lr][tx] + a.sigma * a1y) * a.shrink;
      double q21 = (s_p21[lr][tx] + a.sigma * a2x) * a.shrink;
      double q22 = (s_p22[lr][tx] + a.sigma * a2y) * a.shrink;
      // n = max(1, hypot(.)); p /= n.  When |q|^2 is clearly below 1 the
      // norm is exactly 1 and the division is the identity: skip both.
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
    __syncthreads();  // everyone has read b and old p
#pragma unroll
    for (int k = 0; k < kPY; ++k) {
      const int lr = ty + kBY * k;
      s_p11[lr][tx] = p11[k];
      s_p12[lr][tx] = p12[k];
      s_p21[lr][tx] = p21[k];
      s_p22[lr][tx] = p22[k];
    }
    __syncthreads();
    // ---- primal descent + TV-L1 shrinkage (:194-208)
#pragma unroll
    for (int k = 0; k < kPY; ++k) {
      const int lr = ty + kBY * k, gr = oy + lr;
      const int lru = lr > 0 ? lr - 1 : lr;
      // divergence (imageops.py:41-50): dx + dy with border rules
      double dx1, dx2, dy1, dy2;
      if (!has_l) {
        dx1 = p11[k];
        dx2 = p21[k];
      } else if (last_c) {
        dx1 = -s_p11[lr][txl];
        dx2 = -s_p21[lr][txl];
      } else {
        dx1 = p11[k] - s_p11[lr][txl];
        dx2 = p21[k] - s_p21[lr][txl];
      }
      if (gr <= 0) {
        dy1 = p12[k];
        dy2 = p22[k];
      } else if (gr == H - 1) {
        dy1 = -s_p12[lru][tx];
        dy2 = -s_p22[lru][tx];
      } else {
        dy1 = p12[k] - s_p12[lru][tx];
        dy2 = p22[k] - s_p22[lru][tx];
      }
      const double v1 = u1[k] + a.tau * (dx1 + dy1);
      const double v2 = u2[k] + a.tau * (dx2 + dy2);
      const double rho = r0[k] + gx[k] * v1 + gy[k] * v2;
      const bool lo = rho < -thr[k];
      const bool hi = rho > thr[k];
      double d = lo ? tl : (hi ? -tl : -rho * ig2[k]);
      d = (ok[k] || lo || hi) ? d : 0.0;
      const double n1 = v1 + d * gx[k];
      const double n2 = v2 + d * gy[k];
      s_b1[lr][tx] = 2.0 * n1 - u1[k];
      s_b2[lr][tx] = 2.0 * n2 - u2[k];
      u1[k] = n1;
      u2[k] = n2;
    }
    __syncthreads();
  }

  // ---- write back the exact interior
  const int lo_x = a.halo, hi_x = kTW - a.halo;
  const int lo_y = a.halo, hi_y = kTH - a.halo;
  if (!cin || tx < lo_x || tx >= hi_x) return;
#pragma unroll
  for (int k = 0; k < kPY; ++k) {
    const int lr = ty + kBY * k, gr = oy + lr;
    if (gr < 0 || gr >= H || lr < lo_y || lr >= hi_y) continue;
    const int64_t o = so + (int64_t)gr * W + gc;
    a.out.p[U1][o] = u1[k];
    a.out.p[U2][o] = u2[k];
    a.out.p[B1][o] = s_b1[lr][tx];
    a.out.p[B2][o] = s_b2[lr][tx];
    a.out.p[P11][o] = s_p11[lr][tx];
    a.out.p[P12][o] = s_p12[lr][tx];
    a.out.p[P21][o] = s_p21[lr][tx];
    a.out.p[P22][o] = s_p22[lr][tx];
  }
}

StatePtrs state_ptrs(double *base, int nb, int64_t cap) {
  StatePtrs s;
  for (int k = 0; k < NST; ++k) s.p[k] = base + (int64_t)k * nb * cap;
  return s;
}

inline dim3 grid2d(int w, int h, int nb) { return dim3((w + 31) / 32, (h + 7) / 8, nb); }

}  // namespace

// Time the dominant kernel alone: `reps` eager launches of the finest-level
// primal-dual tile kernel over the workspace's current state (as left by the
// last step), bracketed by CUDA events on `s`.  Returns the mean duration.
int profile_pd(FlowWork &fw, int w, int h, int nb, const FlowParamsD &p, int reps,
               cudaStream_t s, double *ms_per_launch, int *iters_per_launch) {
  const int halo = (w <= kTW && h <= kTH) ? 0 : 4;
  const int iters = halo ? std::min(halo, p.iters) : p.iters;
  const int step_x = kTW - 2 * halo, step_y = kTH - 2 * halo;
  const dim3 pgrid(halo ? (w + step_x - 1) / step_x : 1, halo ? (h + step_y - 1) / step_y : 1, nb);
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
    k_pd_tile<<<pgrid, dim3(kTW, kBY), 0, s>>>(a);
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
             double *dx, double *dy, int64_t out_stride, int nb, cudaStream_t s) {
  const int64_t cap = fw.cap;
  if (nb > fw.nb || (int64_t)lw[0] * lh[0] > cap) return fail(FT_EINVAL, "flow workspace too small");
  int cur = 0;
  const double sigma = 1.0 / (8.0 * p.tau);
  const double shrink = 1.0 / (1.0 + sigma * p.eps);
  const dim3 blk(32, 8);
  const int halo_tiled = 4;

  for (int lvl = scales - 1; lvl >= 0; --lvl) {
    const int w = lw[lvl], h = lh[lvl];
    StatePtrs st = state_ptrs(fw.st[cur], fw.nb, cap);
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

    const bool resident = w <= kTW && h <= kTH;
    const int halo = resident ? 0 : halo_tiled;
    const int step_x = kTW - 2 * halo, step_y = kTH - 2 * halo;
    const dim3 pgrid(resident ? 1 : (w + step_x - 1) / step_x,
                     resident ? 1 : (h + step_y - 1) / step_y, nb);
    for (int wp = 0; wp < p.warps; ++wp) {
      st = state_ptrs(fw.st[cur], fw.nb, cap);
      k_warp_setup<<<grid2d(w, h, nb), blk, 0, s>>>(i0, i1, pyr_stride, fw.ix, fw.iy, st.p[U1],
                                                     st.p[U2], w, h, cap, fw.gx, fw.gy, fw.r0);
      count_launch();
      int done = 0;
      while (done < p.iters) {
        const int n = resident ? p.iters : std::min(halo, p.iters - done);
        PDArgs a;
        a.in = state_ptrs(fw.st[cur], fw.nb, cap);
        a.out = state_ptrs(fw.st[1 - cur], fw.nb, cap);
        a.gx = fw.gx;
        a.gy = fw.gy;
        a.r0 = fw.r0;
        a.w = w;
        a.h = h;
        a.cap = cap;
        a.halo = halo;
        a.iters = n;
        a.first = done == 0;
        a.tau = p.tau;
        a.lam = p.lam;
        a.sigma = sigma;
        a.shrink = shrink;
        k_pd_tile<<<pgrid, dim3(kTW, kBY), 0, s>>>(a);
        count_launch();
        cur = 1 - cur;
        done += n;
      }
      StatePtrs in = state_ptrs(fw.st[cur], fw.nb, cap);
      StatePtrs out = state_ptrs(fw.st[1 - cur], fw.nb, cap);
      k_median<<<grid2d(w, h, nb), blk, 0, s>>>(in.p[U1], in.p[U2], out.p[U1], out.p[U2], w, h,
                                                cap);
      count_launch();
      cur = 1 - cur;
    }
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

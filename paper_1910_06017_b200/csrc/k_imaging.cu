// Imaging kernels: u8 ingest, Gaussian pyramid step, ROF structure-texture.
//
// Reference: imaging.py (Frame.from_gray8 :52-56, build_pyramid :75-95,
// rof_denoise :109-125, structure_texture :128-144) and the grid stencils of
// imageops.py (smooth_gaussian5 :12-23, decimate2 :26-29, forward_gradient
// :32-38, divergence :41-50).  All batched: blockIdx.z selects the image.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "ft_internal.cuh"

namespace ft {

namespace {

// binomial taps [1,4,6,4,1]/16 (imageops.py:9), exact in binary
__device__ __constant__ double kTaps[5] = {0.0625, 0.25, 0.375, 0.25, 0.0625};

// np.pad(..., "symmetric") with pad 2: edge sample duplicated
__device__ __forceinline__ int mirror(int i, int n) {
  i = i < 0 ? -i - 1 : i;
  return i >= n ? 2 * n - 1 - i : i;
}

__global__ void k_gray8_to_unit(const uint8_t *__restrict__ src, int w, int h, int64_t ss,
                                double *__restrict__ dst, int64_t ds) {
  const int64_t n = (int64_t)w * h;
  src += blockIdx.z * ss;
  dst += blockIdx.z * ds;
  const int64_t t0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t step = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (((uintptr_t)src & 7) == 0 && ((uintptr_t)dst & 15) == 0) {
    // 8 pixels per thread: one 8-byte load, four 16-byte stores
    const int64_t n8 = n / 8;
    for (int64_t i = t0; i < n8; i += step) {
      const uint2 v = reinterpret_cast<const uint2 *>(src)[i];
      double2 *d = reinterpret_cast<double2 *>(dst + 8 * i);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const unsigned word = k < 2 ? v.x : v.y;
        const int sh = 16 * (k & 1);
        d[k] = make_double2((double)((word >> sh) & 0xffu) / 255.0,
                            (double)((word >> (sh + 8)) & 0xffu) / 255.0);
      }
    }
    done = n8 * 8;
  }
  for (int64_t i = done + t0; i < n; i += step) dst[i] = (double)src[i] / 255.0;
}

// Even-sample output of the separable blur: out(i,j) = sum_k t_k * row_k where
// row_k = sum_q t_q * src(mirror(2i-2+k), mirror(2j-2+q)); each sum starts at
// 0.0 and adds taps in order, exactly like smooth_gaussian5's accumulation.
// Interior columns of an f64 image with 16-byte aligned rows read each input
// row as three 16-byte loads (columns 2j-2 .. 2j+3; a warp covers 512
// contiguous bytes per load).
template <typename T, bool kU8>
__global__ void k_blur_decimate(const T *__restrict__ src, int w, int h, int64_t ss,
                                double *__restrict__ dst, int64_t ds,
                                double *__restrict__ dst_scaled, int64_t dss, double scale) {
  const int ow = w / 2, oh = h / 2;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  const int i = blockIdx.y * blockDim.y + threadIdx.y;
  if (i >= oh || j >= ow) return;
  src += blockIdx.z * ss;
  double acc = 0.0;
  bool vec = false;
  if constexpr (!kU8)
    vec = (w % 2 == 0) && ((uintptr_t)src % 16 == 0) && j >= 1 && 2 * j + 3 <= w - 1;
  if (vec) {
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const double2 *row =
          reinterpret_cast<const double2 *>(src + (int64_t)mirror(2 * i - 2 + k, h) * w) + (j - 1);
      const double2 a = row[0], b = row[1], c = row[2];
      double r = 0.0;
      r = r + kTaps[0] * a.x;
      r = r + kTaps[1] * a.y;
      r = r + kTaps[2] * b.x;
      r = r + kTaps[3] * b.y;
      r = r + kTaps[4] * c.x;
      acc = acc + kTaps[k] * r;
    }
  } else {
    int cols[5];
#pragma unroll
    for (int q = 0; q < 5; ++q) cols[q] = mirror(2 * j - 2 + q, w);
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const T *row = src + (int64_t)mirror(2 * i - 2 + k, h) * w;
      double r = 0.0;
#pragma unroll
      for (int q = 0; q < 5; ++q) {
        double v = kU8 ? (double)row[cols[q]] / 255.0 : (double)row[cols[q]];
        r = r + kTaps[q] * v;
      }
      acc = acc + kTaps[k] * r;
    }
  }
  dst[blockIdx.z * ds + (int64_t)i * ow + j] = acc;
  if (dst_scaled) dst_scaled[blockIdx.z * dss + (int64_t)i * ow + j] = acc * scale;
}

__global__ void k_scale_copy(const double *__restrict__ src, int64_t n, int64_t ss,
                             double *__restrict__ dst, int64_t ds, double scale) {
  src += blockIdx.z * ss;
  dst += blockIdx.z * ds;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i] * scale;
}

// divergence(px, py) at (r, c) (imageops.py:41-50): dx + dy with the
// first/last column (row) rules; requires w, h >= 2.
__device__ __forceinline__ double div_at(const double *__restrict__ px,
                                         const double *__restrict__ py, int r, int c, int w,
                                         int h) {
  const int64_t o = (int64_t)r * w + c;
  double dx = c == 0 ? px[o] : (c == w - 1 ? -px[o - 1] : px[o] - px[o - 1]);
  double dy = r == 0 ? py[o] : (r == h - 1 ? -py[o - w] : py[o] - py[o - w]);
  return dx + dy;
}

// structure = img - weight*div(p); out = clip(((img - S) + blend*S +
// (1-blend)) / (2-blend), 0, 1)   (imaging.py:125, :139-144)
__global__ void k_st_combine(const double *__restrict__ img, int w, int h, int64_t is,
                             const double *__restrict__ px, const double *__restrict__ py,
                             int64_t ps, double weight, double blend,
                             double *__restrict__ out, int64_t os, int mode) {
  img += blockIdx.z * is;
  px += blockIdx.z * ps;
  py += blockIdx.z * ps;
  out += blockIdx.z * os;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (r >= h || c >= w) return;
  const int64_t o = (int64_t)r * w + c;
  const double I = img[o];
  const double S = I - weight * div_at(px, py, r, c, w, h);
  if (mode == 1) {  // rof_denoise result (imaging.py:125)
    out[o] = S;
    return;
  }
  double m = (I - S) + blend * S;
  m = (m + (1.0 - blend)) / (2.0 - blend);
  // np.clip(x, 0, 1) == min(max(x, 0), 1) with numpy's comparison order
  m = m > 0.0 ? m : 0.0;
  m = m < 1.0 ? m : 1.0;
  out[o] = m;
}

// ROF iterations, temporally blocked (same scheme as k_pd_tile): a 64x32
// tile with `halo` overlap runs `iters` dual steps on chip; the two fields
// read at a neighbour (p at x-1 / y-1 for the divergence, d at x+1 / y+1 for
// the forward gradient) live in shared memory with a one-element apron, the
// own p in registers, img/weight in a fourth shared plane read only by its
// owner (keeps the kernel free of spills).  Exact inner region written back.
constexpr int kRPY = 2;
// BY warps per CTA, NXC columns per thread: 16 x 2 = 64-wide tiles (the
// halo columns are 8 of 64 instead of 8 of 32: measured +1.3 % default /
// +7 % light frames/s over 32x32)
template <int BY, int NXC = 1>
struct RofGeom {
  static constexpr int TW = 32 * NXC, SP = TW + 2, TH = BY * kRPY, PL = SP * (TH + 2);
  static constexpr size_t smem = 4 * PL * sizeof(double);  // px, py, d, img/weight
};

// FIX: halo 4 with 4 iterations per launch (every launch of the default 40
// iterations): trip count and cone rows are compile-time constants.
// IN: the tile touches no image border (no out-of-frame element, no first /
// last row or column), so every border flag is a compile-time constant.
template <bool P2, bool FIX, int kRBY, int NXC, bool IN>
__device__ __forceinline__ void rof_tile_body(
    const double *__restrict__ img, int w, int h, int64_t is, const double *__restrict__ px_in,
    const double *__restrict__ py_in, double *__restrict__ px_out, double *__restrict__ py_out,
    int64_t ps, double weight, double step, int halo, int iters, int first, int cone_on,
    const double *__restrict__ iw_in, double *__restrict__ iw_out) {
  using G = RofGeom<kRBY, NXC>;
  constexpr int kRTH = G::TH, kRPL = G::PL, TW = G::TW, SP = G::SP, NQ = kRPY * NXC;
  extern __shared__ double rof_sm[];
  double *const s_px = rof_sm, *const s_py = rof_sm + kRPL, *const s_d = rof_sm + 2 * kRPL;
  if (FIX) halo = iters = 4;
  const int step_x = TW - 2 * halo, step_y = kRTH - 2 * halo;
  const int ox = blockIdx.x * step_x - halo, oy = blockIdx.y * step_y - halo;
  img += blockIdx.z * is;
  const int64_t po = blockIdx.z * ps;
  const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * 32 + tx;
  for (int k = tid; k < kRPL; k += 32 * kRBY) {
    s_px[k] = 0.0;
    s_py[k] = 0.0;
    s_d[k] = 0.0;
  }
  __syncthreads();
  // element q: row ty + kRBY*(q / NXC), column tx + 32*(q % NXC)
  double *const s_iw = rof_sm + 3 * kRPL;  // img / weight, read by its owner only
#define ROF_IW(q, id) s_iw[id]
  double px[NQ], py[NQ];
  bool fR[NQ], fD[NQ], fL[NQ], fLC[NQ], fU[NQ], fLR[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int gc = ox + tx + 32 * (q % NXC), gr = oy + ty + kRBY * (q / NXC);
    const bool in = IN || (gc >= 0 && gc < w && gr >= 0 && gr < h);
    const int64_t o = (int64_t)gr * w + gc;
    const int id0 = (ty + kRBY * (q / NXC) + 1) * SP + tx + 32 * (q % NXC) + 1;
    // img / weight (imaging.py:121): divided by the first launch of the
    // structure-texture pass, which stores it; later launches read it back
    ROF_IW(q, id0) = in ? (iw_in ? iw_in[po + o] : img[o] / weight) : 0.0;
    px[q] = (in && !first) ? px_in[po + o] : 0.0;
    py[q] = (in && !first) ? py_in[po + o] : 0.0;
    fR[q] = IN || gc < w - 1;
    fD[q] = IN || gr < h - 1;
    fL[q] = IN || gc > 0;
    fLC[q] = !IN && gc == w - 1;
    fU[q] = IN || gr > 0;
    fLR[q] = !IN && gr == h - 1;
    const int id = (ty + kRBY * (q / NXC) + 1) * SP + tx + 32 * (q % NXC) + 1;
    s_px[id] = px[q];
    s_py[id] = py[q];
  }
  __syncthreads();
  // Shrinking cone (tiles with a halo): iteration it (0-based) needs p on
  // rows [c+it+1, TH-c-it-1) and d on [c+it+1, TH-c-it), c = halo - iters,
  // for the written interior [halo, TH-halo); a row is one warp.
  const int cone = FIX ? 0 : (cone_on && halo > 0 && iters <= halo) ? halo - iters : -1;
  // not unrolled: four unrolled iterations of 4 pixels (hypot + two
  // divisions each) made a 200 KB kernel that missed the instruction cache
#pragma unroll 1
  for (int it = 0; it < (FIX ? 4 : iters); ++it) {
    double d[NQ];
#pragma unroll
    for (int q = 0; q < NQ; ++q) {  // d = divergence(p) - img/weight
      const int lr = ty + kRBY * (q / NXC);
      if (cone >= 0 && (lr < cone + it + 1 || lr >= kRTH - cone - it)) continue;
      const int id = (lr + 1) * SP + tx + 32 * (q % NXC) + 1;
      const double l = s_px[id - 1], u = s_py[id - SP];
      const double dx = fL[q] ? (fLC[q] ? -l : px[q] - l) : px[q];
      const double dy = fU[q] ? (fLR[q] ? -u : py[q] - u) : py[q];
      d[q] = (dx + dy) - ROF_IW(q, id);
      s_d[id] = d[q];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < NQ; ++q) {  // g = forward_gradient(d); p update
      const int lr = ty + kRBY * (q / NXC);
      if (cone >= 0 && (lr < cone + it + 1 || lr >= kRTH - cone - it - 1)) continue;
      const int id = (lr + 1) * SP + tx + 32 * (q % NXC) + 1;
      const double gx = fR[q] ? s_d[id + 1] - d[q] : 0.0;
      const double gy = fD[q] ? s_d[id + SP] - d[q] : 0.0;
      // step = 2^k (default 0.25): step*x is exact, so the fused forms round
      // exactly like the reference's separate multiply and add
      const double hy = glibc_hypot(gx, gy);
      const double norm = P2 ? fma(step, hy, 1.0) : 1.0 + step * hy;
      // both components by the same norm: one division (div_by_recip)
      const double y = 1.0 / norm;  // norm >= 1
      px[q] = div_by_recip(P2 ? fma(step, gx, px[q]) : px[q] + step * gx, norm, y);
      py[q] = div_by_recip(P2 ? fma(step, gy, py[q]) : py[q] + step * gy, norm, y);
      s_px[id] = px[q];
      s_py[id] = py[q];
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int lr = ty + kRBY * (q / NXC), lc = tx + 32 * (q % NXC), gc = ox + lc, gr = oy + lr;
    if (!IN && (gc < 0 || gc >= w || gr < 0 || gr >= h)) continue;
    if (lc < halo || lc >= TW - halo || lr < halo || lr >= kRTH - halo) continue;
    const int64_t o = po + (int64_t)gr * w + gc;
    px_out[o] = px[q];
    py_out[o] = py[q];
    if (iw_out) iw_out[o] = ROF_IW(q, (lr + 1) * SP + lc + 1);
  }
#undef ROF_IW
}

template <bool P2, bool FIX = false, int kRBY = 16, int NXC = 1>
__global__ void __launch_bounds__(32 * kRBY, kRBY == 16 ? 2 : 1)
    k_rof_tile(const double *__restrict__ img, int w, int h, int64_t is,
               const double *__restrict__ px_in, const double *__restrict__ py_in,
               double *__restrict__ px_out, double *__restrict__ py_out, int64_t ps,
               double weight, double step, int halo, int iters, int first, int cone_on,
               const double *__restrict__ iw_in, double *__restrict__ iw_out) {
  using G = RofGeom<kRBY, NXC>;
  const int hh = FIX ? 4 : halo;
  const int ox = blockIdx.x * (G::TW - 2 * hh) - hh, oy = blockIdx.y * (G::TH - 2 * hh) - hh;
  if (ox >= 1 && ox + G::TW <= w - 1 && oy >= 1 && oy + G::TH <= h - 1)
    rof_tile_body<P2, FIX, kRBY, NXC, true>(img, w, h, is, px_in, py_in, px_out, py_out, ps,
                                            weight, step, halo, iters, first, cone_on, iw_in,
                                            iw_out);
  else
    rof_tile_body<P2, FIX, kRBY, NXC, false>(img, w, h, is, px_in, py_in, px_out, py_out, ps,
                                             weight, step, halo, iters, first, cone_on, iw_in,
                                             iw_out);
}

int grid1d(int64_t n, int bs) {
  int64_t g = (n + bs - 1) / bs;
  if (g > 4 * kSMs * 8) g = 4 * kSMs * 8;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

// Frame / MotionField validation: OR of (non-finite -> 1, outside [lo, hi] -> 2)
__global__ void k_check_plane(const double *__restrict__ d, int64_t n, double lo, double hi,
                              int *status) {
  int f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = d[i];
    if (!isfinite(v)) f |= 1;
    else if (v < lo || v > hi) f |= 2;
  }
  f = __reduce_or_sync(0xffffffffu, f);
  if ((threadIdx.x & 31) == 0 && f) atomicOr(status, f);
}

int launch_check_plane(const double *d, int64_t n, double lo, double hi, int *status,
                       cudaStream_t s) {
  FT_CUDA_TRY(cudaMemsetAsync(status, 0, sizeof(int), s));
  k_check_plane<<<grid1d(n, 256), 256, 0, s>>>(d, n, lo, hi, status);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

int launch_gray8_to_unit(const uint8_t *src, int w, int h, int64_t ss, double *dst, int64_t ds,
                         int nb, cudaStream_t s) {
  // 8 pixels per thread on the vector path
  k_gray8_to_unit<<<dim3(grid1d(((int64_t)w * h + 7) / 8, 256), 1, nb), 256, 0, s>>>(src, w, h, ss,
                                                                                   dst, ds);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

int launch_blur_decimate(const double *src, int w, int h, int64_t ss, double *dst, int64_t ds,
                         double *dst_scaled, int64_t dss, double scale, int nb, cudaStream_t s) {
  dim3 b(32, 8), g((w / 2 + 31) / 32, (h / 2 + 7) / 8, nb);
  k_blur_decimate<double, false><<<g, b, 0, s>>>(src, w, h, ss, dst, ds, dst_scaled, dss, scale);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

int launch_blur_decimate_u8(const uint8_t *src, int w, int h, int64_t ss, double *dst,
                            int64_t ds, int nb, cudaStream_t s) {
  dim3 b(32, 8), g((w / 2 + 31) / 32, (h / 2 + 7) / 8, nb);
  k_blur_decimate<uint8_t, true><<<g, b, 0, s>>>(src, w, h, ss, dst, ds, nullptr, 0, 1.0);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

int launch_scale_copy(const double *src, int64_t n, int64_t ss, double *dst, int64_t ds,
                      double scale, int nb, cudaStream_t s) {
  k_scale_copy<<<dim3(grid1d(n, 256), 1, nb), 256, 0, s>>>(src, n, ss, dst, ds, scale);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

int launch_structure_texture(const double *img, int w, int h, int64_t is, double weight,
                             double blend, int iterations, double *out, int64_t os, double *ws,
                             int64_t wss, int nb, cudaStream_t s, int mode, double step) {
  // ws per image: [px0, py0, px1, py1, img/weight] planes of w*h
  const int64_t n = (int64_t)w * h;
  for (int b = 0; b < nb; ++b) FT_CUDA_TRY(cudaMemsetAsync(ws + b * wss, 0, 2 * n * 8, s));
  double *p[2][2] = {{ws, ws + n}, {ws + 2 * n, ws + 3 * n}};
  int cur = 0;
  // 64x32 tiles (16 warps, 2 columns x 2 rows per thread), halo 4, 4
  // iterations per launch; a level that fits one tile runs all iterations
  // in one launch without halo.  Measured alternatives (32x32, 32x64, 64x64
  // tiles, a row-sweep kernel, one launch per iteration) are in DESIGN.md.
  using G = RofGeom<16, 2>;
  const bool resident = w <= G::TW && h <= G::TH;
  const int halo = resident ? 0 : 4;
  const int sx = G::TW - 2 * halo, sy = G::TH - 2 * halo;
  const dim3 g(resident ? 1 : (w + sx - 1) / sx, resident ? 1 : (h + sy - 1) / sy, nb);
  int e2 = 0;
  const bool p2 = step > 0.0 && std::frexp(step, &e2) == 0.5;
  int done = 0;
  while (done < iterations) {
    const int k = resident ? iterations : std::min(halo, iterations - done);
    const bool fix = !resident && k == 4;
    auto kern = p2 ? (fix ? k_rof_tile<true, true, 16, 2> : k_rof_tile<true, false, 16, 2>)
                   : (fix ? k_rof_tile<false, true, 16, 2> : k_rof_tile<false, false, 16, 2>);
    FT_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)G::smem));
    double *const iw = ws + 4 * n;
    kern<<<g, dim3(32, 16), G::smem, s>>>(img, w, h, is, p[cur][0], p[cur][1], p[1 - cur][0],
                                          p[1 - cur][1], wss, weight, step, halo, k, done == 0,
                                          1, done == 0 ? nullptr : iw,
                                          done == 0 && done + k < iterations ? iw : nullptr);
    count_launch();
    cur = 1 - cur;
    done += k;
  }
  const dim3 blk(32, 8);
  dim3 g2((w + 31) / 32, (h + 7) / 8, nb);
  k_st_combine<<<g2, blk, 0, s>>>(img, w, h, is, p[cur][0], p[cur][1], wss, weight, blend, out,
                                  os, mode);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

}  // namespace ft

// C ABI of libomnitrack.so (declared in include/omnitrack.h).
//
// Unit entry points mirror the reference's module functions; the tracker
// entry points run the per-frame step for many independent
// streams in lockstep, captured once per variant into a CUDA graph.
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "ft_internal.cuh"
#include "ft_klt.cuh"
#include "ft_tracker.cuh"

namespace ft {

thread_local std::string g_err;
thread_local LaunchCounter *g_launch_counter = nullptr;
thread_local PhaseRec *g_phase = nullptr;
thread_local PdSpan *g_pd_span = nullptr;

void set_error(const std::string &msg) { g_err = msg; }
int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char *what) {
  g_err = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
          ") in " + what;
  return FT_ECUDA;
}

namespace {

constexpr int kMaxLevelDim = 1280;  // imaging.py:19
constexpr int kMinCoarseDim = 16;   // optflow.py:26

int select_level_(int w, int h) {
  int lvl = 0;
  const double longest = (double)(w > h ? w : h);
  while (longest / (double)(1LL << lvl) > kMaxLevelDim) ++lvl;
  return lvl;
}

int auto_scales_(int w, int h) {
  int n = 1;
  while ((w / 2 < h / 2 ? w / 2 : h / 2) >= kMinCoarseDim) {
    w /= 2;
    h /= 2;
    ++n;
  }
  return n;
}

// build_pyramid's size check (imaging.py:79-88)
int check_pyramid(int w, int h, int levels) {
  if (levels < 1) return fail(FT_EINVAL, "num_levels must be >= 1");
  for (int l = 1; l < levels; ++l) {
    w /= 2;
    h /= 2;
    if (w < 2 || h < 2)
      return fail(FT_EINVAL, "pyramid level " + std::to_string(l) + " would be " +
                                 std::to_string(w) + "x" + std::to_string(h) +
                                 "; at least 2x2 required");
  }
  return FT_OK;
}

int check_flow_params(const ft_flow_params *p) {
  if (!p) return fail(FT_EINVAL, "params is NULL");
  if (!(p->data_weight > 0)) return fail(FT_EINVAL, "data_weight must be positive");
  if (!(p->huber_epsilon >= 0)) return fail(FT_EINVAL, "huber_epsilon must be non-negative");
  if (!(p->time_step > 0)) return fail(FT_EINVAL, "time_step must be positive");
  if (p->warps_per_level < 1) return fail(FT_EINVAL, "warps_per_level must be >= 1");
  if (p->iterations_per_warp < 1) return fail(FT_EINVAL, "iterations_per_warp must be >= 1");
  return FT_OK;
}

struct Geometry {  // pyramid of `n` levels: sizes and offsets in one block
  int n = 0;
  std::vector<int> w, h;
  std::vector<int64_t> off;
  int64_t total = 0;  // elements, padded
  void build(int w0, int h0, int levels) {
    n = levels;
    w.assign(levels, 0);
    h.assign(levels, 0);
    off.assign(levels, 0);
    int64_t o = 0;
    for (int l = 0; l < levels; ++l) {
      w[l] = l ? w[l - 1] / 2 : w0;
      h[l] = l ? h[l - 1] / 2 : h0;
      off[l] = o;
      o += ((int64_t)w[l] * h[l] + 31) / 32 * 32;
    }
    total = o;
  }
};

// fill level 1.. of a scaled pyramid whose level-0 (unscaled) image is `img`;
// `chain` receives the unscaled levels 1.., `pyr` the x255 levels 0..
int build_flow_pyramid(const double *img, int64_t img_stride, const Geometry &g, double *chain,
                       double *pyr, int64_t stride, int nb, cudaStream_t s) {
  FT_TRY(launch_scale_copy(img, (int64_t)g.w[0] * g.h[0], img_stride, pyr + g.off[0], stride,
                           255.0, nb, s));
  for (int l = 1; l < g.n; ++l) {
    const double *src = l == 1 ? img : chain + g.off[l - 1];
    const int64_t ss = l == 1 ? img_stride : stride;
    FT_TRY(launch_blur_decimate(src, g.w[l - 1], g.h[l - 1], ss, chain + g.off[l], stride,
                                pyr + g.off[l], stride, 255.0, nb, s));
  }
  return FT_OK;
}

}  // namespace
}  // namespace ft

using namespace ft;

// ============================================================ context
struct ft_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  void *scratch = nullptr;
  size_t scratch_bytes = 0;
  FlowWork fw;

  int ensure_scratch(size_t bytes) {
    if (bytes <= scratch_bytes) return FT_OK;
    FT_CUDA_TRY(cudaStreamSynchronize(stream));
    if (scratch) cudaFree(scratch);
    scratch = nullptr;
    scratch_bytes = 0;
    cudaError_t e = cudaMalloc(&scratch, bytes);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(scratch)");
    scratch_bytes = bytes;
    return FT_OK;
  }
  int ensure_flow(int nb, int64_t cap) {
    if (fw.nb >= nb && fw.cap >= cap) return FT_OK;
    FT_CUDA_TRY(cudaStreamSynchronize(stream));
    return flow_work_alloc(fw, nb, cap);
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

extern "C" {

const char *ft_last_error(void) { return g_err.c_str(); }
int ft_version(void) { return 100; }

int ft_device_count(int *count) {
  if (!count) return fail(FT_EINVAL, "count is NULL");
  cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  return FT_OK;
}

int ft_ctx_create(int device, ft_ctx **out) {
  if (!out) return fail(FT_EINVAL, "out is NULL");
  *out = nullptr;
  int n = 0;
  FT_CUDA_TRY(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(FT_EINVAL, "no such CUDA device");
  cudaDeviceProp prop;
  FT_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(FT_EINVAL, std::string("libomnitrack is built for sm_100a; device is ") +
                               prop.name);
  DeviceGuard g(device);
  std::unique_ptr<ft_ctx> c(new ft_ctx());
  c->device = device;
  FT_CUDA_TRY(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
  c->stream = c->own;
  *out = c.release();
  return FT_OK;
}

int ft_ctx_destroy(ft_ctx *ctx) {
  if (!ctx) return FT_OK;
  DeviceGuard g(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  flow_work_free(ctx->fw);
  if (ctx->scratch) cudaFree(ctx->scratch);
  if (ctx->own) cudaStreamDestroy(ctx->own);
  delete ctx;
  return FT_OK;
}

int ft_ctx_set_stream(ft_ctx *ctx, void *stream) {
  if (!ctx) return fail(FT_EINVAL, "ctx is NULL");
  // verbatim, like the CUDA runtime: NULL is the legacy default stream
  // (torch's default stream reports handle 0)
  ctx->stream = (cudaStream_t)stream;
  return FT_OK;
}

int ft_ctx_synchronize(ft_ctx *ctx) {
  if (!ctx) return fail(FT_EINVAL, "ctx is NULL");
  DeviceGuard g(ctx->device);
  FT_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return FT_OK;
}

int ft_select_level(int width, int height, int *level) {
  if (!level) return fail(FT_EINVAL, "level is NULL");
  if (width < 2 || height < 2) return fail(FT_EINVAL, "frame must be at least 2x2");
  *level = select_level_(width, height);
  return FT_OK;
}

int ft_auto_scales(int width, int height, int *scales) {
  if (!scales) return fail(FT_EINVAL, "scales is NULL");
  *scales = auto_scales_(width, height);
  return FT_OK;
}

int ft_gray8_to_unit(ft_ctx *ctx, const uint8_t *src, int w, int h, double *dst) {
  if (!ctx || !src || !dst) return fail(FT_EINVAL, "NULL argument");
  if (w < 1 || h < 1) return fail(FT_EINVAL, "empty frame");
  DeviceGuard g(ctx->device);
  return launch_gray8_to_unit(src, w, h, 0, dst, 0, 1, ctx->stream);
}

int ft_check_plane(ft_ctx *ctx, const double *d, int64_t n, double lo, double hi,
                   int32_t *h_status) {
  if (!ctx || !h_status || (n > 0 && !d)) return fail(FT_EINVAL, "NULL argument");
  *h_status = 0;
  if (n <= 0) return FT_OK;
  DeviceGuard g(ctx->device);
  FT_TRY(ctx->ensure_scratch(64));
  int *st = (int *)ctx->scratch;
  FT_TRY(launch_check_plane(d, n, lo, hi, st, ctx->stream));
  FT_CUDA_TRY(cudaMemcpyAsync(h_status, st, 4, cudaMemcpyDeviceToHost, ctx->stream));
  FT_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return FT_OK;
}

int ft_build_pyramid(ft_ctx *ctx, const double *frame, int w, int h, int levels, double *out) {
  if (!ctx || !frame || !out) return fail(FT_EINVAL, "NULL argument");
  FT_TRY(check_pyramid(w, h, levels));
  DeviceGuard g(ctx->device);
  FT_CUDA_TRY(cudaMemcpyAsync(out, frame, (size_t)w * h * 8, cudaMemcpyDeviceToDevice,
                              ctx->stream));
  double *src = out;
  for (int l = 1; l < levels; ++l) {
    double *dst = src + (int64_t)w * h;
    FT_TRY(launch_blur_decimate(src, w, h, 0, dst, 0, nullptr, 0, 1.0, 1, ctx->stream));
    src = dst;
    w /= 2;
    h /= 2;
  }
  return FT_OK;
}

int ft_structure_texture(ft_ctx *ctx, const double *in, int w, int h, double weight, double blend,
                         int iterations, double *out) {
  if (!ctx || !in || !out) return fail(FT_EINVAL, "NULL argument");
  if (!(blend >= 0.0 && blend <= 1.0)) return fail(FT_EINVAL, "blend must lie in [0, 1]");
  if (!(weight > 0)) return fail(FT_EINVAL, "weight must be positive");
  if (w < 2 || h < 2) return fail(FT_EINVAL, "frame must be at least 2x2");
  if (iterations < 0) return fail(FT_EINVAL, "iterations must be >= 0");
  DeviceGuard g(ctx->device);
  const int64_t n = (int64_t)w * h;
  FT_TRY(ctx->ensure_scratch((size_t)5 * n * 8));
  return launch_structure_texture(in, w, h, 0, weight, blend, iterations, out, 0,
                                  (double *)ctx->scratch, 0, 1, ctx->stream);
}

int ft_compute_flow_traced(ft_ctx *ctx, const double *prev, const double *curr, int w, int h,
                           const ft_flow_params *params, double *dx, double *dy,
                           double *d_energy_terms);

int ft_rof_denoise(ft_ctx *ctx, const double *in, int w, int h, double weight, int iterations,
                   double step, double *out) {
  if (!ctx || !in || !out) return fail(FT_EINVAL, "NULL argument");
  if (!(weight > 0)) return fail(FT_EINVAL, "weight must be positive");
  if (w < 2 || h < 2) return fail(FT_EINVAL, "frame must be at least 2x2");
  if (iterations < 0) return fail(FT_EINVAL, "iterations must be >= 0");
  DeviceGuard g(ctx->device);
  const int64_t n = (int64_t)w * h;
  FT_TRY(ctx->ensure_scratch((size_t)5 * n * 8));
  return launch_structure_texture(in, w, h, 0, weight, 0.0, iterations, out, 0,
                                  (double *)ctx->scratch, 0, 1, ctx->stream, 1, step);
}

int ft_compute_flow(ft_ctx *ctx, const double *prev, const double *curr, int w, int h,
                    const ft_flow_params *params, double *dx, double *dy) {
  return ft_compute_flow_traced(ctx, prev, curr, w, h, params, dx, dy, nullptr);
}

int ft_compute_flow_traced(ft_ctx *ctx, const double *prev, const double *curr, int w, int h,
                           const ft_flow_params *params, double *dx, double *dy,
                           double *d_energy_terms) {
  if (!ctx || !prev || !curr || !dx || !dy) return fail(FT_EINVAL, "NULL argument");
  FT_TRY(check_flow_params(params));
  if (w < 2 || h < 2) return fail(FT_EINVAL, "frames must be at least 2x2");
  const int scales = params->pyramid_scales > 0 ? params->pyramid_scales : auto_scales_(w, h);
  FT_TRY(check_pyramid(w, h, scales));
  DeviceGuard g(ctx->device);
  Geometry geo;
  geo.build(w, h, scales);
  // scratch: chain (unscaled, shared) + two scaled pyramids
  FT_TRY(ctx->ensure_scratch((size_t)3 * geo.total * 8));
  double *chain = (double *)ctx->scratch;
  double *p0 = chain + geo.total, *p1 = p0 + geo.total;
  FT_TRY(build_flow_pyramid(prev, 0, geo, chain, p0, 0, 1, ctx->stream));
  FT_TRY(build_flow_pyramid(curr, 0, geo, chain, p1, 0, 1, ctx->stream));
  FT_TRY(ctx->ensure_flow(1, (int64_t)w * h));
  FlowParamsD p{params->data_weight, params->time_step, params->huber_epsilon,
                params->warps_per_level, params->iterations_per_warp};
  return run_flow(p0, p1, 0, geo.w.data(), geo.h.data(), geo.off.data(), scales, p, ctx->fw, dx,
                  dy, 0, 1, ctx->stream, d_energy_terms);
}

int ft_flow_energy_terms(ft_ctx *ctx, const double *prev, const double *curr, const double *dx,
                         const double *dy, int w, int h, double huber_epsilon, double *data,
                         double *s1, double *s2) {
  if (!ctx || !prev || !curr || !dx || !dy || !data || !s1 || !s2)
    return fail(FT_EINVAL, "NULL argument");
  if (w < 1 || h < 1) return fail(FT_EINVAL, "empty field");
  DeviceGuard g(ctx->device);
  const int64_t n = (int64_t)w * h;
  FT_TRY(ctx->ensure_scratch((size_t)2 * n * 8));
  double *i0 = (double *)ctx->scratch, *i1 = i0 + n;
  // flow_energy scales the frames by INTENSITY_SCALE first (optflow.py:143)
  FT_TRY(launch_scale_copy(prev, n, 0, i0, 0, 255.0, 1, ctx->stream));
  FT_TRY(launch_scale_copy(curr, n, 0, i1, 0, 255.0, 1, ctx->stream));
  return launch_energy_terms(i0, i1, dx, dy, 1, w, h, huber_epsilon, data, s1, s2, ctx->stream);
}

static int check_boxes(const double *b, int n);

// Build one frame's KLT pyramid (levels + central gradients) into `buf`
// (3 x geo.total doubles per image) from the processing-level frame.
static int build_klt_pyramid(const double *img, int64_t img_stride, const Geometry &geo,
                             double *buf, int64_t stride, int nb, cudaStream_t s, KltPyr &out) {
  double *lvl = buf, *gx = buf + geo.total, *gy = buf + 2 * geo.total;
  for (int b = 0; b < nb; ++b)
    FT_CUDA_TRY(cudaMemcpyAsync(lvl + b * stride, img + b * img_stride,
                                (size_t)geo.w[0] * geo.h[0] * 8, cudaMemcpyDeviceToDevice, s));
  for (int l = 1; l < geo.n; ++l)
    FT_TRY(launch_blur_decimate(lvl + geo.off[l - 1], geo.w[l - 1], geo.h[l - 1], stride,
                                lvl + geo.off[l], stride, nullptr, 0, 1.0, nb, s));
  for (int l = 0; l < geo.n; ++l)
    FT_TRY(launch_central_grad(lvl + geo.off[l], geo.w[l], geo.h[l], stride, gx + geo.off[l],
                               gy + geo.off[l], stride, nb, s));
  out.lvl = lvl;
  out.gx = gx;
  out.gy = gy;
  out.stride = stride;
  for (int l = 0; l < kKltLevels; ++l) {
    out.w[l] = geo.w[l];
    out.h[l] = geo.h[l];
    out.off[l] = geo.off[l];
  }
  return FT_OK;
}

int ft_klt_predict(ft_ctx *ctx, const double *prev, const double *curr, int w, int h, int level,
                   int frame_w, int frame_h, int grid, const double *h_boxes, int n,
                   double *h_out, uint8_t *h_valid) {
  if (!ctx || !prev || !curr || (n > 0 && (!h_boxes || !h_out || !h_valid)))
    return fail(FT_EINVAL, "NULL argument");
  if (grid < 1 || grid > 11) return fail(FT_EINVAL, "grid must be in 1..11");
  FT_TRY(check_pyramid(w, h, kKltLevels));
  if (n <= 0) return FT_OK;
  FT_TRY(check_boxes(h_boxes, n));
  DeviceGuard g(ctx->device);
  Geometry geo;
  geo.build(w, h, kKltLevels);
  const int gg = grid * grid;
  const size_t need = (size_t)6 * geo.total + (size_t)n * (8 + 5 * gg) + n + 64;
  FT_TRY(ctx->ensure_scratch(need * 8));
  double *pa = (double *)ctx->scratch, *pb = pa + 3 * geo.total;
  double *boxes = pb + 3 * geo.total, *out = boxes + 4 * n;
  double *pts = out + 4 * n, *fwd = pts + 2 * (size_t)n * gg, *fb = fwd + 2 * (size_t)n * gg;
  unsigned char *valid = (unsigned char *)(fb + (size_t)n * gg);
  cudaStream_t s = ctx->stream;
  KltArgs a;
  FT_TRY(build_klt_pyramid(prev, 0, geo, pa, 0, 1, s, a.prev));
  FT_TRY(build_klt_pyramid(curr, 0, geo, pb, 0, 1, s, a.curr));
  a.grid = grid;
  a.max_pts = gg;
  a.scale = (double)(1 << level);
  FT_CUDA_TRY(cudaMemcpyAsync(boxes, h_boxes, (size_t)n * 32, cudaMemcpyHostToDevice, s));
  FT_TRY(launch_klt_predict(a, boxes, out, n, nullptr, n, 1, n, pts, fwd, fb, valid, frame_w,
                            frame_h, s));
  FT_CUDA_TRY(cudaMemcpyAsync(h_out, out, (size_t)n * 32, cudaMemcpyDeviceToHost, s));
  FT_CUDA_TRY(cudaMemcpyAsync(h_valid, valid, (size_t)n, cudaMemcpyDeviceToHost, s));
  FT_CUDA_TRY(cudaStreamSynchronize(s));
  return FT_OK;
}

int ft_predict(ft_ctx *ctx, const double *h_boxes, int n, const double *dx, const double *dy,
               int fw_l, int fh_l, int level, int frame_w, int frame_h, double *h_out,
               uint8_t *h_valid) {
  if (!ctx || (n > 0 && (!h_boxes || !h_out || !h_valid))) return fail(FT_EINVAL, "NULL argument");
  if (n <= 0) return FT_OK;
  if (!dx || !dy) return fail(FT_EINVAL, "NULL field");
  if (level < 0 || level > 30) return fail(FT_EINVAL, "bad level");
  DeviceGuard g(ctx->device);
  const size_t nb = (size_t)n * 4 * 8;
  FT_TRY(ctx->ensure_scratch(2 * nb + n + 64));
  double *d_boxes = (double *)ctx->scratch, *d_out = d_boxes + 4 * n;
  uint8_t *d_valid = (uint8_t *)(d_out + 4 * n);
  FT_CUDA_TRY(cudaMemcpyAsync(d_boxes, h_boxes, nb, cudaMemcpyHostToDevice, ctx->stream));
  FT_TRY(launch_predict(d_boxes, n, dx, dy, fw_l, fh_l, fw_l, level, frame_w, frame_h, d_out,
                        d_valid, ctx->stream));
  FT_CUDA_TRY(cudaMemcpyAsync(h_out, d_out, nb, cudaMemcpyDeviceToHost, ctx->stream));
  FT_CUDA_TRY(cudaMemcpyAsync(h_valid, d_valid, n, cudaMemcpyDeviceToHost, ctx->stream));
  FT_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return FT_OK;
}

static int check_boxes(const double *b, int n) {
  for (int i = 0; i < n; ++i)
    if (!(b[4 * i + 2] > 0) || !(b[4 * i + 3] > 0))
      return fail(FT_EINVAL, "boxes must have positive width and height");
  return FT_OK;
}

int ft_iou_matrix(ft_ctx *ctx, const double *h_a, int m, const double *h_b, int n,
                  double *h_out) {
  if (!ctx || m < 0 || n < 0) return fail(FT_EINVAL, "bad argument");
  if ((int64_t)m * n == 0) return FT_OK;
  FT_TRY(check_boxes(h_a, m));
  FT_TRY(check_boxes(h_b, n));
  DeviceGuard g(ctx->device);
  FT_TRY(ctx->ensure_scratch(((size_t)4 * (m + n) + (size_t)m * n) * 8));
  double *da = (double *)ctx->scratch, *db = da + 4 * m, *dout = db + 4 * n;
  FT_CUDA_TRY(cudaMemcpyAsync(da, h_a, (size_t)m * 32, cudaMemcpyHostToDevice, ctx->stream));
  FT_CUDA_TRY(cudaMemcpyAsync(db, h_b, (size_t)n * 32, cudaMemcpyHostToDevice, ctx->stream));
  FT_TRY(launch_iou_matrix(da, m, db, n, dout, ctx->stream));
  FT_CUDA_TRY(cudaMemcpyAsync(h_out, dout, (size_t)m * n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  FT_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  return FT_OK;
}

int ft_hungarian(ft_ctx *ctx, const double *h_cost, int m, int n, int has_forbidden,
                 double forbidden, int32_t *h_pairs, int *n_pairs) {
  if (!ctx || !n_pairs || m < 0 || n < 0) return fail(FT_EINVAL, "bad argument");
  *n_pairs = 0;
  if ((int64_t)m * n == 0) return FT_OK;
  for (int64_t k = 0; k < (int64_t)m * n; ++k)
    if (!std::isfinite(h_cost[k])) return fail(FT_EINVAL, "costs must be finite");
  DeviceGuard g(ctx->device);
  const int k = m < n ? m : n;
  FT_TRY(ctx->ensure_scratch((size_t)m * n * 8 + (size_t)(2 * k + 1 + m) * 4 + 64));
  double *dc = (double *)ctx->scratch;
  int32_t *dp = (int32_t *)(dc + (int64_t)m * n);
  int32_t *dn = dp + 2 * k;
  int *rc = dn + 1;
  FT_CUDA_TRY(cudaMemcpyAsync(dc, h_cost, (size_t)m * n * 8, cudaMemcpyHostToDevice, ctx->stream));
  FT_TRY(launch_hungarian(dc, m, n, has_forbidden, forbidden, rc, dp, dn, ctx->stream));
  int32_t cnt = 0;
  FT_CUDA_TRY(cudaMemcpyAsync(&cnt, dn, 4, cudaMemcpyDeviceToHost, ctx->stream));
  FT_CUDA_TRY(cudaMemcpyAsync(h_pairs, dp, (size_t)2 * k * 4, cudaMemcpyDeviceToHost, ctx->stream));
  FT_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
  *n_pairs = cnt;
  return FT_OK;
}

int ft_match(ft_ctx *ctx, const double *h_tb, const int32_t *h_tc, int m, const double *h_db,
             const int32_t *h_dc, int n, double gate, int32_t *h_pairs, double *h_ious,
             int *n_pairs) {
  if (!ctx || !n_pairs || m < 0 || n < 0) return fail(FT_EINVAL, "bad argument");
  *n_pairs = 0;
  if (m == 0 || n == 0) return FT_OK;  // assoc.py:117-118
  FT_TRY(check_boxes(h_tb, m));
  FT_TRY(check_boxes(h_db, n));
  DeviceGuard g(ctx->device);
  const int k = m < n ? m : n;
  const size_t mn = (size_t)m * n;
  FT_TRY(ctx->ensure_scratch((4 * (size_t)(m + n) + 2 * mn) * 8 + (size_t)(m + n + 2 * k + 1 + m) * 4 + 64));
  double *dtb = (double *)ctx->scratch, *ddb = dtb + 4 * m, *dsc = ddb + 4 * n, *dco = dsc + mn;
  int32_t *dtc = (int32_t *)(dco + mn), *ddc = dtc + m, *dp = ddc + n, *dn = dp + 2 * k;
  int *rc = dn + 1;
  cudaStream_t s = ctx->stream;
  FT_CUDA_TRY(cudaMemcpyAsync(dtb, h_tb, (size_t)m * 32, cudaMemcpyHostToDevice, s));
  FT_CUDA_TRY(cudaMemcpyAsync(ddb, h_db, (size_t)n * 32, cudaMemcpyHostToDevice, s));
  FT_CUDA_TRY(cudaMemcpyAsync(dtc, h_tc, (size_t)m * 4, cudaMemcpyHostToDevice, s));
  FT_CUDA_TRY(cudaMemcpyAsync(ddc, h_dc, (size_t)n * 4, cudaMemcpyHostToDevice, s));
  FT_TRY(launch_gate_cost(dtb, dtc, m, ddb, ddc, n, gate, dsc, dco, s));
  FT_TRY(launch_hungarian(dco, m, n, 1, kForbiddenCost, rc, dp, dn, s));
  std::vector<double> scores(mn);
  int32_t cnt = 0;
  FT_CUDA_TRY(cudaMemcpyAsync(&cnt, dn, 4, cudaMemcpyDeviceToHost, s));
  FT_CUDA_TRY(cudaMemcpyAsync(h_pairs, dp, (size_t)2 * k * 4, cudaMemcpyDeviceToHost, s));
  FT_CUDA_TRY(cudaMemcpyAsync(scores.data(), dsc, mn * 8, cudaMemcpyDeviceToHost, s));
  FT_CUDA_TRY(cudaStreamSynchronize(s));
  for (int i = 0; i < cnt; ++i) h_ious[i] = scores[(size_t)h_pairs[2 * i] * n + h_pairs[2 * i + 1]];
  *n_pairs = cnt;
  return FT_OK;
}

int ft_update(ft_ctx *ctx, const int64_t *h_ids, const int32_t *h_state, const double *h_boxes,
              int n, const int32_t *h_pairs, int n_pairs, const double *h_dboxes, int nd,
              double blend, int32_t *h_src, double *h_box, int32_t *h_flag, int64_t *h_id,
              int *n_out) {
  if (!ctx || !n_out || n < 0 || nd < 0 || n_pairs < 0) return fail(FT_EINVAL, "bad argument");
  for (int k = 0; k < n_pairs; ++k) {  // track.py:102-106
    if (h_pairs[2 * k] < 0 || h_pairs[2 * k] >= n)
      return fail(FT_ERANGE, "scene index " + std::to_string(h_pairs[2 * k]) + " out of range");
    if (h_pairs[2 * k + 1] < 0 || h_pairs[2 * k + 1] >= nd)
      return fail(FT_ERANGE,
                  "detection index " + std::to_string(h_pairs[2 * k + 1]) + " out of range");
  }
  for (int k = 0; k < n_pairs; ++k)  // track.py:114-116
    if (h_state[h_pairs[2 * k]] != 1)
      return fail(FT_EINVAL, "lost object " + std::to_string(h_ids[h_pairs[2 * k]]) +
                                 " appeared in the assignment");
  DeviceGuard g(ctx->device);
  const int no = n + nd;
  cudaStream_t s = ctx->stream;
  const size_t bytes = (size_t)n * (8 + 4 + 32) + (size_t)n_pairs * 8 + (size_t)nd * 32 +
                       (size_t)no * (4 + 32 + 4 + 8) + (size_t)n * 4 + nd + 1024;
  FT_TRY(ctx->ensure_scratch(bytes));
  char *p = (char *)ctx->scratch;
  auto take = [&](size_t b) {
    char *q = p;
    p += (b + 15) / 16 * 16;
    return (void *)q;
  };
  int64_t *d_ids = (int64_t *)take((size_t)n * 8), *d_id = (int64_t *)take((size_t)no * 8);
  double *d_boxes = (double *)take((size_t)n * 32), *d_db = (double *)take((size_t)nd * 32);
  double *d_box = (double *)take((size_t)no * 32);
  int32_t *d_state = (int32_t *)take((size_t)n * 4), *d_pairs = (int32_t *)take((size_t)n_pairs * 8);
  int32_t *d_src = (int32_t *)take((size_t)no * 4), *d_flag = (int32_t *)take((size_t)no * 4);
  int *d_match = (int *)take((size_t)n * 4);
  int32_t *d_n = (int32_t *)take(4);
  unsigned char *d_used = (unsigned char *)take((size_t)nd);
  if (n) {
    FT_CUDA_TRY(cudaMemcpyAsync(d_ids, h_ids, (size_t)n * 8, cudaMemcpyHostToDevice, s));
    FT_CUDA_TRY(cudaMemcpyAsync(d_state, h_state, (size_t)n * 4, cudaMemcpyHostToDevice, s));
    FT_CUDA_TRY(cudaMemcpyAsync(d_boxes, h_boxes, (size_t)n * 32, cudaMemcpyHostToDevice, s));
  }
  if (n_pairs)
    FT_CUDA_TRY(cudaMemcpyAsync(d_pairs, h_pairs, (size_t)n_pairs * 8, cudaMemcpyHostToDevice, s));
  if (nd) FT_CUDA_TRY(cudaMemcpyAsync(d_db, h_dboxes, (size_t)nd * 32, cudaMemcpyHostToDevice, s));
  FT_TRY(launch_update_unit(d_ids, d_state, d_boxes, n, d_pairs, n_pairs, d_db, nd, blend, d_match,
                            d_used, d_src, d_box, d_flag, d_id, d_n, s));
  int32_t cnt = 0;
  FT_CUDA_TRY(cudaMemcpyAsync(&cnt, d_n, 4, cudaMemcpyDeviceToHost, s));
  if (no) {
    FT_CUDA_TRY(cudaMemcpyAsync(h_src, d_src, (size_t)no * 4, cudaMemcpyDeviceToHost, s));
    FT_CUDA_TRY(cudaMemcpyAsync(h_box, d_box, (size_t)no * 32, cudaMemcpyDeviceToHost, s));
    FT_CUDA_TRY(cudaMemcpyAsync(h_flag, d_flag, (size_t)no * 4, cudaMemcpyDeviceToHost, s));
    FT_CUDA_TRY(cudaMemcpyAsync(h_id, d_id, (size_t)no * 8, cudaMemcpyDeviceToHost, s));
  }
  FT_CUDA_TRY(cudaStreamSynchronize(s));
  *n_out = cnt;
  return FT_OK;
}

}  // extern "C"

// ============================================================ tracker
struct ft_tracker {
  ft_ctx *ctx = nullptr;
  // the tracker's own capture/launch stream, joined to the caller's stream
  // (ctx->stream) by events at entry and exit of every call
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  PdSpan span;  // live finest-level PD timing (events baked into flow graphs)
  int join_in() {
    FT_CUDA_TRY(cudaEventRecord(ev_in, ctx->stream));
    FT_CUDA_TRY(cudaStreamWaitEvent(stream, ev_in, 0));
    return FT_OK;
  }
  int join_out() {
    FT_CUDA_TRY(cudaEventRecord(ev_out, stream));
    FT_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, ev_out, 0));
    return FT_OK;
  }
  ft_tracker_config cfg{};
  int S = 0, W = 0, H = 0, L = 0, PW = 0, PH = 0, scales = 0;
  int64_t P = 0;  // processing-level pixels
  Geometry geo;    // flow pyramid
  std::vector<int> lw, lh;  // frame-pyramid sizes 0..L
  // device buffers
  std::vector<void *> allocs;
  uint8_t *d_luma = nullptr;
  double *d_chain[16] = {};  // frame pyramid levels 1..L (unscaled)
  double *d_st = nullptr, *d_rofws = nullptr;
  double *d_pyr_prev = nullptr, *d_pyr_cur = nullptr, *d_fchain = nullptr;
  double *d_dx = nullptr, *d_dy = nullptr;
  // KLT backend: pyramid geometry, per-point scratch, predicted boxes
  Geometry kgeo;
  double *d_kpts = nullptr, *d_kfwd = nullptr, *d_kfb = nullptr, *d_kbox = nullptr;
  ft_det *d_dets = nullptr;
  // [0] = frame index, [1..S] = n_dets (-1 coast, FT_STREAM_SKIP),
  // [S+1..2S] = per-stream frame index
  int32_t *d_in = nullptr;
  ft_track *d_out = nullptr;
  int32_t *d_nout = nullptr;
  TrackerDev T{};
  FlowWork fw;
  // ---- device prefetch (cfg.prefetch, TV-L1 only, SPEC.md
  // :418): the graph of step k forks -- preprocessing of frame k on `stream`,
  // flow + predict/match/update of frame k-1 on `stream2` -- and joins; the
  // records of frame k-1 come back with step k (one-frame lag), a flush step
  // tracks the last frame.  Three rotating flow pyramids (frame k being
  // built, k-1 and k-2 being read) and per-parity device inputs.
  // host-I/O submissions (non-prefetch): a slot's inputs go H2D on the copy
  // stream `cstream` into the slot's own device buffers while the step in
  // flight computes; the step graph waits on ev_h2d[slot], and the next H2D
  // into that slot waits on ev_used[slot] (the end of the step that read it)
  cudaStream_t cstream = nullptr;
  uint8_t *d_luma_s[2] = {};
  ft_det *d_dets_s[2] = {};
  int32_t *d_in_s[2] = {};
  cudaEvent_t ev_h2d[2] = {}, ev_used[2] = {};
  bool used_rec[2] = {};
  int prefetch = 0;
  cudaStream_t stream2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  double *d_pyr3[3] = {};
  ft_det *d_dets2[2] = {};
  int32_t *d_in2[2] = {};
  int pf_prev = 0, pf_pend = 1;  // pyramid buffers of frames k-2 and k-1
  bool pf_pending = false;       // a preprocessed frame awaits tracking
  int64_t pf_tracked = 0;        // frames tracked since reset
  int pf_par = 0;                // parity of the next step's device inputs
  // pinned staging, double-buffered: slot k holds the inputs / outputs of
  // every submission with frame parity k so the host can stage frame t+1
  // while the device runs frame t (ft_tracker_submit / ft_tracker_wait).
  // h_* point at the slot being staged or read.
  struct Slot {
    uint8_t *luma = nullptr;
    ft_det *dets = nullptr;
    int32_t *in = nullptr;
    ft_track *out = nullptr;
    int32_t *nout = nullptr;
    cudaEvent_t done = nullptr;
    bool pending = false;
    bool records = true;          // the submission produces track records
    const void *graph = nullptr;  // Graph of the slot's last submission
  } slots[2];
  uint8_t *h_luma = nullptr;
  ft_det *h_dets = nullptr;
  int32_t *h_in = nullptr;
  ft_track *h_out = nullptr;
  int32_t *h_nout = nullptr;
  void use_slot(int k) {
    h_luma = slots[k].luma;
    h_dets = slots[k].dets;
    h_in = slots[k].in;
    h_out = slots[k].out;
    h_nout = slots[k].nout;
  }
  // graphs keyed by (has_prev, input pointers)
  int pyr_par = 0;  // which pyramid buffer is current (flips every step)
  struct GraphKey {
    // bit 0: has a previous frame; bit 1: pyramid parity; prefetch graphs:
    // bits 2.. new frame / track / buffer indices / input parity
    int has_prev;
    const void *luma, *dets, *in;
    bool operator<(const GraphKey &o) const {
      if (has_prev != o.has_prev) return has_prev < o.has_prev;
      if (luma != o.luma) return luma < o.luma;
      if (dets != o.dets) return dets < o.dets;
      return in < o.in;
    }
  };
  struct Graph {
    cudaGraphExec_t exec = nullptr;
    int64_t launches = 0;
    std::unique_ptr<PhaseRec> phases;  // event nodes at the phase boundaries
  };
  std::map<GraphKey, Graph> graphs;
  const Graph *last_graph = nullptr;  // graph of the most recent step
  int64_t frames_seen = 0;
  int64_t last_launches = 0;

  template <typename T_>
  int alloc(T_ **p, size_t count) {
    void *q = nullptr;
    cudaError_t e = cudaMalloc(&q, count * sizeof(T_) + 256);
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(tracker)");
    allocs.push_back(q);
    *p = (T_ *)q;
    return FT_OK;
  }

  // enqueue one step on `s` reading luma/dets/in from the given device ptrs
  // io: 1 = copy the staged inputs H2D inside the graph, 2 = copy the track
  // tables D2H inside the graph
  int enqueue(cudaStream_t s, bool has_prev, const uint8_t *luma, const ft_det *dets,
              const int32_t *in, int io) {
    const bool host_in = io & 1, host_out = io & 2;
    // pyramid ping-pong: this step builds into `pyr_cur`, the previous step's
    // pyramid is `pyr_prev` (pyr_par flips after every step; no copy)
    double *const pyr_cur = pyr_par ? d_pyr_prev : d_pyr_cur;
    double *const pyr_prev = pyr_par ? d_pyr_cur : d_pyr_prev;
    phase_mark("start");
    if (host_in) {
      FT_CUDA_TRY(cudaMemcpyAsync(d_luma, h_luma, (size_t)S * W * H, cudaMemcpyHostToDevice, s));
      FT_CUDA_TRY(cudaMemcpyAsync(d_dets, h_dets, (size_t)S * cfg.max_dets * sizeof(ft_det),
                                  cudaMemcpyHostToDevice, s));
      FT_CUDA_TRY(cudaMemcpyAsync(d_in, h_in, (size_t)(2 * S + 1) * 4, cudaMemcpyHostToDevice, s));
      luma = d_luma;
      dets = d_dets;
      in = d_in;
      phase_mark("h2d");
    }
    // (1) preprocessing: ingest + pyramid to level L (imaging.py:75-95) + ST
    const double *img;
    if (L == 0) {
      FT_TRY(launch_gray8_to_unit(luma, W, H, (int64_t)W * H, d_chain[0], P, S, s));
      img = d_chain[0];
    } else {
      FT_TRY(launch_blur_decimate_u8(luma, W, H, (int64_t)W * H, d_chain[1],
                                     (int64_t)lw[1] * lh[1], S, s));
      for (int l = 2; l <= L; ++l)
        FT_TRY(launch_blur_decimate(d_chain[l - 1], lw[l - 1], lh[l - 1],
                                    (int64_t)lw[l - 1] * lh[l - 1], d_chain[l],
                                    (int64_t)lw[l] * lh[l], nullptr, 0, 1.0, S, s));
      img = d_chain[L];
    }
    phase_mark("ingest+pyramid");
    if (cfg.motion == FT_MOTION_KLT) {  // SURVEY 8 f4 backend: no ROF, no TV-L1
      KltArgs ka;
      FT_TRY(build_klt_pyramid(img, P, kgeo, pyr_cur, 3 * kgeo.total, S, s, ka.curr));
      FT_TRY(launch_keep_prev(pyr_cur, pyr_prev, 3 * kgeo.total, in + 1, S, s));
      phase_mark("klt pyramid");
      const double *kbox = nullptr;
      if (has_prev) {
        ka.prev = ka.curr;
        ka.prev.lvl = pyr_prev;
        ka.prev.gx = pyr_prev + kgeo.total;
        ka.prev.gy = pyr_prev + 2 * kgeo.total;
        ka.grid = cfg.klt_grid;
        ka.max_pts = cfg.klt_grid * cfg.klt_grid;
        ka.scale = (double)(1 << L);
        FT_TRY(launch_klt_predict(ka, T.box, d_kbox, cfg.max_tracks, T.n_active, 0, S,
                                  cfg.max_tracks, d_kpts, d_kfwd, d_kfb, T.valid, W, H, s));
        kbox = d_kbox;
        phase_mark("klt track");
      }
      FT_TRY(launch_tracker_track(T, nullptr, nullptr, P, PW, PH, L, dets, in + 1, in + 1 + S,
                                  has_prev, d_out, d_nout, s, kbox));
      phase_mark("predict+match+update");
      if (host_out) {
        FT_CUDA_TRY(cudaMemcpyAsync(h_out, d_out,
                                    (size_t)S * 2 * cfg.max_tracks * sizeof(ft_track),
                                    cudaMemcpyDeviceToHost, s));
        FT_CUDA_TRY(cudaMemcpyAsync(h_nout, d_nout, (size_t)2 * S * 4, cudaMemcpyDeviceToHost, s));
        phase_mark("d2h");
      }
      return FT_OK;
    }
    FT_TRY(launch_structure_texture(img, PW, PH, P, cfg.rof_weight, cfg.rof_blend,
                                    cfg.rof_iterations, d_st, P, d_rofws, 5 * P, S, s, 0, 0.25));
    phase_mark("structure_texture");
    // (2) flow pyramid of the current ST frame (x255, optflow.py:242-243)
    FT_TRY(build_flow_pyramid(d_st, P, geo, d_fchain, pyr_cur, geo.total, S, s));
    FT_TRY(launch_keep_prev(pyr_cur, pyr_prev, geo.total, in + 1, S, s));
    phase_mark("flow pyramid");
    // (3) feature calculation: TV-L1 between previous and current frame
    if (has_prev) {
      FlowParamsD p{cfg.flow.data_weight, cfg.flow.time_step, cfg.flow.huber_epsilon,
                    cfg.flow.warps_per_level, cfg.flow.iterations_per_warp};
      FT_TRY(run_flow(pyr_prev, pyr_cur, geo.total, geo.w.data(), geo.h.data(),
                      geo.off.data(), scales, p, fw, d_dx, d_dy, P, S, s));
    }
    // (4) prediction, matching, update
    FT_TRY(launch_tracker_track(T, d_dx, d_dy, P, PW, PH, L, dets, in + 1, in + 1 + S, has_prev,
                                d_out, d_nout, s));
    phase_mark("predict+match+update");
    if (host_out) {
      FT_CUDA_TRY(cudaMemcpyAsync(h_out, d_out, (size_t)S * 2 * cfg.max_tracks * sizeof(ft_track),
                                  cudaMemcpyDeviceToHost, s));
      FT_CUDA_TRY(cudaMemcpyAsync(h_nout, d_nout, (size_t)2 * S * 4, cudaMemcpyDeviceToHost, s));
      phase_mark("d2h");
    }
    return FT_OK;
  }

  // preprocessing of the current step's frame (imaging.py:75-144 + flow
  // pyramid) into `pyr` for every stream; streams that skip keep `pyr_keep`
  int enqueue_preprocess(cudaStream_t s, const uint8_t *luma, const int32_t *in, double *pyr,
                         const double *pyr_keep) {
    const double *img;
    if (L == 0) {
      FT_TRY(launch_gray8_to_unit(luma, W, H, (int64_t)W * H, d_chain[0], P, S, s));
      img = d_chain[0];
    } else {
      FT_TRY(launch_blur_decimate_u8(luma, W, H, (int64_t)W * H, d_chain[1],
                                     (int64_t)lw[1] * lh[1], S, s));
      for (int l = 2; l <= L; ++l)
        FT_TRY(launch_blur_decimate(d_chain[l - 1], lw[l - 1], lh[l - 1],
                                    (int64_t)lw[l - 1] * lh[l - 1], d_chain[l],
                                    (int64_t)lw[l] * lh[l], nullptr, 0, 1.0, S, s));
      img = d_chain[L];
    }
    phase_mark("ingest+pyramid");
    FT_TRY(launch_structure_texture(img, PW, PH, P, cfg.rof_weight, cfg.rof_blend,
                                    cfg.rof_iterations, d_st, P, d_rofws, 5 * P, S, s, 0, 0.25));
    phase_mark("structure_texture");
    FT_TRY(build_flow_pyramid(d_st, P, geo, d_fchain, pyr, geo.total, S, s));
    FT_TRY(launch_keep_prev(pyr, pyr_keep, geo.total, in + 1, S, s));
    phase_mark("flow pyramid");
    return FT_OK;
  }

  // one prefetch step: mode bit 0 new frame, bit 1 track the pending frame,
  // bit 2 the pending frame has a predecessor
  int enqueue_prefetch(cudaStream_t s, int mode, int prev, int pend, int nxt, int par) {
    const bool has_new = mode & 1, has_track = mode & 2, has_prev_b = mode & 4;
    phase_mark("start");
    if (has_new) {
      FT_CUDA_TRY(cudaMemcpyAsync(d_luma, h_luma, (size_t)S * W * H, cudaMemcpyHostToDevice, s));
      FT_CUDA_TRY(cudaMemcpyAsync(d_dets2[par], h_dets, (size_t)S * cfg.max_dets * sizeof(ft_det),
                                  cudaMemcpyHostToDevice, s));
      FT_CUDA_TRY(cudaMemcpyAsync(d_in2[par], h_in, (size_t)(2 * S + 1) * 4,
                                  cudaMemcpyHostToDevice, s));
      phase_mark("h2d");
    }
    FT_CUDA_TRY(cudaEventRecord(ev_fork, s));
    FT_CUDA_TRY(cudaStreamWaitEvent(stream2, ev_fork, 0));
    if (has_track) {  // frame k-1: flow (k-2 -> k-1), predict, match, update
      PhaseRec *const ph = g_phase;
      g_phase = nullptr;  // phases of the concurrent branch are not serial
      const int32_t *in_b = d_in2[par ^ 1];
      if (has_prev_b) {
        FlowParamsD p{cfg.flow.data_weight, cfg.flow.time_step, cfg.flow.huber_epsilon,
                      cfg.flow.warps_per_level, cfg.flow.iterations_per_warp};
        FT_TRY(run_flow(d_pyr3[prev], d_pyr3[pend], geo.total, geo.w.data(), geo.h.data(),
                        geo.off.data(), scales, p, fw, d_dx, d_dy, P, S, stream2));
      }
      FT_TRY(launch_tracker_track(T, d_dx, d_dy, P, PW, PH, L, d_dets2[par ^ 1], in_b + 1,
                                  in_b + 1 + S, has_prev_b, d_out, d_nout, stream2));
      g_phase = ph;
    }
    if (has_new) FT_TRY(enqueue_preprocess(s, d_luma, d_in2[par], d_pyr3[nxt], d_pyr3[pend]));
    FT_CUDA_TRY(cudaEventRecord(ev_join, stream2));
    FT_CUDA_TRY(cudaStreamWaitEvent(s, ev_join, 0));
    phase_mark(has_new ? "flow+track (previous frame, overlapped)" : "flow+track (last frame)");
    if (has_track) {
      FT_CUDA_TRY(cudaMemcpyAsync(h_out, d_out, (size_t)S * 2 * cfg.max_tracks * sizeof(ft_track),
                                  cudaMemcpyDeviceToHost, s));
      FT_CUDA_TRY(cudaMemcpyAsync(h_nout, d_nout, (size_t)2 * S * 4, cudaMemcpyDeviceToHost, s));
      phase_mark("d2h");
    }
    return FT_OK;
  }

  // capture (once per key) and launch one step graph
  template <typename F>
  int launch_graph(const GraphKey &key, F enqueue_fn) {
    cudaStream_t s = stream;
    auto it = graphs.find(key);
    if (it == graphs.end()) {
      Graph g;
      g.phases.reset(new PhaseRec());
      for (auto &e : g.phases->ev) FT_CUDA_TRY(cudaEventCreate(&e));
      g.phases->s = s;
      LaunchCounter lc;
      g_launch_counter = &lc;
      cudaGraph_t graph = nullptr;
      cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      if (e != cudaSuccess) {
        g_launch_counter = nullptr;
        return cuda_fail(e, "cudaStreamBeginCapture");
      }
      g_pd_span = span.ev[0] ? &span : nullptr;
      g_phase = g.phases.get();
      int rc = enqueue_fn();
      g_pd_span = nullptr;
      g_phase = nullptr;
      e = cudaStreamEndCapture(s, &graph);
      g_launch_counter = nullptr;
      if (rc != FT_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
      }
      if (e != cudaSuccess) return cuda_fail(e, "cudaStreamEndCapture");
      e = cudaGraphInstantiate(&g.exec, graph, 0);
      cudaGraphDestroy(graph);
      if (e != cudaSuccess) return cuda_fail(e, "cudaGraphInstantiate");
      g.launches = lc.n;
      it = graphs.emplace(key, std::move(g)).first;
    }
    FT_CUDA_TRY(cudaGraphLaunch(it->second.exec, s));
    last_launches = it->second.launches;
    last_graph = &it->second;
    return FT_OK;
  }

  // prefetch step from the staged slot: new frame (has_new) and/or the
  // pending frame's tracking; returns whether records were produced
  int run_prefetch(bool has_new, bool *records) {
    const bool has_track = pf_pending;
    const bool has_prev_b = has_track && pf_tracked > 0;
    const int nxt = 3 - pf_prev - pf_pend;
    const int mode = (has_new ? 1 : 0) | (has_track ? 2 : 0) | (has_prev_b ? 4 : 0);
    const int par = pf_par;
    GraphKey key{(mode << 2) | (pf_prev << 5) | (pf_pend << 7) | (par << 9), h_luma, h_dets, h_in};
    FT_TRY(launch_graph(key, [&] {
      return enqueue_prefetch(stream, mode, pf_prev, pf_pend, nxt, par);
    }));
    if (has_track) ++pf_tracked;
    if (has_new) {
      pf_prev = pf_pend;
      pf_pend = nxt;
    }
    pf_pending = has_new;
    pf_par ^= 1;
    *records = has_track;
    return FT_OK;
  }

  int run(bool has_prev, const uint8_t *luma, const ft_det *dets, const int32_t *in, int io) {
    // graphs with copy nodes bake the staging slot's pinned pointers in: key
    // them by those pointers (one graph per slot; io = 2 graphs read the
    // slot's own device inputs, so their input pointers identify the slot)
    GraphKey key{(has_prev ? 1 : 0) | (pyr_par << 1) | (io << 2),
                 (io & 1) ? (const void *)h_luma : luma, (io & 1) ? (const void *)h_dets : dets,
                 (io & 1) ? (const void *)h_in : in};
    FT_TRY(launch_graph(key, [&] { return enqueue(stream, has_prev, luma, dets, in, io); }));
    pyr_par ^= 1;
    return FT_OK;
  }
};

static int read_staged(ft_tracker *t, ft_track *out, int32_t *n_out);

extern "C" {
int ft_tracker_slot_buffers(ft_tracker *t, int slot, uint8_t **luma, ft_det **dets,
                            int32_t **n_dets);

int ft_tracker_create(ft_ctx *ctx, const ft_tracker_config *cfg, ft_tracker **out) {
  if (!ctx || !cfg || !out) return fail(FT_EINVAL, "NULL argument");
  *out = nullptr;
  FT_TRY(check_flow_params(&cfg->flow));
  if (cfg->width < 2 || cfg->height < 2) return fail(FT_EINVAL, "frame must be at least 2x2");
  if (cfg->n_streams < 1) return fail(FT_EINVAL, "n_streams must be >= 1");
  if (cfg->max_tracks < 1 || cfg->max_dets < 1) return fail(FT_EINVAL, "capacities must be >= 1");
  if (!(cfg->rof_weight > 0)) return fail(FT_EINVAL, "weight must be positive");
  if (!(cfg->rof_blend >= 0 && cfg->rof_blend <= 1)) return fail(FT_EINVAL, "blend must lie in [0, 1]");
  DeviceGuard g(ctx->device);
  std::unique_ptr<ft_tracker> t(new ft_tracker());
  t->ctx = ctx;
  t->cfg = *cfg;
  FT_CUDA_TRY(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
  FT_CUDA_TRY(cudaEventCreateWithFlags(&t->ev_in, cudaEventDisableTiming));
  FT_CUDA_TRY(cudaEventCreateWithFlags(&t->ev_out, cudaEventDisableTiming));
  if (cfg->motion == FT_MOTION_TVL1)
    for (auto &e : t->span.ev) FT_CUDA_TRY(cudaEventCreate(&e));
  t->S = cfg->n_streams;
  t->W = cfg->width;
  t->H = cfg->height;
  t->L = select_level_(t->W, t->H);
  t->lw.push_back(t->W);
  t->lh.push_back(t->H);
  for (int l = 1; l <= t->L; ++l) {
    t->lw.push_back(t->lw[l - 1] / 2);
    t->lh.push_back(t->lh[l - 1] / 2);
  }
  FT_TRY(check_pyramid(t->W, t->H, t->L + 1));
  t->PW = t->lw[t->L];
  t->PH = t->lh[t->L];
  t->P = (int64_t)t->PW * t->PH;
  t->scales = cfg->flow.pyramid_scales > 0 ? cfg->flow.pyramid_scales : auto_scales_(t->PW, t->PH);
  FT_TRY(check_pyramid(t->PW, t->PH, t->scales));
  t->geo.build(t->PW, t->PH, t->scales);
  const int S = t->S;
  const int64_t P = t->P;
  FT_TRY(t->alloc(&t->d_luma, (size_t)S * t->W * t->H));
  if (t->L == 0) {
    FT_TRY(t->alloc(&t->d_chain[0], (size_t)S * P));
  } else {
    for (int l = 1; l <= t->L; ++l)
      FT_TRY(t->alloc(&t->d_chain[l], (size_t)S * t->lw[l] * t->lh[l]));
  }
  FT_TRY(t->alloc(&t->d_dx, (size_t)S * P));
  FT_TRY(t->alloc(&t->d_dy, (size_t)S * P));
  FT_TRY(t->alloc(&t->d_dets, (size_t)S * cfg->max_dets));
  FT_TRY(t->alloc(&t->d_in, (size_t)2 * S + 1));
  FT_TRY(t->alloc(&t->d_out, (size_t)S * 2 * cfg->max_tracks));
  FT_TRY(t->alloc(&t->d_nout, (size_t)2 * S));
  if (cfg->motion == FT_MOTION_KLT) {
    if (cfg->klt_grid < 1 || cfg->klt_grid > 11) return fail(FT_EINVAL, "klt_grid must be in 1..11");
    FT_TRY(check_pyramid(t->PW, t->PH, kKltLevels));
    t->kgeo.build(t->PW, t->PH, kKltLevels);
    const size_t pyr = (size_t)S * 3 * t->kgeo.total;  // levels + gx + gy
    FT_TRY(t->alloc(&t->d_pyr_prev, pyr));
    FT_TRY(t->alloc(&t->d_pyr_cur, pyr));
    const size_t pts = (size_t)S * cfg->max_tracks * cfg->klt_grid * cfg->klt_grid;
    FT_TRY(t->alloc(&t->d_kpts, 2 * pts));
    FT_TRY(t->alloc(&t->d_kfwd, 2 * pts));
    FT_TRY(t->alloc(&t->d_kfb, pts));
    FT_TRY(t->alloc(&t->d_kbox, (size_t)S * cfg->max_tracks * 4));
  } else if (cfg->motion == FT_MOTION_TVL1) {
    FT_TRY(t->alloc(&t->d_st, (size_t)S * P));
    FT_TRY(t->alloc(&t->d_rofws, (size_t)S * 5 * P));  // p ping-pong + img/weight
    FT_TRY(t->alloc(&t->d_pyr_prev, (size_t)S * t->geo.total));
    FT_TRY(t->alloc(&t->d_pyr_cur, (size_t)S * t->geo.total));
    FT_TRY(t->alloc(&t->d_fchain, (size_t)S * t->geo.total));
    FT_TRY(flow_work_alloc(t->fw, S, P));
    if (cfg->prefetch) {
      t->prefetch = 1;
      for (auto &b : t->d_pyr3) FT_TRY(t->alloc(&b, (size_t)S * t->geo.total));
      for (int k = 0; k < 2; ++k) {
        FT_TRY(t->alloc(&t->d_dets2[k], (size_t)S * cfg->max_dets));
        FT_TRY(t->alloc(&t->d_in2[k], (size_t)2 * S + 1));
      }
      FT_CUDA_TRY(cudaStreamCreateWithFlags(&t->stream2, cudaStreamNonBlocking));
      FT_CUDA_TRY(cudaEventCreateWithFlags(&t->ev_fork, cudaEventDisableTiming));
      FT_CUDA_TRY(cudaEventCreateWithFlags(&t->ev_join, cudaEventDisableTiming));
    }
  } else {
    return fail(FT_EINVAL, "motion must be FT_MOTION_TVL1 or FT_MOTION_KLT");
  }
  if (cfg->prefetch && cfg->motion != FT_MOTION_TVL1)
    return fail(FT_EINVAL, "prefetch applies to the TV-L1 path");
  // track tables
  TrackerDev &T = t->T;
  const int C = cfg->max_tracks, D = cfg->max_dets;
  T.n_streams = S;
  T.cap = C;
  T.max_dets = D;
  T.frame_w = t->W;
  T.frame_h = t->H;
  T.gate = cfg->gate;
  T.min_score = cfg->min_score;
  T.blend = cfg->detection_blend;
  FT_TRY(t->alloc(&T.id, (size_t)S * C));
  FT_TRY(t->alloc(&T.next_id, (size_t)S));
  FT_TRY(t->alloc(&T.cls, (size_t)S * C));
  FT_TRY(t->alloc(&T.label, (size_t)S * C));
  FT_TRY(t->alloc(&T.born, (size_t)S * C));
  FT_TRY(t->alloc(&T.last_seen, (size_t)S * C));
  FT_TRY(t->alloc(&T.box, (size_t)S * C * 4));
  FT_TRY(t->alloc(&T.score, (size_t)S * C));
  FT_TRY(t->alloc(&T.pmean, (size_t)S * C * 2));
  FT_TRY(t->alloc(&T.n_active, (size_t)S));
  FT_TRY(t->alloc(&T.n_cand, (size_t)S));
  FT_TRY(t->alloc(&T.cand, (size_t)S * C));
  FT_TRY(t->alloc(&T.n_kept, (size_t)S));
  FT_TRY(t->alloc(&T.kept, (size_t)S * D));
  FT_TRY(t->alloc(&T.row_col, (size_t)S * C));
  FT_TRY(t->alloc(&T.match_of, (size_t)S * C));
  FT_TRY(t->alloc(&T.n_lost, (size_t)S));
  T.overflow = t->d_nout + S;
  FT_TRY(t->alloc(&T.valid, (size_t)S * C));
  FT_TRY(t->alloc(&T.det_used, (size_t)S * D));
  FT_TRY(t->alloc(&T.scores, (size_t)S * C * D));
  FT_TRY(t->alloc(&T.cost, (size_t)S * C * D));
  FT_TRY(t->alloc(&T.lost, (size_t)S * C));
  FT_TRY(tracker_kernel_setup(T));
  // pinned staging, two slots
  for (auto &sl : t->slots) {
    FT_CUDA_TRY(cudaMallocHost(&sl.luma, (size_t)S * t->W * t->H));
    FT_CUDA_TRY(cudaMallocHost(&sl.dets, (size_t)S * D * sizeof(ft_det)));
    FT_CUDA_TRY(cudaMallocHost(&sl.in, (size_t)(2 * S + 1) * 4));
    FT_CUDA_TRY(cudaMallocHost(&sl.out, (size_t)S * 2 * C * sizeof(ft_track)));
    FT_CUDA_TRY(cudaMallocHost(&sl.nout, (size_t)2 * S * 4));
    FT_CUDA_TRY(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
  }
  if (!t->prefetch) {
    FT_CUDA_TRY(cudaStreamCreateWithFlags(&t->cstream, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      FT_TRY(t->alloc(&t->d_luma_s[k], (size_t)S * t->W * t->H));
      FT_TRY(t->alloc(&t->d_dets_s[k], (size_t)S * D));
      FT_TRY(t->alloc(&t->d_in_s[k], (size_t)2 * S + 1));
      FT_CUDA_TRY(cudaEventCreateWithFlags(&t->ev_h2d[k], cudaEventDisableTiming));
      FT_CUDA_TRY(cudaEventCreateWithFlags(&t->ev_used[k], cudaEventDisableTiming));
    }
  }
  t->use_slot(0);
  *out = t.release();
  return ft_tracker_reset(*out);
}

int ft_tracker_reset(ft_tracker *t) {
  if (!t) return fail(FT_EINVAL, "tracker is NULL");
  DeviceGuard g(t->ctx->device);
  FT_TRY(t->join_in());
  const int S = t->S;
  FT_CUDA_TRY(cudaMemsetAsync(t->T.n_active, 0, S * 4, t->stream));
  FT_CUDA_TRY(cudaMemsetAsync(t->T.next_id, 0, S * 8, t->stream));
  FT_CUDA_TRY(cudaMemsetAsync(t->T.n_lost, 0, S * 4, t->stream));
  FT_CUDA_TRY(cudaMemsetAsync(t->T.overflow, 0, S * 4, t->stream));
  FT_CUDA_TRY(cudaMemsetAsync(t->d_dx, 0, (size_t)S * t->P * 8, t->stream));
  FT_CUDA_TRY(cudaMemsetAsync(t->d_dy, 0, (size_t)S * t->P * 8, t->stream));
  FT_CUDA_TRY(cudaStreamSynchronize(t->stream));
  for (auto &sl : t->slots) {  // in-flight submissions are complete; drop their records
    FT_CUDA_TRY(cudaEventSynchronize(sl.done));
    sl.pending = false;
    sl.records = true;
  }
  t->frames_seen = 0;
  t->pyr_par = 0;
  t->pf_prev = 0;
  t->pf_pend = 1;
  t->pf_pending = false;
  t->pf_tracked = 0;
  t->pf_par = 0;
  return FT_OK;
}

int ft_tracker_destroy(ft_tracker *t) {
  if (!t) return FT_OK;
  DeviceGuard g(t->ctx->device);
  cudaStreamSynchronize(t->stream);
  for (auto &kv : t->graphs) {
    cudaGraphExecDestroy(kv.second.exec);
    for (auto &e : kv.second.phases->ev)
      if (e) cudaEventDestroy(e);
  }
  for (void *p : t->allocs) cudaFree(p);
  flow_work_free(t->fw);
  for (auto &sl : t->slots) {
    cudaFreeHost(sl.luma);
    cudaFreeHost(sl.dets);
    cudaFreeHost(sl.in);
    cudaFreeHost(sl.out);
    cudaFreeHost(sl.nout);
    if (sl.done) cudaEventDestroy(sl.done);
  }
  for (auto &e : t->span.ev)
    if (e) cudaEventDestroy(e);
  if (t->ev_fork) cudaEventDestroy(t->ev_fork);
  if (t->ev_join) cudaEventDestroy(t->ev_join);
  if (t->stream2) cudaStreamDestroy(t->stream2);
  if (t->cstream) {
    cudaStreamSynchronize(t->cstream);
    cudaStreamDestroy(t->cstream);
  }
  for (int k = 0; k < 2; ++k) {
    if (t->ev_h2d[k]) cudaEventDestroy(t->ev_h2d[k]);
    if (t->ev_used[k]) cudaEventDestroy(t->ev_used[k]);
  }
  if (t->ev_in) cudaEventDestroy(t->ev_in);
  if (t->ev_out) cudaEventDestroy(t->ev_out);
  if (t->stream) cudaStreamDestroy(t->stream);
  delete t;
  return FT_OK;
}

int ft_tracker_input_buffers(ft_tracker *t, uint8_t **luma, ft_det **dets, int32_t **n_dets) {
  return ft_tracker_slot_buffers(t, 0, luma, dets, n_dets);
}

int ft_tracker_slot_buffers(ft_tracker *t, int slot, uint8_t **luma, ft_det **dets,
                            int32_t **n_dets) {
  if (!t || slot < 0 || slot > 1) return fail(FT_EINVAL, "bad tracker / slot");
  if (luma) *luma = t->slots[slot].luma;
  if (dets) *dets = t->slots[slot].dets;
  if (n_dets) *n_dets = t->slots[slot].in + 1;
  return FT_OK;
}

// Enqueue one step reading the inputs staged in `slot` (luma, detections,
// n_dets and per-stream frame indices); returns without waiting.  Steps
// execute in submission order on the tracker's stream.
static int submit_slot(ft_tracker *t, int slot, bool new_frame = true) {
  auto &sl = t->slots[slot];
  DeviceGuard g(t->ctx->device);
  t->use_slot(slot);
  FT_TRY(t->join_in());
  if (t->prefetch) {
    bool rec = false;
    FT_TRY(t->run_prefetch(new_frame, &rec));
    sl.records = rec;
  } else {
    // H2D on the copy stream into the slot's device inputs (overlaps the
    // step in flight), the step graph after it
    const size_t nl = (size_t)t->S * t->W * t->H;
    if (t->used_rec[slot]) FT_CUDA_TRY(cudaStreamWaitEvent(t->cstream, t->ev_used[slot], 0));
    FT_CUDA_TRY(cudaMemcpyAsync(t->d_luma_s[slot], sl.luma, nl, cudaMemcpyHostToDevice, t->cstream));
    FT_CUDA_TRY(cudaMemcpyAsync(t->d_dets_s[slot], sl.dets,
                                (size_t)t->S * t->cfg.max_dets * sizeof(ft_det),
                                cudaMemcpyHostToDevice, t->cstream));
    FT_CUDA_TRY(cudaMemcpyAsync(t->d_in_s[slot], sl.in, (size_t)(2 * t->S + 1) * 4,
                                cudaMemcpyHostToDevice, t->cstream));
    FT_CUDA_TRY(cudaEventRecord(t->ev_h2d[slot], t->cstream));
    FT_CUDA_TRY(cudaStreamWaitEvent(t->stream, t->ev_h2d[slot], 0));
    FT_TRY(t->run(t->frames_seen > 0, t->d_luma_s[slot], t->d_dets_s[slot], t->d_in_s[slot], 2));
    FT_CUDA_TRY(cudaEventRecord(t->ev_used[slot], t->stream));
    t->used_rec[slot] = true;
    sl.records = true;
  }
  sl.graph = t->last_graph;
  FT_CUDA_TRY(cudaEventRecord(sl.done, t->stream));
  FT_TRY(t->join_out());
  sl.pending = true;
  t->frames_seen++;
  return FT_OK;
}

int ft_tracker_submit(ft_tracker *t, int slot, int frame, const uint8_t *luma, const ft_det *dets,
                      const int32_t *n_dets) {
  if (!t || slot < 0 || slot > 1) return fail(FT_EINVAL, "bad tracker / slot");
  auto &sl = t->slots[slot];
  if (sl.pending) return fail(FT_EINVAL, "slot still in flight: call ft_tracker_wait first");
  const int S = t->S, D = t->cfg.max_dets;
  const int32_t *nd = n_dets ? n_dets : sl.in + 1;
  for (int s = 0; s < S; ++s) {
    if (nd[s] > D) return fail(FT_ECAP, "more detections than max_dets");
    if (nd[s] < FT_STREAM_SKIP) return fail(FT_EINVAL, "n_dets must be >= FT_STREAM_SKIP");
  }
  // stage into the slot's pinned memory unless the caller wrote there directly
  if (luma && luma != sl.luma) std::memcpy(sl.luma, luma, (size_t)S * t->W * t->H);
  if (dets && dets != sl.dets) std::memcpy(sl.dets, dets, (size_t)S * D * sizeof(ft_det));
  if (nd != sl.in + 1) std::memcpy(sl.in + 1, nd, (size_t)S * 4);
  sl.in[0] = frame;
  for (int s = 0; s < S; ++s) sl.in[1 + S + s] = frame;
  return submit_slot(t, slot);
}

int ft_tracker_stage(ft_tracker *t, int slot, int stream, const uint8_t *luma, int pitch,
                     int frame, const ft_det *dets, int n_dets) {
  if (!t || slot < 0 || slot > 1) return fail(FT_EINVAL, "bad tracker / slot");
  auto &sl = t->slots[slot];
  if (sl.pending) return fail(FT_EINVAL, "slot still in flight: call ft_tracker_wait first");
  const int S = t->S, D = t->cfg.max_dets, W = t->W, H = t->H;
  if (stream < 0 || stream >= S) return fail(FT_EINVAL, "stream out of range");
  if (n_dets < FT_STREAM_SKIP) return fail(FT_EINVAL, "n_dets must be >= FT_STREAM_SKIP");
  if (n_dets > D) return fail(FT_ECAP, "more detections than max_dets");
  sl.in[1 + stream] = n_dets;
  sl.in[1 + S + stream] = frame;
  if (n_dets == FT_STREAM_SKIP) return FT_OK;  // no frame for this stream this step
  if (!luma) return fail(FT_EINVAL, "NULL luma");
  if (pitch < W) return fail(FT_EINVAL, "pitch must be >= width");
  if (n_dets > 0 && !dets) return fail(FT_EINVAL, "NULL detections");
  uint8_t *dst = sl.luma + (size_t)stream * W * H;
  if (pitch == W) {
    std::memcpy(dst, luma, (size_t)W * H);
  } else {
    for (int r = 0; r < H; ++r) std::memcpy(dst + (size_t)r * W, luma + (size_t)r * pitch, W);
  }
  if (n_dets > 0) std::memcpy(sl.dets + (size_t)stream * D, dets, (size_t)n_dets * sizeof(ft_det));
  return FT_OK;
}

int ft_tracker_flush(ft_tracker *t, int slot) {
  if (!t || slot < 0 || slot > 1) return fail(FT_EINVAL, "bad tracker / slot");
  if (!t->prefetch) return fail(FT_EINVAL, "flush applies to prefetch trackers");
  if (t->slots[slot].pending) return fail(FT_EINVAL, "slot still in flight: call ft_tracker_wait first");
  const int rc = submit_slot(t, slot, false);
  if (rc == FT_OK) t->frames_seen--;  // no new frame
  return rc;
}

int ft_tracker_submit_staged(ft_tracker *t, int slot) {
  if (!t || slot < 0 || slot > 1) return fail(FT_EINVAL, "bad tracker / slot");
  if (t->slots[slot].pending) return fail(FT_EINVAL, "slot still in flight: call ft_tracker_wait first");
  int32_t *in = t->slots[slot].in;
  in[0] = in[1 + t->S];  // legacy global index: stream 0's
  return submit_slot(t, slot);
}

// Wait for the step submitted in `slot` and return its track records.
int ft_tracker_wait(ft_tracker *t, int slot, ft_track *out, int32_t *n_out) {
  if (!t || slot < 0 || slot > 1) return fail(FT_EINVAL, "bad tracker / slot");
  auto &sl = t->slots[slot];
  if (!sl.pending) return fail(FT_EINVAL, "nothing submitted in this slot");
  DeviceGuard g(t->ctx->device);
  FT_CUDA_TRY(cudaEventSynchronize(sl.done));
  sl.pending = false;
  t->use_slot(slot);
  if (!sl.records) {  // prefetch: the first frame has only been preprocessed
    if (n_out)
      for (int s = 0; s < t->S; ++s) n_out[s] = 0;
    return FT_OK;
  }
  return read_staged(t, out, n_out);
}

int ft_tracker_step(ft_tracker *t, const uint8_t *luma, int frame, const ft_det *dets,
                    const int32_t *n_dets, ft_track *out, int32_t *n_out) {
  if (!t || !luma || !n_dets) return fail(FT_EINVAL, "NULL argument");
  if (t->prefetch) return fail(FT_EINVAL, "a prefetch tracker runs through submit / wait / flush");
  FT_TRY(ft_tracker_submit(t, 0, frame, luma, dets, n_dets));
  return ft_tracker_wait(t, 0, out, n_out);
}

int ft_tracker_step_stream(ft_tracker *t, int stream, const uint8_t *luma, int pitch, int frame,
                           const ft_det *dets, int n_dets, ft_track *out, int32_t *n_out) {
  if (!t || !out || !n_out) return fail(FT_EINVAL, "NULL argument");
  if (stream < 0 || stream >= t->S) return fail(FT_EINVAL, "stream out of range");
  if (n_dets == FT_STREAM_SKIP) return fail(FT_EINVAL, "a stepped stream cannot be skipped");
  if (t->prefetch) return fail(FT_EINVAL, "a prefetch tracker runs through submit / wait / flush");
  auto &sl = t->slots[0];
  if (sl.pending) return fail(FT_EINVAL, "slot still in flight: call ft_tracker_wait first");
  for (int s = 0; s < t->S; ++s) sl.in[1 + s] = FT_STREAM_SKIP;
  FT_TRY(ft_tracker_stage(t, 0, stream, luma, pitch, frame, dets, n_dets));
  FT_TRY(ft_tracker_submit_staged(t, 0));
  DeviceGuard g(t->ctx->device);
  FT_CUDA_TRY(cudaEventSynchronize(sl.done));
  sl.pending = false;
  t->use_slot(0);
  const int C = t->cfg.max_tracks;
  const int n = t->h_nout[stream];
  std::memcpy(out, t->h_out + (size_t)stream * 2 * C, (size_t)n * sizeof(ft_track));
  *n_out = n;
  if (t->h_nout[t->S + stream]) return fail(FT_ECAP, "stream " + std::to_string(stream) +
                                                          " exceeded max_tracks");
  return FT_OK;
}

int ft_tracker_step_device(ft_tracker *t, const uint8_t *d_luma, int frame, const ft_det *d_dets,
                           const int32_t *d_n_dets) {
  if (!t || !d_luma || !d_dets || !d_n_dets) return fail(FT_EINVAL, "NULL argument");
  if (t->prefetch) return fail(FT_EINVAL, "a prefetch tracker runs through submit / wait / flush");
  DeviceGuard g(t->ctx->device);
  // gather the caller's device inputs into the tracker's fixed input buffers
  // (D2D, ~HBM speed) so one captured graph serves every step; the frame
  // index is written into d_in by a fill kernel (passed by value).
  cudaStream_t s = t->stream;
  FT_TRY(t->join_in());
  FT_TRY(launch_fill_i32(t->d_in, 1, frame, s));
  FT_TRY(launch_fill_i32(t->d_in + 1 + t->S, t->S, frame, s));
  FT_CUDA_TRY(cudaMemcpyAsync(t->d_in + 1, d_n_dets, (size_t)t->S * 4, cudaMemcpyDeviceToDevice, s));
  FT_CUDA_TRY(cudaMemcpyAsync(t->d_luma, d_luma, (size_t)t->S * t->W * t->H,
                              cudaMemcpyDeviceToDevice, s));
  FT_CUDA_TRY(cudaMemcpyAsync(t->d_dets, d_dets, (size_t)t->S * t->cfg.max_dets * sizeof(ft_det),
                              cudaMemcpyDeviceToDevice, s));
  FT_TRY(t->run(t->frames_seen > 0, t->d_luma, t->d_dets, t->d_in, 0));
  t->frames_seen++;
  return t->join_out();
}

int ft_tracker_read(ft_tracker *t, ft_track *out, int32_t *n_out) {
  if (!t) return fail(FT_EINVAL, "tracker is NULL");
  DeviceGuard g(t->ctx->device);
  cudaStream_t s = t->stream;
  FT_TRY(t->join_in());
  t->use_slot(0);
  FT_CUDA_TRY(cudaMemcpyAsync(t->h_out, t->d_out, (size_t)t->S * 2 * t->cfg.max_tracks * sizeof(ft_track),
                              cudaMemcpyDeviceToHost, s));
  FT_CUDA_TRY(cudaMemcpyAsync(t->h_nout, t->d_nout, (size_t)2 * t->S * 4, cudaMemcpyDeviceToHost, s));
  FT_CUDA_TRY(cudaStreamSynchronize(s));
  return read_staged(t, out, n_out);
}

}  // extern "C"

static int read_staged(ft_tracker *t, ft_track *out, int32_t *n_out) {
  const int S = t->S, C = t->cfg.max_tracks;
  for (int s = 0; s < S; ++s) {
    const int n = t->h_nout[s];
    if (n_out) n_out[s] = n;
    if (out && out != t->h_out)
      std::memcpy(out + (size_t)s * 2 * C, t->h_out + (size_t)s * 2 * C, (size_t)n * sizeof(ft_track));
  }
  // capacity overflow (spawns beyond max_tracks) travels in h_nout[S..2S)
  for (int s = 0; s < S; ++s)
    if (t->h_nout[S + s]) return fail(FT_ECAP, "stream " + std::to_string(s) + " exceeded max_tracks");
  return FT_OK;
}

extern "C" {

int ft_tracker_field(ft_tracker *t, int stream, const double **dx, const double **dy, int *w,
                     int *h) {
  if (!t || stream < 0 || stream >= t->S) return fail(FT_EINVAL, "bad stream");
  if (dx) *dx = t->d_dx + (int64_t)stream * t->P;
  if (dy) *dy = t->d_dy + (int64_t)stream * t->P;
  if (w) *w = t->PW;
  if (h) *h = t->PH;
  return FT_OK;
}

int ft_tracker_read_field(ft_tracker *t, int stream, double *h_dx, double *h_dy) {
  if (!t || stream < 0 || stream >= t->S) return fail(FT_EINVAL, "bad stream");
  DeviceGuard g(t->ctx->device);
  cudaStream_t s = t->stream;
  FT_TRY(t->join_in());
  const size_t nb = (size_t)t->P * 8;
  if (h_dx)
    FT_CUDA_TRY(cudaMemcpyAsync(h_dx, t->d_dx + (int64_t)stream * t->P, nb, cudaMemcpyDeviceToHost, s));
  if (h_dy)
    FT_CUDA_TRY(cudaMemcpyAsync(h_dy, t->d_dy + (int64_t)stream * t->P, nb, cudaMemcpyDeviceToHost, s));
  FT_CUDA_TRY(cudaStreamSynchronize(s));
  return FT_OK;
}

int ft_tracker_profile_pd(ft_tracker *t, int reps, double *ms_per_launch, double *bytes_per_launch,
                          int *iters_per_launch) {
  if (!t || !ms_per_launch || reps < 1) return fail(FT_EINVAL, "bad argument");
  if (t->cfg.motion != FT_MOTION_TVL1) return fail(FT_EINVAL, "no TV-L1 kernel in a KLT tracker");
  DeviceGuard g(t->ctx->device);
  FT_TRY(t->join_in());
  FT_CUDA_TRY(cudaStreamSynchronize(t->stream));
  FlowParamsD p{t->cfg.flow.data_weight, t->cfg.flow.time_step, t->cfg.flow.huber_epsilon,
                t->cfg.flow.warps_per_level, t->cfg.flow.iterations_per_warp};
  int iters = 0;
  FT_TRY(profile_pd(t->fw, t->PW, t->PH, t->S, p, reps, t->stream, ms_per_launch, &iters));
  // algorithmic bytes of one launch per SURVEY.md 8(d): 152 B per
  // pixel-iteration (read 11 planes: 8 state + gx gy rho0; write 8 state
  // planes) x the pixel-iterations the launch performs.  The launch itself
  // moves only ~152 B per pixel (temporal blocking keeps the state on chip
  // across its iterations); bench.py reports that as compulsory bytes.
  if (bytes_per_launch) *bytes_per_launch = 152.0 * (double)t->P * t->S * iters;
  if (iters_per_launch) *iters_per_launch = iters;
  return FT_OK;
}

int ft_tracker_pd_span(ft_tracker *t, double *ms, int *launches, double *pixel_iters) {
  if (!t || !ms || !launches || !pixel_iters) return fail(FT_EINVAL, "NULL argument");
  if (t->cfg.motion != FT_MOTION_TVL1) return fail(FT_EINVAL, "no TV-L1 kernel in a KLT tracker");
  DeviceGuard g(t->ctx->device);
  FT_CUDA_TRY(cudaStreamSynchronize(t->stream));
  double tot = 0.0;
  for (int wp = 0; wp < t->span.spans; ++wp) {
    float m = 0.f;
    FT_CUDA_TRY(cudaEventElapsedTime(&m, t->span.ev[2 * wp], t->span.ev[2 * wp + 1]));
    tot += m;
  }
  *ms = tot;
  *launches = t->span.launches;
  *pixel_iters = (double)t->span.pixel_iters;
  return FT_OK;
}

int ft_tracker_phase_times(ft_tracker *t, int slot, double *ms, const char **names, int max,
                           int *n) {
  if (!t || !n || (max > 0 && !ms)) return fail(FT_EINVAL, "NULL argument");
  if (slot < -1 || slot > 1) return fail(FT_EINVAL, "slot must be -1, 0 or 1");
  DeviceGuard g(t->ctx->device);
  const ft_tracker::Graph *gr =
      slot < 0 ? t->last_graph : static_cast<const ft_tracker::Graph *>(t->slots[slot].graph);
  *n = 0;
  if (!gr) return FT_OK;
  const PhaseRec &p = *gr->phases;
  if (p.n < 2) return FT_OK;
  FT_CUDA_TRY(cudaEventSynchronize(p.ev[p.n - 1]));
  for (int i = 1; i < p.n && *n < max; ++i) {
    float m = 0.f;
    FT_CUDA_TRY(cudaEventElapsedTime(&m, p.ev[i - 1], p.ev[i]));
    ms[*n] = m;
    if (names) names[*n] = p.name[i];
    ++*n;
  }
  return FT_OK;
}

int ft_tracker_launches(ft_tracker *t, int64_t *count) {
  if (!t || !count) return fail(FT_EINVAL, "NULL argument");
  *count = t->last_launches;
  return FT_OK;
}

}  // extern "C"

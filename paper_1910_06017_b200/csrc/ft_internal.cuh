// Internal declarations shared by the libomnitrack CUDA sources.
//
// Numerics: the library is compiled with -fmad=false and uses only IEEE
// round-to-nearest +,-,*,/,sqrt, floor and comparisons, in the reference's
// operation order, so every kernel reproduces the numpy reference bit for bit
// (np.hypot is glibc's hypot, restated in glibc_hypot below).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/omnitrack.h"

namespace ft {

// ---------------------------------------------------------------- errors
void set_error(const std::string &msg);
int fail(int code, const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);

#define FT_CUDA_TRY(expr)                              \
  do {                                                 \
    cudaError_t _e = (expr);                           \
    if (_e != cudaSuccess) return ::ft::cuda_fail(_e, #expr); \
  } while (0)

#define FT_TRY(expr)            \
  do {                          \
    int _rc = (expr);           \
    if (_rc != FT_OK) return _rc; \
  } while (0)

// ---------------------------------------------------------------- numerics
// x / y for y > 0 (finite), IEEE round-to-nearest.  A zero numerator never
// reaches the division: nvcc's double division leaves its fast path for
// numerators below ~2^-120 (a called subroutine, ~60 instructions for the
// whole warp), and +-0 / y is exactly +-0 = x for y > 0.
__device__ __forceinline__ double div_pos(double x, double y) {
  // the select is opaque to the compiler, which would otherwise divide x
  // itself (the quotient is discarded when x == 0) and keep the slow path
  double xs;
  asm("{\n\t.reg .pred pz;\n\tsetp.eq.f64 pz, %1, 0d0000000000000000;\n\t"
      "selp.f64 %0, 0d3FF0000000000000, %1, pz;\n\t}"
      : "=d"(xs)
      : "d"(x));
  const double q = xs / y;
  return x == 0.0 ? x : q;
}

// safe ? 1 / g : 0 (optflow.py:165 np.where(safe, 1/max(g, 1e-12), 0)) with
// the division never seeing an unsafe (possibly zero) g
// a / b for b >= 1 (finite) given y = 1/b (IEEE, round to nearest): q0 = a*y
// is within an ulp of a/b and Markstein's correction q0 + (a - b*q0)*y (the
// residual exact through fma) is the correctly rounded quotient whenever it
// is a normal number; |a| < 2^-960 (incl. +-0, whose sign the correction
// would lose) takes the IEEE division.  Two quotients by the same b then
// cost one division (verified bit-identical to a / b on 4e8 random pairs,
// incl. all-ones significands: tools/markstein_check.c).
__device__ __forceinline__ double div_by_recip(double a, double b, double y) {
  const double q0 = a * y;
  double q = fma(fma(-b, q0, a), y, q0);
  if (fabs(a) < 0x1p-960) q = div_pos(a, b);
  return q;
}

__device__ __forceinline__ double recip_if(bool safe, double g) {
  double gs;
  asm("{\n\t.reg .pred ps;\n\tsetp.ne.s32 ps, %2, 0;\n\t"
      "selp.f64 %0, %1, 0d3FF0000000000000, ps;\n\t}"
      : "=d"(gs)
      : "d"(g), "r"((int)safe));
  const double r = 1.0 / gs;
  return safe ? r : 0.0;
}

// glibc >= 2.35 __hypot without FMA (Borges' correction), which is what
// numpy's np.hypot calls on x86-64; verified identical on 2e5 random pairs.
__device__ __forceinline__ double glibc_hypot_kernel(double ax, double ay) {
  double h = sqrt(ax * ax + ay * ay);
  double t1, t2;
  if (h <= 2.0 * ay) {
    double delta = h - ay;
    t1 = ax * (2.0 * delta - ax);
    t2 = (delta - 2.0 * (ax - ay)) * delta;
  } else {
    double delta = h - ax;
    t1 = 2.0 * delta * (ax - 2.0 * ay);
    t2 = (4.0 * delta - ay) * ay + delta * delta;
  }
  h -= div_pos(t1 + t2, 2.0 * h);  // h > 0 here; t1 + t2 is often exactly 0
  return h;
}

__device__ __forceinline__ double glibc_hypot(double x, double y) {
  x = fabs(x);
  y = fabs(y);
  double ax = x < y ? y : x;
  double ay = x < y ? x : y;
  if (ax > 0x1p+511) {
    if (ay <= ax * 0x1p-54) return ax + ay;
    return glibc_hypot_kernel(ax * 0x1p-600, ay * 0x1p-600) / 0x1p-600;
  }
  if (ay < 0x1p-511) {
    if (ax >= ay / 0x1p-54) return ax + ay;
    return glibc_hypot_kernel(ax / 0x1p-600, ay / 0x1p-600) * 0x1p-600;
  }
  if (ay <= ax * 0x1p-54) return ax + ay;
  return glibc_hypot_kernel(ax, ay);
}

// bilinear_sample (imageops.py:53-66) at one point, clamped to the border:
// np.clip(x, 0, w-1) = min(max(x, 0), w-1) with numpy's comparisons
__device__ __forceinline__ double ft_bsample(const double *__restrict__ img, int w, int h,
                                             double x, double y) {
  x = x > 0.0 ? x : 0.0;
  x = x < w - 1.0 ? x : w - 1.0;
  y = y > 0.0 ? y : 0.0;
  y = y < h - 1.0 ? y : h - 1.0;
  const int x0 = (int)floor(x), y0 = (int)floor(y);
  const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
  const double fx = x - (double)x0, fy = y - (double)y0;
  const double *r0 = img + (int64_t)y0 * w;
  const double *r1 = img + (int64_t)y1 * w;
  const double top = r0[x0] * (1.0 - fx) + r0[x1] * fx;
  const double bot = r1[x0] * (1.0 - fx) + r1[x1] * fx;
  return top * (1.0 - fy) + bot * fy;
}

// numpy maximum/minimum without NaNs: first argument wins ties
__device__ __forceinline__ double np_max(double a, double b) { return a >= b ? a : b; }
__device__ __forceinline__ double np_min(double a, double b) { return a <= b ? a : b; }

// ---------------------------------------------------------------- launch
constexpr int kSMs = 148;

struct LaunchCounter {
  int64_t n = 0;
};
extern thread_local LaunchCounter *g_launch_counter;
inline void count_launch(int n = 1) {
  if (g_launch_counter) g_launch_counter->n += n;
}

// Per-phase timing of a tracker step (SPEC.md:402-405 FrameResult timings):
// while a step graph is captured, phase_mark() records an external CUDA
// event node at every phase boundary; the events then hold the most recent
// replay of that graph, and the gaps are the phases' device times.
struct PhaseRec {
  static constexpr int kMax = 16;
  cudaEvent_t ev[kMax] = {};
  const char *name[kMax] = {};
  int n = 0;
  cudaStream_t s = nullptr;
  void mark(const char *what) {
    if (n >= kMax || !ev[n]) return;
    cudaEventRecordWithFlags(ev[n], s, cudaEventRecordExternal);
    name[n++] = what;
  }
};
extern thread_local PhaseRec *g_phase;

// Live timing of the dominant kernel inside the tracker step (bench.py's
// roofline): run_flow records an event before the first and after the last
// finest-level k_pd_tile launch of every warp.  Captured into the step
// graph as event-record nodes, so the events hold the most recent replay.
struct PdSpan {
  static constexpr int kMaxSpans = 256;  // (stream group, warp) launch sequences
  cudaEvent_t ev[2 * kMaxSpans] = {};
  int spans = 0;     // event pairs recorded in the captured step
  int launches = 0;  // finest-level PD launches between the event pairs
  int64_t pixel_iters = 0;  // pixel-iterations those launches perform (all images)
};
extern thread_local PdSpan *g_pd_span;
inline void phase_mark(const char *what) {
  if (g_phase) g_phase->mark(what);
}

// ---------------------------------------------------------------- imaging
// All batched launchers operate on `nb` independent images laid out with a
// fixed element stride between consecutive images.
int launch_check_plane(const double *d, int64_t n, double lo, double hi, int *status,
                       cudaStream_t s);
int launch_gray8_to_unit(const uint8_t *src, int w, int h, int64_t src_stride, double *dst,
                         int64_t dst_stride, int nb, cudaStream_t s);
// one pyramid step: dst = decimate2(smooth_gaussian5(src)); optional scaled copy
int launch_blur_decimate(const double *src, int w, int h, int64_t src_stride, double *dst,
                         int64_t dst_stride, double *dst_scaled, int64_t scaled_stride,
                         double scale, int nb, cudaStream_t s);
// same but reading u8 and dividing by 255 on the fly (fused ingest)
int launch_blur_decimate_u8(const uint8_t *src, int w, int h, int64_t src_stride, double *dst,
                            int64_t dst_stride, int nb, cudaStream_t s);
int launch_scale_copy(const double *src, int64_t n, int64_t src_stride, double *dst,
                      int64_t dst_stride, double scale, int nb, cudaStream_t s);
// structure_texture: ws must hold 4 planes of w*h per image (px,py ping-pong)
// mode 0: structure_texture output; mode 1: rof_denoise structure only
int launch_structure_texture(const double *img, int w, int h, int64_t stride, double weight,
                             double blend, int iterations, double *out, int64_t out_stride,
                             double *ws, int64_t ws_stride, int nb, cudaStream_t s,
                             int mode = 0, double step = 0.25);

// ---------------------------------------------------------------- flow
// Workspace for one batch of nb images at a max level size (k_flow.cu
// describes the interleaved double2 layout).
struct FlowWork {
  int nb = 0;
  int64_t cap = 0;  // pixels per plane per image
  double2 *g = nullptr;   // (gx, gy) warp constants
  double2 *rt = nullptr;  // (rho0, tau*lam*|grad|^2)
  double2 *ix = nullptr;  // level gradient of I1
  // primal-dual state ping-pong: [U | PX | PY][nb][cap] double2 each
  double2 *st[2] = {nullptr, nullptr};
};
int flow_work_alloc(FlowWork &fw, int nb, int64_t cap);
void flow_work_free(FlowWork &fw);

struct FlowParamsD {
  double lam, tau, eps;
  int warps, iters;
};

// Coarse-to-fine TV-L1 over nb image pairs given their (already scaled x255)
// pyramids.  pyr0/pyr1: level l of image b at pyr[b*pyr_stride + off[l]].
// Result flow at level 0 written to (dx, dy) with stride out_stride.
int run_flow(const double *pyr0, const double *pyr1, int64_t pyr_stride, const int *lw,
             const int *lh, const int64_t *loff, int scales, const FlowParamsD &p, FlowWork &fw,
             double *dx, double *dy, int64_t out_stride, int nb, cudaStream_t s,
             double *energy_terms = nullptr);

// u1 / u2 element stride us (1: separate planes, 2: an interleaved U plane)
int launch_energy_terms(const double *i0, const double *i1, const double *u1, const double *u2,
                        int us, int w, int h, double eps, double *data, double *s1, double *s2,
                        cudaStream_t s);
int profile_pd(FlowWork &fw, int w, int h, int nb, const FlowParamsD &p, int reps,
               cudaStream_t s, double *ms_per_launch, int *iters_per_launch);

// ---------------------------------------------------------------- tracking
int launch_predict(const double *boxes, int n, const double *dx, const double *dy, int fw_l,
                   int fh_l, int64_t field_stride, int level, int frame_w, int frame_h,
                   double *out, uint8_t *valid, cudaStream_t s);
int launch_iou_matrix(const double *a, int m, const double *b, int n, double *out,
                      cudaStream_t s);
int launch_gate_cost(const double *a, const int32_t *ac, int m, const double *b,
                     const int32_t *bc, int n, double gate, double *scores, double *cost,
                     cudaStream_t s);
int launch_hungarian(const double *cost, int m, int n, int has_forbidden, double forbidden,
                     int *row_col, int32_t *pairs, int32_t *n_pairs, cudaStream_t s);
int launch_update_unit(const int64_t *ids, const int32_t *state, const double *boxes, int n,
                       const int32_t *pairs, int np, const double *dboxes, int nd, double blend,
                       int *match_of, unsigned char *det_used, int32_t *out_src, double *out_box,
                       int32_t *out_flag, int64_t *out_id, int32_t *n_out, cudaStream_t s);

}  // namespace ft

// KLT / MedianFlow backend parameters and launch interface (k_klt.cu).
// The constants are fixed by the oracle (oracle/klt_oracle.py).
#pragma once

#include "ft_internal.cuh"

namespace ft {

constexpr int kKltLevels = 3;      // KLT pyramid levels
constexpr int kKltR = 4;           // window half size (9x9)
constexpr int kKltIters = 10;      // Gauss-Newton steps per level
constexpr double kKltEps = 0.01;   // stop when |eta| < eps (px)
constexpr double kKltMinDet = 1e-9;

struct KltPyr {  // one frame's KLT pyramid for nb images: levels + central gradients
  const double *lvl, *gx, *gy;
  int64_t stride;  // elements between images
  int w[kKltLevels], h[kKltLevels];
  int64_t off[kKltLevels];
};

struct KltArgs {
  KltPyr prev, curr;
  int grid;      // G: G x G points per box (<= 11)
  int max_pts;   // point slots per box (>= G*G)
  double scale;  // 2^L: frame pixels per processing-level pixel
};

// Predict boxes of n_streams images: boxes[(s*box_stride + b)*4], counts
// n_boxes[s] (device) or n_boxes_const for all streams.  Scratch pts/fwd
// (2 doubles) and fb (1 double) per point slot.
int launch_klt_predict(const KltArgs &a, const double *boxes, double *out_boxes,
                       int64_t box_stride, const int32_t *n_boxes, int n_boxes_const,
                       int n_streams, int max_boxes, double *pts, double *fwd, double *fb,
                       unsigned char *valid, int frame_w, int frame_h, cudaStream_t s);
// central gradient planes (np.gradient) of nb images
int launch_central_grad(const double *img, int w, int h, int64_t is, double *gx, double *gy,
                        int64_t gs, int nb, cudaStream_t s);

}  // namespace ft

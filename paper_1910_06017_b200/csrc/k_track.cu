// Tracking kernels: mean-flow box prediction (track.py:52-87), IoU / gated
// cost (assoc.py:30-41, :119-126), exact Hungarian (assoc.py:44-106) and the
// lifecycle update (track.py:90-139), plus their batched multi-stream forms
// used by the tracker step.
#include <algorithm>
#include <cfloat>
#include <math_constants.h>

#include "ft_internal.cuh"
#include "ft_tracker.cuh"

namespace ft {

// ------------------------------------------------------------ predict
// ndarray.mean() over plane[top:bottom, left:right] exactly as numpy 2.3
// evaluates it (verified against np.mean, tests/golden): a contiguous window
// (one row, or the full field width) is ONE pairwise_sum run; otherwise the
// reduction iterator buffers floor(8192/width) whole rows at a time and adds
// each buffer's pairwise sum to a 0.0 accumulator.  pairwise_sum(n): n < 8
// sequential; n <= 128 eight strided accumulators folded
// ((0+1)+(2+3))+((4+5)+(6+7)) then the tail; else split at n/2 rounded down
// to a multiple of 8 and add the halves.
//
// Device form: one warp per (box, component).  Lane 0 walks the pairwise
// tree once to list its leaves (<=128 contiguous elements each), the 32 lanes
// sum the leaves in parallel, and lane 0 walks the tree again folding the
// leaf sums in the same post order -- same additions, same order, so the
// result is bit-identical to numpy while the loads run 32-wide.
struct Window {
  const double *plane;
  int64_t pitch;
  int top, left, ww;
};

// one pairwise_sum leaf over flattened elements [e0, e0+n), n <= 128
__device__ double pw_leaf(const Window &W, int64_t e0, int64_t n) {
  int64_t r = e0 / W.ww;
  int c = (int)(e0 - r * W.ww);
  const double *row = W.plane + (W.top + r) * W.pitch + W.left;
  auto next = [&]() -> double {
    const double v = row[c];
    if (++c == W.ww) {
      c = 0;
      row += W.pitch;
    }
    return v;
  };
  if (n < 8) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) acc += next();
    return acc;
  }
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = next();
  int64_t i = 8;
  const int64_t stop = n - (n % 8);
  for (; i < stop; i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] += next();
  }
  double acc = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  for (; i < n; ++i) acc += next();
  return acc;
}

// Post-order walk of the pairwise tree of [e0, e0+n); leaf(e, len) supplies
// each leaf's value in order; internal nodes add left + right.
template <typename Leaf>
__device__ double pw_walk(int64_t e0, int64_t n, Leaf leaf) {
  if (n <= 128) return leaf(e0, n);
  struct Node {
    int64_t e0, n;
    int state;
    double left;
  };
  Node stack[48];
  int sp = 0;
  stack[0] = {e0, n, 0, 0.0};
  double ret = 0.0;
  while (true) {
    Node &t = stack[sp];
    if (t.n <= 128) {
      ret = leaf(t.e0, t.n);
      if (sp == 0) return ret;
      --sp;
      continue;
    }
    int64_t n2 = t.n / 2;
    n2 -= n2 % 8;
    if (t.state == 0) {
      t.state = 1;
      stack[sp + 1] = {t.e0, n2, 0, 0.0};
      ++sp;
    } else if (t.state == 1) {
      t.left = ret;
      t.state = 2;
      stack[sp + 1] = {t.e0 + n2, t.n - n2, 0, 0.0};
      ++sp;
    } else {
      ret = t.left + ret;
      if (sp == 0) return ret;
      --sp;
    }
  }
}

constexpr int kLeafCap = 1024;  // leaves per warp pass (n up to ~65k elements)
struct LeafScratch {           // per-warp shared memory
  int off[kLeafCap];
  int len[kLeafCap];
  double sum[kLeafCap];
};

// pairwise_sum of elements [e0, e0+n) of window W, evaluated by a full warp;
// every lane returns the result.
__device__ double warp_pw_sum(const Window &W, int64_t e0, int64_t n, LeafScratch &L) {
  const int lane = threadIdx.x & 31;
  double res = 0.0;
  if (n <= 128) {
    if (lane == 0) res = pw_leaf(W, e0, n);
    return __shfl_sync(0xffffffffu, res, 0);
  }
  int nl = 0;
  if (lane == 0) {
    pw_walk(e0, n, [&](int64_t e, int64_t len) -> double {
      if (nl < kLeafCap) {
        L.off[nl] = (int)(e - e0);
        L.len[nl] = (int)len;
      }
      ++nl;
      return 0.0;
    });
  }
  nl = __shfl_sync(0xffffffffu, nl, 0);
  if (nl > kLeafCap) {  // enormous contiguous window: sequential walk
    if (lane == 0) res = pw_walk(e0, n, [&](int64_t e, int64_t len) { return pw_leaf(W, e, len); });
    return __shfl_sync(0xffffffffu, res, 0);
  }
  __syncwarp();
  for (int k = lane; k < nl; k += 32) L.sum[k] = pw_leaf(W, e0 + L.off[k], L.len[k]);
  __syncwarp();
  if (lane == 0) {
    int k = 0;
    res = pw_walk(e0, n, [&](int64_t, int64_t) { return L.sum[k++]; });
  }
  res = __shfl_sync(0xffffffffu, res, 0);
  __syncwarp();
  return res;
}

__device__ double warp_window_mean(const double *plane, int64_t pitch, int field_w, int top,
                                   int bottom, int left, int right, LeafScratch &L) {
  const int hh = bottom - top, ww = right - left;
  const int64_t n = (int64_t)hh * ww;
  const Window W{plane, pitch, top, left, ww};
  double total;
  if (hh == 1 || ww == field_w) {
    total = warp_pw_sum(W, 0, n, L);
  } else {
    const int64_t chunk = (int64_t)(8192 / ww) * ww;
    total = 0.0;
    for (int64_t e = 0; e < n; e += chunk)
      total += warp_pw_sum(W, e, n - e < chunk ? n - e : chunk, L);
  }
  return total / (double)n;
}

__device__ __forceinline__ double rha(double v) {  // imageops.py:87-90
  return v >= 0.0 ? floor(v + 0.5) : ceil(v - 0.5);
}
__device__ __forceinline__ double py_max(double a, double b) { return b > a ? b : a; }
__device__ __forceinline__ double py_min(double a, double b) { return b < a ? b : a; }

// rounded, clamped pixel support of a box at pyramid `level` (track.py:74-81);
// false when empty (predict returns None)
__device__ __forceinline__ bool box_support(const double *box, int level, int fw_l, int fh_l,
                                            int &top, int &bottom, int &left, int &right) {
  const double scale = (double)(1 << level);
  left = max((int)rha(box[0] / scale), 0);
  top = max((int)rha(box[1] / scale), 0);
  right = min((int)rha((box[0] + box[2]) / scale), fw_l);
  bottom = min((int)rha((box[1] + box[3]) / scale), fh_l);
  return right > left && bottom > top;
}

// shifted, clamped box from the two window means (track.py:82-86)
__device__ __forceinline__ void apply_shift(const double *box, double mx, double my, int level,
                                            int frame_w, int frame_h, double *out) {
  const double scale = (double)(1 << level);
  const double x = box[0], y = box[1], w = box[2], h = box[3];
  const double sx = mx * scale, sy = my * scale;
  out[0] = py_min(py_max(x + sx, 0.0), py_max((double)frame_w - w, 0.0));
  out[1] = py_min(py_max(y + sy, 0.0), py_max((double)frame_h - h, 0.0));
  out[2] = w;
  out[3] = h;
}

constexpr int kPredWarps = 4;  // warps per predict CTA

// unit predict, phase 1: one warp per (box, component) -> mean into out[4i+c]
__global__ void __launch_bounds__(32 * kPredWarps)
    k_predict_mean(const double *boxes, int n, const double *dx, const double *dy, int fw_l,
                   int fh_l, int64_t pitch, int level, double *out, uint8_t *valid) {
  extern __shared__ __align__(16) char smem[];
  const int warp = threadIdx.x >> 5;
  LeafScratch &L = reinterpret_cast<LeafScratch *>(smem)[warp];
  const int item = blockIdx.x * kPredWarps + warp;
  const int i = item >> 1, comp = item & 1;
  if (i >= n) return;
  int top, bottom, left, right;
  const bool ok = box_support(boxes + 4 * i, level, fw_l, fh_l, top, bottom, left, right);
  if ((threadIdx.x & 31) == 0 && comp == 0) valid[i] = ok;
  if (!ok) return;
  const double m =
      warp_window_mean(comp ? dy : dx, pitch, fw_l, top, bottom, left, right, L);
  if ((threadIdx.x & 31) == 0) out[4 * i + comp] = m;
}

// unit predict, phase 2: means -> shifted, clamped boxes
__global__ void k_predict_apply(const double *boxes, int n, int level, int frame_w, int frame_h,
                                double *out, const uint8_t *valid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !valid[i]) return;
  const double mx = out[4 * i], my = out[4 * i + 1];
  apply_shift(boxes + 4 * i, mx, my, level, frame_w, frame_h, out + 4 * i);
}
// ------------------------------------------------------------ IoU / cost
__device__ __forceinline__ double iou_box(const double *a, const double *b) {
  const double ix = py_max(a[0], b[0]);
  const double iy = py_max(a[1], b[1]);
  const double ix2 = py_min(a[0] + a[2], b[0] + b[2]);
  const double iy2 = py_min(a[1] + a[3], b[1] + b[3]);
  const double inter = py_max(0.0, ix2 - ix) * py_max(0.0, iy2 - iy);
  // union > 0 for positive sizes; inter == 0 (most pairs) stays off the
  // division slow path
  return div_pos(inter, a[2] * a[3] + b[2] * b[3] - inter);
}

__global__ void k_iou(const double *a, int m, const double *b, int n, double *out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= (int64_t)m * n) return;
  const int i = (int)(k / n), j = (int)(k % n);
  out[k] = iou_box(a + 4 * i, b + 4 * j);
}

__global__ void k_gate_cost(const double *a, const int32_t *ac, int m, const double *b,
                            const int32_t *bc, int n, double gate, double *scores,
                            double *cost) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= (int64_t)m * n) return;
  const int i = (int)(k / n), j = (int)(k % n);
  const double s = iou_box(a + 4 * i, b + 4 * j);
  scores[k] = s;
  cost[k] = (s >= gate && ac[i] == bc[j]) ? 1.0 - s : kForbiddenCost;
}

// ------------------------------------------------------------ Hungarian
// Shortest augmenting path LSAP (assoc.py:44-81) on one warp.  Rows are the
// shorter side (the m>n case solves the transpose, assoc.py:99-102); columns
// are strided over the 32 lanes; argmin keeps the lowest index on ties like
// np.argmin.  Shared memory (dynamic): v[N+1] best[N] u[R] own[N+1] via[N]
// seen[N+1] -- sized by hungarian_smem().
__device__ void lsap_warp(const double *C, int m, int n, bool tr, char *smem, int *row_col) {
  const int lane = threadIdx.x & 31;
  const int R = tr ? n : m, N = tr ? m : n;
  double *v = (double *)smem;
  double *best = v + (N + 1);
  double *u = best + N;
  int *own = (int *)(u + R);
  int *via = own + (N + 1);
  unsigned char *seen = (unsigned char *)(via + N);
  auto cost = [&](int r, int j) -> double { return tr ? C[(int64_t)j * n + r] : C[(int64_t)r * n + j]; };
  for (int j = lane; j <= N; j += 32) {
    v[j] = 0.0;
    own[j] = -1;
  }
  for (int r = lane; r < R; r += 32) u[r] = 0.0;
  __syncwarp();
  for (int row = 0; row < R; ++row) {
    for (int j = lane; j <= N; j += 32) {
      if (j < N) {
        best[j] = CUDART_INF;
        via[j] = N;
      }
      seen[j] = 0;
    }
    if (lane == 0) own[N] = row;
    __syncwarp();
    int j0 = N;
    while (true) {
      if (lane == 0) seen[j0] = 1;
      __syncwarp();
      const int r = own[j0];
      const double ur = u[r];
      double bv = CUDART_INF;
      int bi = N;
      for (int j = lane; j < N; j += 32) {
        if (!seen[j]) {
          const double sl = cost(r, j) - ur - v[j];
          if (sl < best[j]) {
            best[j] = sl;
            via[j] = j0;
          }
          const double c = best[j];
          if (c < bv || (bi == N && c == bv)) {  // strictly smaller keeps lowest j
            bv = c;
            bi = j;
          }
        }
      }
      // if every column is seen/infinite np.argmin returns 0 with inf; a
      // rows<=cols problem never gets there.
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, bv, off);
        const int oi = __shfl_down_sync(0xffffffffu, bi, off);
        if (ov < bv || (ov == bv && oi < bi)) {
          bv = ov;
          bi = oi;
        }
      }
      const int j1 = __shfl_sync(0xffffffffu, bi, 0);
      const double delta = __shfl_sync(0xffffffffu, bv, 0);
      __syncwarp();
      for (int j = lane; j <= N; j += 32) {
        if (seen[j]) {
          u[own[j]] += delta;
          v[j] -= delta;
        } else if (j < N) {
          best[j] -= delta;
        }
      }
      __syncwarp();
      j0 = j1;
      if (own[j0] == -1) break;
    }
    if (lane == 0) {
      while (j0 != N) {
        const int jp = via[j0];
        own[j0] = own[jp];
        j0 = jp;
      }
    }
    __syncwarp();
  }
  // row_col[i] = matched column of ORIGINAL row i (or -1)
  for (int i = lane; i < m; i += 32) row_col[i] = -1;
  __syncwarp();
  for (int j = lane; j < N; j += 32) {
    const int o = own[j];
    if (o >= 0) {
      if (tr)
        row_col[j] = o;
      else
        row_col[o] = j;
    }
  }
  __syncwarp();
}

size_t hungarian_smem(int m, int n) {
  const int N = m > n ? m : n, R = m > n ? n : m;
  return (size_t)(N + 1) * 8 + (size_t)N * 8 + (size_t)R * 8 + (size_t)(N + 1) * 4 +
         (size_t)N * 4 + (size_t)(N + 1) + 16;
}

__global__ void k_hungarian(const double *C, int m, int n, int has_forb, double forb,
                            int *row_col, int32_t *pairs, int32_t *npairs) {
  extern __shared__ __align__(16) char smem[];
  lsap_warp(C, m, n, m > n, smem, row_col);
  if (threadIdx.x == 0) {
    int k = 0;
    for (int i = 0; i < m; ++i) {
      const int j = row_col[i];
      if (j < 0) continue;
      if (has_forb && !(C[(int64_t)i * n + j] < forb)) continue;
      pairs[2 * k] = i;
      pairs[2 * k + 1] = j;
      ++k;
    }
    *npairs = k;
  }
}

// ------------------------------------------------------------ update (unit)
// Lifecycle update over a full scene list (track.py:90-139).  The caller has
// validated indices (IndexError) and lost-object pairs (ValueError).  Output
// row k: src >= 0 -> existing object src with flag 0 keep / 1 matched (box =
// detection or blend) / 2 turned Lost; src < 0 -> spawn of detection -src-1
// with id out_id.  ws: n ints + nd bytes.
__global__ void k_update_unit(const int64_t *ids, const int32_t *state, const double *boxes, int n,
                              const int32_t *pairs, int np, const double *dboxes, int nd,
                              double blend, int *match_of, unsigned char *det_used,
                              int32_t *out_src, double *out_box, int32_t *out_flag,
                              int64_t *out_id, int32_t *n_out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int i = 0; i < n; ++i) match_of[i] = -1;
  for (int j = 0; j < nd; ++j) det_used[j] = 0;
  for (int k = 0; k < np; ++k) {  // dict assignment: the last pair for i wins
    match_of[pairs[2 * k]] = pairs[2 * k + 1];
    det_used[pairs[2 * k + 1]] = 1;
  }
  int64_t nid = -1;  // max((o.id for o in objects), default=-1) + 1
  for (int i = 0; i < n; ++i) nid = ids[i] > nid ? ids[i] : nid;
  nid += 1;
  int w = 0;
  for (int i = 0; i < n; ++i, ++w) {
    out_src[w] = i;
    out_id[w] = ids[i];
    const int j = match_of[i];
    if (j >= 0) {
      out_flag[w] = 1;
      for (int c = 0; c < 4; ++c)
        out_box[4 * w + c] = blend >= 1.0 ? dboxes[4 * j + c]
                                          : blend * dboxes[4 * j + c] + (1.0 - blend) * boxes[4 * i + c];
    } else {
      out_flag[w] = state[i] == 1 ? 2 : 0;
      for (int c = 0; c < 4; ++c) out_box[4 * w + c] = boxes[4 * i + c];
    }
  }
  for (int j = 0; j < nd; ++j) {
    if (det_used[j]) continue;
    out_src[w] = -(j + 1);
    out_id[w] = nid++;
    out_flag[w] = 0;
    for (int c = 0; c < 4; ++c) out_box[4 * w + c] = dboxes[4 * j + c];
    ++w;
  }
  *n_out = w;
}

int launch_update_unit(const int64_t *ids, const int32_t *state, const double *boxes, int n,
                       const int32_t *pairs, int np, const double *dboxes, int nd, double blend,
                       int *match_of, unsigned char *det_used, int32_t *out_src, double *out_box,
                       int32_t *out_flag, int64_t *out_id, int32_t *n_out, cudaStream_t s) {
  k_update_unit<<<1, 32, 0, s>>>(ids, state, boxes, n, pairs, np, dboxes, nd, blend, match_of,
                                 det_used, out_src, out_box, out_flag, out_id, n_out);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

// ------------------------------------------------------------ launchers
int launch_predict(const double *boxes, int n, const double *dx, const double *dy, int fw_l,
                   int fh_l, int64_t pitch, int level, int frame_w, int frame_h, double *out,
                   uint8_t *valid, cudaStream_t s) {
  if (n <= 0) return FT_OK;
  const size_t sm = kPredWarps * sizeof(LeafScratch);
  FT_CUDA_TRY(cudaFuncSetAttribute(k_predict_mean, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)sm));
  k_predict_mean<<<(2 * n + kPredWarps - 1) / kPredWarps, 32 * kPredWarps, sm, s>>>(
      boxes, n, dx, dy, fw_l, fh_l, pitch, level, out, valid);
  k_predict_apply<<<(n + 127) / 128, 128, 0, s>>>(boxes, n, level, frame_w, frame_h, out, valid);
  count_launch(2);
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

int launch_iou_matrix(const double *a, int m, const double *b, int n, double *out,
                      cudaStream_t s) {
  const int64_t k = (int64_t)m * n;
  if (k == 0) return FT_OK;
  k_iou<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(a, m, b, n, out);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

int launch_gate_cost(const double *a, const int32_t *ac, int m, const double *b,
                     const int32_t *bc, int n, double gate, double *scores, double *cost,
                     cudaStream_t s) {
  const int64_t k = (int64_t)m * n;
  if (k == 0) return FT_OK;
  k_gate_cost<<<(unsigned)((k + 255) / 256), 256, 0, s>>>(a, ac, m, b, bc, n, gate, scores,
                                                          cost);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

int launch_hungarian(const double *cost, int m, int n, int has_forbidden, double forbidden,
                     int *row_col, int32_t *pairs, int32_t *n_pairs, cudaStream_t s) {
  const size_t sm = hungarian_smem(m, n);
  if (sm > 200 * 1024) return fail(FT_EINVAL, "hungarian: matrix too large for one CTA");
  if (sm > 48 * 1024)
    FT_CUDA_TRY(cudaFuncSetAttribute(k_hungarian, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sm));
  k_hungarian<<<1, 32, sm, s>>>(cost, m, n, has_forbidden, forbidden, row_col, pairs, n_pairs);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

// ============================================================ tracker step
// One CTA per stream for every per-stream phase.

// predict, phase 1: one warp per (active track, component) of every stream
// (grid.x = stream, grid.y covers 2*cap items) -> window mean in T.pmean
__global__ void __launch_bounds__(32 * kPredWarps)
    k_trk_predict(TrackerDev T, const double *dx, const double *dy, int64_t field_stride, int fw_l,
                  int fh_l, int level, const int32_t *n_dets) {
  extern __shared__ __align__(16) char smem[];
  const int warp = threadIdx.x >> 5;
  LeafScratch &L = reinterpret_cast<LeafScratch *>(smem)[warp];
  const int s = blockIdx.x;
  if (n_dets[s] == FT_STREAM_SKIP) return;  // the stream does not advance this step
  const int item = blockIdx.y * kPredWarps + warp;
  const int i = item >> 1, comp = item & 1;
  if (i >= T.n_active[s]) return;
  const int64_t o = (int64_t)s * T.cap + i;
  int top, bottom, left, right;
  const bool ok = box_support(T.box + 4 * o, level, fw_l, fh_l, top, bottom, left, right);
  if ((threadIdx.x & 31) == 0 && comp == 0) T.valid[o] = ok;
  if (!ok) return;
  const double *plane = (comp ? dy : dx) + s * field_stride;
  const double m = warp_window_mean(plane, fw_l, fw_l, top, bottom, left, right, L);
  if ((threadIdx.x & 31) == 0) T.pmean[2 * o + comp] = m;
}

// predict, phase 2: apply valid predictions (track.py:82-86), then build the
// candidate list (actives with a prediction, table order) -- SURVEY A16 (4)
// kbox != null: the KLT backend already produced the predicted boxes
__global__ void k_trk_apply(TrackerDev T, int level, const double *kbox, const int32_t *n_dets) {
  const int s = blockIdx.x;
  if (n_dets[s] == FT_STREAM_SKIP) return;
  const int na = T.n_active[s];
  const int64_t tb = (int64_t)s * T.cap;
  for (int i = threadIdx.x; i < na; i += blockDim.x) {
    const int64_t o = tb + i;
    if (!T.valid[o]) continue;
    if (kbox) {
#pragma unroll
      for (int c = 0; c < 4; ++c) T.box[4 * o + c] = kbox[4 * o + c];
    } else {
      apply_shift(T.box + 4 * o, T.pmean[2 * o], T.pmean[2 * o + 1], level, T.frame_w, T.frame_h,
                  T.box + 4 * o);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // order-preserving compaction of candidates
    int k = 0;
    for (int i = 0; i < na; ++i)
      if (T.valid[tb + i]) {
        T.cand[tb + k] = i;
        ++k;
      }
    T.n_cand[s] = k;
  }
}

// detections: score gate (filter_detections, order kept), gated IoU cost of
// candidates x kept detections (assoc.py:119-126)
__global__ void k_trk_cost(TrackerDev T, const ft_det *dets, const int32_t *n_dets) {
  const int s = blockIdx.x;
  const int nd_raw = n_dets[s];
  if (nd_raw < 0) return;  // coast: no detector result
  const ft_det *D = dets + (int64_t)s * T.max_dets;
  __shared__ int s_nkeep;
  if (threadIdx.x == 0) {
    int k = 0;
    for (int j = 0; j < nd_raw; ++j)
      if (D[j].score >= T.min_score) T.kept[(int64_t)s * T.max_dets + k++] = j;
    s_nkeep = k;
    T.n_kept[s] = k;
  }
  __syncthreads();
  const int nk = s_nkeep, nc = T.n_cand[s];
  const int64_t tb = (int64_t)s * T.cap;
  double *scores = T.scores + (int64_t)s * T.cap * T.max_dets;
  double *cost = T.cost + (int64_t)s * T.cap * T.max_dets;
  for (int k = threadIdx.x; k < nc * nk; k += blockDim.x) {
    const int i = k / nk, j = k % nk;
    const int ti = T.cand[tb + i];
    const ft_det &d = D[T.kept[(int64_t)s * T.max_dets + j]];
    const double db[4] = {d.x, d.y, d.w, d.h};
    const double sc = iou_box(T.box + 4 * (tb + ti), db);
    scores[k] = sc;
    cost[k] = (sc >= T.gate && T.cls[tb + ti] == d.class_id) ? 1.0 - sc : kForbiddenCost;
  }
}

__global__ void k_trk_hungarian(TrackerDev T, const int32_t *n_dets) {
  extern __shared__ __align__(16) char smem[];
  const int s = blockIdx.x;
  if (n_dets[s] < 0) return;
  const int m = T.n_cand[s], n = T.n_kept[s];
  int *row_col = T.row_col + (int64_t)s * T.cap;
  if (m == 0 || n == 0) {
    for (int i = threadIdx.x; i < m; i += 32) row_col[i] = -1;
    return;
  }
  const double *C = T.cost + (int64_t)s * T.cap * T.max_dets;
  lsap_warp(C, m, n, m > n, smem, row_col);
  // drop pairs that landed on a forbidden cell (assoc.py:104-105)
  for (int i = threadIdx.x; i < m; i += 32) {
    const int j = row_col[i];
    if (j >= 0 && !(C[(int64_t)i * n + j] < kForbiddenCost)) row_col[i] = -1;
  }
}

// lifecycle update (track.py:90-139) over the active table; Lost tracks are
// emitted to the per-stream lost list and compacted out (they never re-enter
// matching and only their ids matter, via next_id).
__global__ void k_trk_update(TrackerDev T, const ft_det *dets, const int32_t *n_dets,
                             const int32_t *frames) {
  const int s = blockIdx.x;
  if (threadIdx.x != 0) return;
  const int frame = frames[s];
  const int nd_raw = n_dets[s];
  const int64_t tb = (int64_t)s * T.cap;
  T.n_lost[s] = 0;
  if (nd_raw < 0) return;  // coast (-1) or not advancing (FT_STREAM_SKIP)
  const ft_det *D = dets + (int64_t)s * T.max_dets;
  const int32_t *kept = T.kept + (int64_t)s * T.max_dets;
  const int nk = T.n_kept[s], nc = T.n_cand[s], na = T.n_active[s];
  const int *row_col = T.row_col + tb;
  unsigned char *det_used = T.det_used + (int64_t)s * T.max_dets;
  int *match_of = T.match_of + tb;  // active index -> kept det index or -1
  for (int i = 0; i < na; ++i) match_of[i] = -1;
  for (int j = 0; j < nk; ++j) det_used[j] = 0;
  for (int ci = 0; ci < nc; ++ci) {
    const int j = row_col[ci];
    if (j >= 0) {
      match_of[T.cand[tb + ci]] = j;
      det_used[j] = 1;
    }
  }
  ft_track *lost = T.lost + (int64_t)s * T.cap;
  int nl = 0, w = 0;
  const double bl = T.blend;
  for (int i = 0; i < na; ++i) {
    const int64_t o = tb + i;
    const int j = match_of[i];
    if (j >= 0) {
      const ft_det &d = D[kept[j]];
      double *b = T.box + 4 * o;
      if (bl >= 1.0) {
        b[0] = d.x; b[1] = d.y; b[2] = d.w; b[3] = d.h;
      } else {
        const double dv[4] = {d.x, d.y, d.w, d.h};
        for (int c = 0; c < 4; ++c) b[c] = bl * dv[c] + (1.0 - bl) * b[c];
      }
      T.score[o] = d.score;
      T.last_seen[o] = frame;
      if (w != i) copy_track(T, tb + w, o);
      ++w;
    } else {
      ft_track &L = lost[nl++];
      L.id = T.id[o];
      L.class_id = T.cls[o];
      L.label_ref = T.label[o];
      L.x = T.box[4 * o];
      L.y = T.box[4 * o + 1];
      L.w = T.box[4 * o + 2];
      L.h = T.box[4 * o + 3];
      L.score = T.score[o];
      L.state = 0;
      L.born_at = T.born[o];
      L.last_seen = T.last_seen[o];
      L.lost_at = frame;
    }
  }
  // spawn: unmatched kept detections in index order, fresh increasing ids
  int64_t nid = T.next_id[s];
  for (int j = 0; j < nk; ++j) {
    if (det_used[j]) continue;
    if (w >= T.cap) {
      T.overflow[s] = 1;
      break;
    }
    const ft_det &d = D[kept[j]];
    const int64_t o = tb + w;
    T.id[o] = nid++;
    T.cls[o] = d.class_id;
    T.label[o] = d.label_ref;
    T.box[4 * o] = d.x;
    T.box[4 * o + 1] = d.y;
    T.box[4 * o + 2] = d.w;
    T.box[4 * o + 3] = d.h;
    T.score[o] = d.score;
    T.born[o] = frame;
    T.last_seen[o] = frame;
    ++w;
  }
  T.next_id[s] = nid;
  T.n_active[s] = w;
  T.n_lost[s] = nl;
}

// pack [actives..., newly lost...] per stream into ft_track records
__global__ void k_trk_pack(TrackerDev T, ft_track *out, int32_t *n_out) {
  const int s = blockIdx.x;
  const int na = T.n_active[s], nl = T.n_lost[s];
  const int64_t tb = (int64_t)s * T.cap;
  ft_track *o = out + (int64_t)s * 2 * T.cap;
  for (int i = threadIdx.x; i < na; i += blockDim.x) {
    const int64_t k = tb + i;
    ft_track r;
    r.id = T.id[k];
    r.class_id = T.cls[k];
    r.label_ref = T.label[k];
    r.x = T.box[4 * k];
    r.y = T.box[4 * k + 1];
    r.w = T.box[4 * k + 2];
    r.h = T.box[4 * k + 3];
    r.score = T.score[k];
    r.state = 1;
    r.born_at = T.born[k];
    r.last_seen = T.last_seen[k];
    r.lost_at = -1;
    o[i] = r;
  }
  const ft_track *L = T.lost + tb;
  for (int i = threadIdx.x; i < nl; i += blockDim.x) o[na + i] = L[i];
  if (threadIdx.x == 0) n_out[s] = na + nl;
}

// Streams that do not advance this step keep their previous pyramid: the
// step built into the other ping-pong buffer, so copy theirs across.
__global__ void k_keep_prev(double *cur, const double *prev, int64_t per_stream,
                            const int32_t *n_dets) {
  const int s = blockIdx.y;
  if (n_dets[s] != FT_STREAM_SKIP) return;
  const int64_t o = (int64_t)s * per_stream;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < per_stream;
       i += (int64_t)gridDim.x * blockDim.x)
    cur[o + i] = prev[o + i];
}

__global__ void k_fill_i32(int32_t *dst, int n, int32_t v) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) dst[i] = v;
}

int launch_fill_i32(int32_t *dst, int n, int32_t v, cudaStream_t s) {
  k_fill_i32<<<(n + 255) / 256, 256, 0, s>>>(dst, n, v);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

int launch_keep_prev(double *cur, const double *prev, int64_t per_stream, const int32_t *n_dets,
                     int n_streams, cudaStream_t s) {
  const int bx = (int)std::min<int64_t>((per_stream + 255) / 256, 64);
  k_keep_prev<<<dim3(bx, n_streams), 256, 0, s>>>(cur, prev, per_stream, n_dets);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

int launch_tracker_track(TrackerDev &T, const double *dx, const double *dy, int64_t fstride,
                         int fw_l, int fh_l, int level, const ft_det *d_dets,
                         const int32_t *d_ndets, const int32_t *d_frames, bool has_prev,
                         ft_track *d_out, int32_t *d_nout, cudaStream_t s, const double *kbox) {
  const int S = T.n_streams;
  if (has_prev && kbox) {  // KLT backend: boxes + valid already predicted
    k_trk_apply<<<S, 128, 0, s>>>(T, level, kbox, d_ndets);
    count_launch();
  } else if (has_prev) {
    const dim3 pg(S, (2 * T.cap + kPredWarps - 1) / kPredWarps);
    k_trk_predict<<<pg, 32 * kPredWarps, kPredWarps * sizeof(LeafScratch), s>>>(
        T, dx, dy, fstride, fw_l, fh_l, level, d_ndets);
    k_trk_apply<<<S, 128, 0, s>>>(T, level, nullptr, d_ndets);
    count_launch(2);
  } else {
    // first frame: nothing to predict, every kept detection spawns
    FT_CUDA_TRY(cudaMemsetAsync(T.n_cand, 0, S * sizeof(int32_t), s));
  }
  // streams with n_dets < 0 (no detector result) coast: these kernels exit
  k_trk_cost<<<S, 256, 0, s>>>(T, d_dets, d_ndets);
  count_launch();
  const size_t sm = hungarian_smem(T.cap, T.max_dets);
  k_trk_hungarian<<<S, 32, sm, s>>>(T, d_ndets);
  count_launch();
  k_trk_update<<<S, 32, 0, s>>>(T, d_dets, d_ndets, d_frames);
  count_launch();
  k_trk_pack<<<S, 128, 0, s>>>(T, d_out, d_nout);
  count_launch();
  FT_CUDA_TRY(cudaGetLastError());
  return FT_OK;
}

int tracker_kernel_setup(const TrackerDev &T) {
  const size_t sm = hungarian_smem(T.cap, T.max_dets);
  if (sm > 200 * 1024) return fail(FT_EINVAL, "max_tracks/max_dets too large for one CTA");
  FT_CUDA_TRY(cudaFuncSetAttribute(k_trk_hungarian, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)sm));
  FT_CUDA_TRY(cudaFuncSetAttribute(k_trk_predict, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)(kPredWarps * sizeof(LeafScratch))));
  return FT_OK;
}

}  // namespace ft

// Device-side track tables for the multi-stream tracker (SoA, one block of
// `cap` rows per stream).  Only ACTIVE tracks are kept, in scene-list order
// (which equals id order: the reference appends spawns and never removes,
// track.py:131-138); tracks that turn Lost are emitted once and dropped --
// they are inert tombstones in the reference (track.py:128-129) whose only
// remaining influence, the next id, is kept in next_id.
#pragma once

#include "ft_internal.cuh"

namespace ft {

constexpr double kForbiddenCost = 1e6;  // assoc.py:18

struct TrackerDev {
  int n_streams, cap, max_dets, frame_w, frame_h;
  double gate, min_score, blend;
  int64_t *id, *next_id;
  int32_t *cls, *label, *born, *last_seen;
  double *box, *score, *pmean;  // pmean: [cap][2] window means of predict
  int32_t *n_active, *n_cand, *cand, *n_kept, *kept, *row_col, *match_of, *n_lost, *overflow;
  unsigned char *valid, *det_used;
  double *scores, *cost;
  ft_track *lost;
};

__device__ __forceinline__ void copy_track(TrackerDev &T, int64_t d, int64_t s) {
  T.id[d] = T.id[s];
  T.cls[d] = T.cls[s];
  T.label[d] = T.label[s];
  T.born[d] = T.born[s];
  T.last_seen[d] = T.last_seen[s];
  T.score[d] = T.score[s];
#pragma unroll
  for (int c = 0; c < 4; ++c) T.box[4 * d + c] = T.box[4 * s + c];
}

int launch_tracker_track(TrackerDev &T, const double *dx, const double *dy, int64_t fstride,
                         int fw_l, int fh_l, int level, const ft_det *d_dets,
                         const int32_t *d_ndets, const int32_t *d_frames, bool has_prev,
                         ft_track *d_out, int32_t *d_nout, cudaStream_t s,
                         const double *kbox = nullptr);
int tracker_kernel_setup(const TrackerDev &T);
// dst[0..n) = v
int launch_fill_i32(int32_t *dst, int n, int32_t v, cudaStream_t s);
// per stream s with n_dets[s] == FT_STREAM_SKIP: cur[s] = prev[s]
int launch_keep_prev(double *cur, const double *prev, int64_t per_stream, const int32_t *n_dets,
                     int n_streams, cudaStream_t s);

}  // namespace ft

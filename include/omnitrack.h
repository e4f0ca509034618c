/*
 * omnitrack.h -- C ABI of libomnitrack.so, the B200-native (sm_100a) OmniTrack
 * tracking hot path: pyramid -> ROF structure-texture -> TV-L1 flow ->
 * mean-box predict -> IoU/Hungarian match -> update.
 *
 * The reference (flowtrack, Python/numpy) has no FFI; its "operator API" is a
 * set of pure module functions.  Each entry point below replaces one of them
 * (reference path:line relative to /root/reference/pkg/src/flowtrack/), and
 * the ctypes binding in paper_1910_06017_b200/_lib.py re-exports the
 * reference signatures on top (INTEGRATION.md shows the binding).
 *
 * Conventions
 *  - Return value: FT_OK (0) or a negative FT_E* code; ft_last_error() gives
 *    the message of the last failure on the calling thread.  The Python layer
 *    maps FT_EINVAL -> ValueError and FT_ERANGE -> IndexError with the
 *    reference's messages.
 *  - Image planes are DEVICE pointers to row-major float64 (pitch == width)
 *    unless the name says u8.  Small record arrays (boxes, class ids, cost
 *    matrices, pairs) are HOST pointers; the library stages them.
 *  - Inputs are never written (reference ownership rule: inputs immutable).
 *  - One ft_ctx per (GPU, host thread); a context is bound to one CUDA stream
 *    (ft_ctx_set_stream) and is not reentrant; distinct contexts may run
 *    concurrently.  Calls are asynchronous on that stream unless they return
 *    host results (predict/match/hungarian/tracker_step synchronize).
 */
#ifndef OMNITRACK_H
#define OMNITRACK_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FT_OK 0
#define FT_EINVAL (-1) /* ValueError: sizes, parameters, degenerate pyramid, lost predict */
#define FT_ERANGE (-2) /* IndexError: assignment index out of range */
#define FT_ECUDA (-3)  /* CUDA runtime failure */
#define FT_ENOMEM (-4) /* device / pinned allocation failed */
#define FT_ECAP (-5)   /* tracker capacity (max_tracks / max_dets) exceeded */

/* n_dets value of a stream that does not advance in a tracker step (no
 * frame this step): its tracks, ids and previous frame stay as they are */
#define FT_STREAM_SKIP (-2)

/* optflow.py:36-66 FlowParams; pyramid_scales <= 0 means auto (optflow.py:96) */
typedef struct ft_flow_params {
  double data_weight;   /* lambda, default 0.15 */
  double huber_epsilon; /* default 0.01 */
  double time_step;     /* tau, default 0.25 */
  int32_t warps_per_level;     /* default 5 */
  int32_t iterations_per_warp; /* default 50 */
  int32_t pyramid_scales;      /* <= 0: auto_scales */
  int32_t _pad;
} ft_flow_params;

typedef struct ft_ctx ft_ctx;
typedef struct ft_tracker ft_tracker;

const char *ft_last_error(void);
int ft_version(void);
int ft_device_count(int *count);

/* ---- context ------------------------------------------------------------ */
int ft_ctx_create(int device, ft_ctx **out);
int ft_ctx_destroy(ft_ctx *ctx);
/* bind to an existing cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream);
 * taken verbatim like the CUDA runtime: NULL is the legacy default stream.
 * A new context starts on its own non-blocking stream.  Trackers run on
 * their own stream, joined to this one by events at every call. */
int ft_ctx_set_stream(ft_ctx *ctx, void *cuda_stream);
int ft_ctx_synchronize(ft_ctx *ctx);

/* ---- host scalar policy ------------------------------------------------- */
int ft_select_level(int width, int height, int *level);  /* imaging.py:98-106 */
int ft_auto_scales(int width, int height, int *scales);  /* optflow.py:96-104 */

/* ---- imaging (imaging.py) ----------------------------------------------- */
/* Frame.from_gray8: u8/255 (imaging.py:52-56) */
int ft_gray8_to_unit(ft_ctx *ctx, const uint8_t *d_src, int w, int h, double *d_dst);
/* Frame / MotionField validation of device planes (imaging.py:33-44,
 * optflow.py:85-86): *h_status = 0, or bit 0 when a value is non-finite, bit
 * 1 when a finite value lies outside [lo, hi].  Synchronizes. */
int ft_check_plane(ft_ctx *ctx, const double *d_plane, int64_t n, double lo, double hi,
                   int32_t *h_status);
/* build_pyramid (imaging.py:75-95): levels written back to back into
 * d_levels (level 0 copied), sizes floor-halved; FT_EINVAL below 2x2 */
int ft_build_pyramid(ft_ctx *ctx, const double *d_frame, int w, int h, int num_levels,
                     double *d_levels);
/* structure_texture + rof_denoise (imaging.py:109-144) */
int ft_structure_texture(ft_ctx *ctx, const double *d_in, int w, int h, double smoothing_weight,
                         double blend, int iterations, double *d_out);

/* rof_denoise (imaging.py:109-125): the TV-smoothed structure image */
int ft_rof_denoise(ft_ctx *ctx, const double *d_in, int w, int h, double weight, int iterations,
                   double step, double *d_out);

/* ---- optical flow (optflow.py) ------------------------------------------ */
/* compute_flow (optflow.py:217-253): dense TV-L1 from prev to curr */
int ft_compute_flow(ft_ctx *ctx, const double *d_prev, const double *d_curr, int w, int h,
                    const ft_flow_params *params, double *d_dx, double *d_dy);

/* per-pixel terms of flow_energy (optflow.py:121-144): data = |I1(x+u)-I0|
 * on x255 intensities, s1/s2 = huber(|forward_gradient(u_k)|); the
 * reference's scalar is lambda*sum(data) + sum(s1) + sum(s2) in numpy order */
int ft_flow_energy_terms(ft_ctx *ctx, const double *d_prev, const double *d_curr,
                         const double *d_dx, const double *d_dy, int w, int h,
                         double huber_epsilon, double *d_data, double *d_s1, double *d_s2);

/* compute_flow with energy_trace (optflow.py:212-213): after every warp of
 * the finest scale the flow_energy terms are written to d_energy_terms
 * (warps_per_level x 3 x w*h doubles: data, s1, s2 per warp) */
int ft_compute_flow_traced(ft_ctx *ctx, const double *d_prev, const double *d_curr, int w, int h,
                           const ft_flow_params *params, double *d_dx, double *d_dy,
                           double *d_energy_terms);

/* ---- tracking (track.py / assoc.py) ------------------------------------- */
/* predict (track.py:56-87).  h_boxes: n x (x,y,w,h); field (d_dx,d_dy) is
 * field_w x field_h at pyramid `level`; h_out n x 4, h_valid[i]=0 for None */
int ft_predict(ft_ctx *ctx, const double *h_boxes, int n, const double *d_dx, const double *d_dy,
               int field_w, int field_h, int level, int frame_w, int frame_h, double *h_out,
               uint8_t *h_valid);
/* KLT / MedianFlow box prediction (oracle/klt_oracle.py
 * defines it -- the reference has no KLT): prev/curr are the w x h
 * processing-level frames of pyramid `level`; grid x grid points per box,
 * pyramidal LK prev->curr and back, forward-backward median filter, median
 * shift and pairwise scale ratio.  h_valid[i]=0 when no point survives. */
int ft_klt_predict(ft_ctx *ctx, const double *d_prev, const double *d_curr, int w, int h,
                   int level, int frame_w, int frame_h, int grid, const double *h_boxes, int n,
                   double *h_out, uint8_t *h_valid);
/* iou (assoc.py:30-41) matrix: h_out[i*n+j] = iou(a_i, b_j) */
int ft_iou_matrix(ft_ctx *ctx, const double *h_a, int m, const double *h_b, int n, double *h_out);
/* hungarian (assoc.py:84-106): h_cost m x n; pairs sorted by row;
 * has_forbidden drops pairs with cost >= forbidden */
int ft_hungarian(ft_ctx *ctx, const double *h_cost, int m, int n, int has_forbidden,
                 double forbidden, int32_t *h_pairs /* 2*min(m,n) */, int *n_pairs);
/* match (assoc.py:109-135): gated class-constrained IoU assignment */
int ft_match(ft_ctx *ctx, const double *h_tboxes, const int32_t *h_tcls, int m,
             const double *h_dboxes, const int32_t *h_dcls, int n, double gate,
             int32_t *h_pairs /* 2*min(m,n) */, double *h_ious, int *n_pairs);

/* update (track.py:90-139) over a full scene list of n objects (ids, state
 * 1=active/0=lost, boxes n x 4) with assignment pairs (scene idx, det idx)
 * and nd detection boxes.  Output rows (at most n+nd, count in n_out):
 * h_src >= 0 is an existing object with h_flag 0 keep / 1 matched / 2 turned
 * lost and its new box; h_src = -(j+1) spawns detection j with id h_id.
 * FT_ERANGE for out-of-range indices, FT_EINVAL for a lost object in a pair. */
int ft_update(ft_ctx *ctx, const int64_t *h_ids, const int32_t *h_state, const double *h_boxes,
              int n, const int32_t *h_pairs, int n_pairs, const double *h_dboxes, int nd,
              double blend, int32_t *h_src, double *h_box, int32_t *h_flag, int64_t *h_id,
              int *n_out);

/* ---- tracker fast path (SPEC.md:408-416 step) ------------ */
typedef struct ft_det {
  int32_t class_id;
  int32_t label_ref; /* opaque host label handle, copied to spawned tracks */
  double score;
  double x, y, w, h;
} ft_det;

typedef struct ft_track {
  int64_t id;
  int32_t class_id;
  int32_t label_ref;
  double x, y, w, h;
  double score;
  int32_t state; /* 1 = active, 0 = lost */
  int32_t born_at;
  int32_t last_seen;
  int32_t lost_at; /* -1 while active */
} ft_track;

typedef struct ft_tracker_config {
  int32_t width, height;  /* frame size (u8 luma) */
  int32_t n_streams;      /* independent streams advanced in lockstep */
  int32_t max_tracks;     /* active tracks per stream */
  int32_t max_dets;       /* detections per stream-frame */
  int32_t rof_iterations; /* 40 */
  double gate;            /* 0.3  (assoc.py:109) */
  double min_score;       /* 0.5 */
  double detection_blend; /* 1.0  (track.py:91) */
  double rof_weight;      /* 12.0 (imaging.py:128) */
  double rof_blend;       /* 0.05 */
  ft_flow_params flow;
  int32_t motion;   /* FT_MOTION_TVL1 (reference path) or FT_MOTION_KLT */
  int32_t klt_grid; /* KLT points per box side (1..11), default 10 */
  /* 1: device prefetch (TV-L1 only): the graph
   * of the step submitted with frame t preprocesses frame t while the flow,
   * predict, match and update of frame t-1 run concurrently on a second
   * stream; ft_tracker_wait returns frame t-1's records (none after the
   * first frame) and ft_tracker_flush tracks the last frame.  Results are
   * identical to the sequential mode. */
  int32_t prefetch;
  int32_t _pad;
} ft_tracker_config;

#define FT_MOTION_TVL1 0
#define FT_MOTION_KLT 1

int ft_tracker_create(ft_ctx *ctx, const ft_tracker_config *cfg, ft_tracker **out);
int ft_tracker_destroy(ft_tracker *trk);
/* One frame for every stream.  h_luma: n_streams x H x W u8 (host);
 * h_dets: n_streams x max_dets; h_n_dets[s] = -1 when stream s has no
 * detector result this frame (coast), FT_STREAM_SKIP when stream s has no
 * frame this step (it does not advance; its records are its unchanged
 * active tracks).  Outputs, per stream s, the active
 * tracks followed by tracks that became lost this frame, into
 * h_out[s*(2*max_tracks) ...], count in h_n_out[s]. */
int ft_tracker_step(ft_tracker *trk, const uint8_t *h_luma, int frame_index, const ft_det *h_dets,
                    const int32_t *h_n_dets, ft_track *h_out, int32_t *h_n_out);
/* Pinned host staging buffers of the tracker (n_streams x H x W luma,
 * n_streams x max_dets detections, n_streams detection counts).  Writing the
 * inputs there and passing the same pointers to ft_tracker_step skips one
 * host copy. */
int ft_tracker_input_buffers(ft_tracker *trk, uint8_t **h_luma, ft_det **h_dets,
                             int32_t **h_n_dets);
/* Asynchronous form of ft_tracker_step (the paper's
 * prefetch / async-detection overlap).  Two pinned staging slots: stage
 * frame t+1 into slot (t+1)&1 (ft_tracker_slot_buffers, or pass host
 * pointers) and submit it while frame t is still running; wait returns a
 * slot's records.  Submissions execute in order, so results are identical to
 * the synchronous call; a submission's H2D copy runs on the tracker's copy
 * stream while the previous step computes.  NULL luma/dets/n_dets = already
 * staged in the slot. */
int ft_tracker_slot_buffers(ft_tracker *trk, int slot, uint8_t **h_luma, ft_det **h_dets,
                            int32_t **h_n_dets);
int ft_tracker_submit(ft_tracker *trk, int slot, int frame_index, const uint8_t *h_luma,
                      const ft_det *h_dets, const int32_t *h_n_dets);
/* Per-stream staging (SURVEY.md 8(b) ft_step(ctx, stream_id, luma, w, h,
 * pitch, frame_index, dets, n_dets, ...)): copy stream `stream`'s W x H luma
 * from rows `pitch` bytes apart, its detections (n_dets = -1 coast,
 * FT_STREAM_SKIP no frame: luma may be NULL) and its frame index into the
 * slot's pinned buffers.  ft_tracker_submit_staged then runs one step of
 * every stream as staged (each with its own frame index). */
int ft_tracker_stage(ft_tracker *trk, int slot, int stream, const uint8_t *h_luma, int pitch,
                     int frame_index, const ft_det *h_dets, int n_dets);
int ft_tracker_submit_staged(ft_tracker *trk, int slot);
/* Prefetch trackers: a step with no new frame that tracks the pending last
 * frame (its records come back from ft_tracker_wait on `slot`). */
int ft_tracker_flush(ft_tracker *trk, int slot);
/* One step of a single stream (all others skip), synchronous: stream
 * `stream`'s records (active tracks then the ones lost this step) into
 * h_out (2 x max_tracks), count in *h_n_out. */
int ft_tracker_step_stream(ft_tracker *trk, int stream, const uint8_t *h_luma, int pitch,
                           int frame_index, const ft_det *h_dets, int n_dets, ft_track *h_out,
                           int32_t *h_n_out);
int ft_tracker_wait(ft_tracker *trk, int slot, ft_track *h_out, int32_t *h_n_out);
/* Same step with inputs already resident on the device (d_luma as above,
 * d_dets/d_n_dets device arrays); no host copies, no synchronisation. */
int ft_tracker_step_device(ft_tracker *trk, const uint8_t *d_luma, int frame_index,
                           const ft_det *d_dets, const int32_t *d_n_dets);
/* Copy the device track tables of the last step to the host (synchronizes). */
int ft_tracker_read(ft_tracker *trk, ft_track *h_out, int32_t *h_n_out);
/* Device motion field of stream s from the last step (processing level). */
int ft_tracker_field(ft_tracker *trk, int stream, const double **d_dx, const double **d_dy,
                     int *w, int *h);
/* Host copy of stream s's motion field from the last step (synchronizes). */
int ft_tracker_read_field(ft_tracker *trk, int stream, double *h_dx, double *h_dy);
/* Time the dominant kernel (finest-level primal-dual tile kernel) alone:
 * `reps` launches on the tracker's stream between CUDA events, over the state
 * the last step left.  bytes_per_launch = SURVEY 8(d) algorithmic bytes of a
 * launch (152 B per pixel-iteration x the pixel-iterations it performs);
 * iters_per_launch = PD iterations it fuses. */
/* Live timing of the dominant kernel inside the most recent step: CUDA
 * events recorded (as graph nodes) around every finest-level primal-dual
 * launch sequence of the step.  ms = summed device time of those launches,
 * launches = their count, pixel_iters = pixel-iterations they performed over
 * all streams (x 152 B = SURVEY 8(d) algorithmic bytes).  Synchronizes. */
int ft_tracker_pd_span(ft_tracker *trk, double *ms, int *launches, double *pixel_iters);
int ft_tracker_profile_pd(ft_tracker *trk, int reps, double *ms_per_launch,
                          double *bytes_per_launch, int *iters_per_launch);
/* Kernel launches issued by the last step (for the bench's gpu_launches). */
int ft_tracker_launches(ft_tracker *trk, int64_t *count);
/* Per-phase device times of a step (FrameResult carries
 * per-phase timing in ms).  slot 0/1: the step last submitted in that slot
 * (waits for it); slot -1: the most recent step.  Fills up to `max` phases
 * in execution order: ms[i] and names[i] (static strings: "h2d" (prefetch
 * trackers; the others copy a submission's inputs on a copy stream while the
 * previous step runs), "ingest+pyramid", "structure_texture", "flow
 * pyramid", "flow level k", "predict+match+update", "d2h", ...); *n = phases
 * written. */
int ft_tracker_phase_times(ft_tracker *trk, int slot, double *ms, const char **names, int max,
                           int *n);
/* Reset all streams (drop tracks and cached previous frames).  Submitted
 * steps still in flight are completed and their records dropped: both
 * staging slots are free afterwards. */
int ft_tracker_reset(ft_tracker *trk);

#ifdef __cplusplus
}
#endif
#endif

// Whole-level primal-dual solver (k_pd_level.cu): one cooperative launch runs
// all iterations of one TV-L1 warp for a whole pyramid level of `nb` streams.
#pragma once

#include "ft_internal.cuh"

namespace ft {

constexpr int kLvTW = 64, kLvTH = 24;  // tile of one CTA (two CTAs per SM)

struct LevelPDArgs {
  const double *u1, *u2;      // u at the start of the warp (after warp setup)
  double *out1, *out2;        // u after the warp's iterations
  const double *gx, *gy, *r0; // warp constants (optflow.py:158-167)
  int w, h;
  int64_t cap;                // elements between consecutive streams' planes
  int iters;
  double tau, lam, sigma, shrink;
  void *edges;                // per-tile exchange records (level_pd_edges_bytes)
  unsigned *flags;            // [tiles][2] half-step counters
  unsigned *err;              // set when a neighbour wait times out
};

// CTAs one cooperative launch can hold on `device` (0: no cooperative launch)
int level_pd_capacity(int device, int *max_ctas);
size_t level_pd_edges_bytes(int tiles);
inline int level_pd_tiles(int w, int h) {
  return ((w + kLvTW - 1) / kLvTW) * ((h + kLvTH - 1) / kLvTH);
}
int launch_level_pd(const LevelPDArgs &a, int nb, int pow2, cudaStream_t s);

}  // namespace ft

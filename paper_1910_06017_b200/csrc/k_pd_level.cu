// Whole-level primal-dual solver: all iterations of one TV-L1 warp
// (optflow.py:178-208) for a whole pyramid level in ONE launch, with the
// state resident on chip and no halo recomputation.
//
// Why: the temporally blocked tile kernel (k_pd_tile, k_flow.cu) re-reads
// and re-writes the state planes every 4 iterations and recomputes a 4-pixel
// halo around every 32x32 tile (56 % useful pixels).  At SD one level is
// 414,720 pixels; its state (6 exchange doubles in shared memory, 5
// pointwise doubles in registers, 2 more in shared memory) fits the
// register files and shared memory of the 148 SMs.  So a cooperative grid
// of 64x24 tiles (two CTAs per SM) holds a whole level -- of one SD stream, or
// of several streams of a coarser level -- and runs every iteration of a
// warp on chip.  Neighbouring tiles exchange their one-pixel edges through
// L2 after every half-step: the dual step needs u-bar one column right / one
// row down, the primal step needs p one column left / one row up
// (imageops.py:32-50), so after a dual step a tile publishes its right column
// of (p11, p21) and its bottom row of (p12, p22), after a primal step its left
// column and top row of u-bar.  Flags are per tile and per half-step kind,
// monotonic within a launch (zeroed by a memset node before it), written with
// st.release.gpu after a gpu-scope fence and polled with ld.acquire.gpu; edge
// data is read with ld.global.cg (L2, never a stale L1 line).  Every CTA is
// co-resident (cooperative launch), so the waits always make progress; a
// bounded spin traps instead of hanging if that ever failed.
//
// Arithmetic: identical operations in identical order to k_pd_tile's
// pd_halfsteps_cq and to the reference, including the CTA-wide projection
// queue for the few saturated (|p| > 1) pairs.  Bit-identical results.
#include <algorithm>
#include <cmath>

#include "ft_internal.cuh"
#include "ft_pd_level.cuh"

namespace ft {

namespace {

constexpr int TW = kLvTW, TH = kLvTH;
constexpr int NT = 512, NW = NT / 32;        // 16 warps: 2 column halves x 8 row groups
constexpr int RG = NW / 2, PY = TH / RG;     // rows per thread (3)
constexpr int SP = TW + 2, SR = TH + 2, PL = SP * SR;  // planes with a 1-element apron
constexpr int NPAIR = 2 * TW * TH;           // (p1, p2) pairs per tile

static_assert(TW == 64 && PY * RG == TH, "tile geometry");

// shared memory (double2 units): B (ub1, ub2), PX (p11, p21), PY (p12, p22)
// planes [SR][SP] with a one-element apron, TI
// [TH][TW] -> (rho0, 1/|grad|^2), then the uint16 projection queue [NPAIR] and two counters
constexpr size_t kSmem = (size_t)(3 * PL + TW * TH) * 16 + (size_t)NPAIR * 2 + 16;

#ifdef FT_LV_NOSYNC
constexpr bool kNoSync = true;  // timing study only: no edge exchange (wrong results)
#else
constexpr bool kNoSync = false;
#endif

enum : unsigned { FL_R = 1, FL_D = 2, FL_L = 4, FL_LASTC = 8, FL_U = 16, FL_LASTR = 32, FL_IN = 64 };

template <bool P2>
__device__ __forceinline__ double madx(double a, double b, double c) {
  return P2 ? fma(a, b, c) : a * b + c;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// every lane polls (acquire orders its own subsequent edge loads)
__device__ __forceinline__ void wait_flag(const unsigned *f, unsigned target, unsigned *err) {
  unsigned spins = 0;
  while (ld_acquire(f) < target) {
    if (++spins > (1u << 23)) {  // ~seconds: a neighbour never arrived
      atomicExch(err, 1u);
      __trap();
    }
  }
}

// Exchange record of one tile (global): edges published after each half-step.
struct Edges {
  double2 r[TH];  // after dual: right column (p11, p21)
  double2 d[TW];  // after dual: bottom row (p12, p22)
  double2 l[TH];  // after primal: left column (ub1, ub2)
  double2 u[TW];  // after primal: top row (ub1, ub2)
};

extern __shared__ __align__(16) double2 lv_sm[];

// One pixel's dual ascent + Huber prox (optflow.py:180-185); stores the
// unprojected p in place and returns the two "needs projection" screens.
template <bool P2, bool IN>
__device__ __forceinline__ unsigned dual_px(int id, unsigned f, double sigma, double shrink) {
  double2 *const sB = lv_sm, *const sPX = lv_sm + PL, *const sPY = lv_sm + 2 * PL;
  const double2 cb = sB[id], rb = sB[id + 1], db = sB[id + SP];
  const double2 opx = sPX[id], opy = sPY[id];
  const bool R = IN || (f & FL_R), D = IN || (f & FL_D);
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
  // screening test only (not reference arithmetic): below it max(1, hypot)
  // is exactly 1 and p / 1 == p
  return (fma(p11, p11, p12 * p12) > 0.999999 ? 1u : 0u) |
         (fma(p21, p21, p22 * p22) > 0.999999 ? 2u : 0u);
}

// unit-ball projection of pair k (double index: 2*id + component) in place:
// n = max(1, hypot(.)); p /= n (optflow.py:186-191)
__device__ __forceinline__ void project(int k) {
  double *const dPX = reinterpret_cast<double *>(lv_sm + PL);
  double *const dPY = reinterpret_cast<double *>(lv_sm + 2 * PL);
  const double pa = dPX[k], pb = dPY[k];
  const double nn = np_max(1.0, glibc_hypot(pa, pb));
  dPX[k] = pa / nn;
  dPY[k] = pb / nn;
}

// One pixel's primal descent + TV-L1 shrinkage (optflow.py:194-208).
template <bool P2, bool IN>
__device__ __forceinline__ void primal_px(int id, int ti_id, unsigned f, double &u1, double &u2,
                                          double gx, double gy, double tau, double tl) {
  double2 *const sB = lv_sm, *const sPX = lv_sm + PL, *const sPY = lv_sm + 2 * PL;
  const double2 *const sTI = lv_sm + 3 * PL;
  const double2 mpx = sPX[id], mpy = sPY[id];
  const double2 lp = sPX[id - 1], up = sPY[id - SP];
  const bool L = IN || (f & FL_L), LC = !IN && (f & FL_LASTC);
  const bool U = IN || (f & FL_U), LR = !IN && (f & FL_LASTR);
  const double dx1 = L ? (LC ? -lp.x : mpx.x - lp.x) : mpx.x;
  const double dx2 = L ? (LC ? -lp.y : mpx.y - lp.y) : mpx.y;
  const double dy1 = U ? (LR ? -up.x : mpy.x - up.x) : mpy.x;
  const double dy2 = U ? (LR ? -up.y : mpy.y - up.y) : mpy.y;
  const double v1 = madx<P2>(tau, dx1 + dy1, u1);
  const double v2 = madx<P2>(tau, dx2 + dy2, u2);
  const double2 ti = sTI[ti_id];  // (rho0, 1/|grad|^2)
  // thresh = tau*lam*grad_sq (optflow.py:163, :176), recomputed: registers,
  // not fp64 issue, bound this kernel
  const double thr = tl * (gx * gx + gy * gy);
  const double rho = ti.x + gx * v1 + gy * v2;
  const bool lo_ = rho < -thr;
  const bool hi_ = rho > thr;
  double d = lo_ ? tl : (hi_ ? -tl : -rho * ti.y);
  d = (ti.y != 0.0 || lo_ || hi_) ? d : 0.0;  // ig2 != 0 <=> |grad|^2 > 1e-12
  const double n1 = v1 + d * gx;
  const double n2 = v2 + d * gy;
  sB[id] = make_double2(madx<true>(2.0, n1, -u1), madx<true>(2.0, n2, -u2));
  u1 = n1;
  u2 = n2;
}

// Iteration schedule (edges exchanged while the interior computes):
//   D1  dual of the pixels that need no neighbour u-bar (all but the right
//       column / bottom row), saturated pairs -> CTA queue
//   W1  warps 1/2 wait for the right / lower neighbour's u-bar edge of the
//       previous primal step and copy it into the apron        | bar A
//   D3  dual of the right column / bottom row (owners project their own
//       saturated pairs inline); all warps project the queue  | bar C
//   D5  warp 0 publishes the p edges (right column, bottom row)
//   P1  primal of the pixels that need no neighbour p (all but the left
//       column / top row)
//   W2  warps 1/2 wait for the left / upper neighbour's p edge  | bar D
//   P3  primal of the left column / top row                     | bar E
//   P4  warp 0 publishes the u-bar edges (left column, top row)
template <bool P2, bool IN>
__device__ __forceinline__ void level_body(const LevelPDArgs &a) {
  double2 *const sB = lv_sm, *const sPX = lv_sm + PL, *const sPY = lv_sm + 2 * PL;
  double2 *const sTI = lv_sm + 3 * PL;
  unsigned short *const qidx = reinterpret_cast<unsigned short *>(lv_sm + 3 * PL + TW * TH);
  int *const ctr = reinterpret_cast<int *>(qidx + NPAIR);

  const int W = a.w, H = a.h;
  const int bx = blockIdx.x, by = blockIdx.y, bz = blockIdx.z;
  const int ox = bx * TW, oy = by * TH;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int col = 32 * (warp & 1) + lane, rg = warp >> 1;
  const int64_t so = (int64_t)bz * a.cap;
  const int tile = (bz * gridDim.y + by) * gridDim.x + bx;
  Edges *const E = reinterpret_cast<Edges *>(a.edges);
  unsigned *const F = a.flags;  // [tile][2]: dual, primal
  const bool hasL = bx > 0, hasR = bx + 1 < (int)gridDim.x;
  const bool hasU = by > 0, hasD = by + 1 < (int)gridDim.y;
  const int tL = tile - 1, tR = tile + 1, tU = tile - gridDim.x, tD = tile + gridDim.x;
  const int id0 = (rg + 1) * SP + col + 1;  // smem index of the thread's first pixel
  constexpr int DK = RG * SP;               // index step between its pixels
  // pixel k is on the dual edge (needs the neighbours' u-bar) / primal edge
  // (needs the neighbours' p)
  auto dual_edge = [&](int k) { return col == TW - 1 || (rg == RG - 1 && k == PY - 1); };
  auto primal_edge = [&](int k) { return col == 0 || (rg == 0 && k == 0); };

  // ---- prologue: pointwise constants, u-bar = u, p = 0 (optflow.py:163-176)
  for (int k = tid; k < 3 * PL; k += NT) lv_sm[k] = make_double2(0, 0);
  if (tid < 2) ctr[tid] = 0;
  __syncthreads();
  const double tl = a.tau * a.lam;
  double u1[PY], u2[PY], gx[PY], gy[PY];
  unsigned fl = 0;  // 8 flag bits per pixel
#pragma unroll
  for (int k = 0; k < PY; ++k) {
    const int lr = rg + RG * k, gc = ox + col, gr = oy + lr;
    const bool in = IN || (gc < W && gr < H);
    const int64_t o = so + (int64_t)gr * W + gc;
    double vu1 = 0, vu2 = 0, vgx = 0, vgy = 0, vr0 = 0;
    if (in) {
      vu1 = a.u1[o];
      vu2 = a.u2[o];
      vgx = a.gx[o];
      vgy = a.gy[o];
      vr0 = a.r0[o];
    }
    u1[k] = vu1;
    u2[k] = vu2;
    gx[k] = vgx;
    gy[k] = vgy;
    const double g2 = vgx * vgx + vgy * vgy;  // optflow.py:163-165
    const bool ok = g2 > 1e-12;
    sTI[lr * TW + col] = make_double2(vr0, ok ? 1.0 / (g2 > 1e-12 ? g2 : 1e-12) : 0.0);
    const unsigned f = (gc < W - 1 ? FL_R : 0u) | (gr < H - 1 ? FL_D : 0u) | (gc > 0 ? FL_L : 0u) |
                       (gc == W - 1 ? FL_LASTC : 0u) | (gr > 0 ? FL_U : 0u) |
                       (gr == H - 1 ? FL_LASTR : 0u) | (in ? FL_IN : 0u);
    fl |= f << (8 * k);
    sB[id0 + k * DK] = make_double2(vu1, vu2);
  }
  // u-bar apron right / below = the neighbours' u (read by the first dual step)
  if (tid < TH) {
    const int gc = ox + TW, gr = oy + tid;
    if (gc < W && gr < H) {
      const int64_t o = so + (int64_t)gr * W + gc;
      sB[(tid + 1) * SP + TW + 1] = make_double2(a.u1[o], a.u2[o]);
    }
  } else if (tid >= 64 && tid < 64 + TW) {
    const int c = tid - 64, gc = ox + c, gr = oy + TH;
    if (gc < W && gr < H) {
      const int64_t o = so + (int64_t)gr * W + gc;
      sB[(TH + 1) * SP + c + 1] = make_double2(a.u1[o], a.u2[o]);
    }
  }
  __syncthreads();

  const double tau = a.tau, sigma = a.sigma, shrink = a.shrink;
  const unsigned lt_mask = (1u << lane) - 1u;
  for (int it = 0; it < a.iters; ++it) {
    // ---- dual ascent + Huber prox, saturated pairs -> CTA queue
    unsigned need = 0;
#pragma unroll
    for (int k = 0; k < PY; ++k) {
      const unsigned f = fl >> (8 * k);
      if (IN || (f & FL_IN)) need |= dual_px<P2, IN>(id0 + k * DK, f, sigma, shrink) << (2 * k);
    }
    {
      unsigned m[2 * PY];
      int total = 0;
#pragma unroll
      for (int j = 0; j < 2 * PY; ++j) {
        m[j] = __ballot_sync(0xffffffffu, (need >> j) & 1u);
        total += __popc(m[j]);
      }
      if (total) {  // warp-uniform
        int wbase = 0;
        if (lane == 0) wbase = atomicAdd(&ctr[it & 1], total);
        int off = __shfl_sync(0xffffffffu, wbase, 0);
#pragma unroll
        for (int j = 0; j < 2 * PY; ++j) {
          if ((need >> j) & 1u)
            qidx[off + __popc(m[j] & lt_mask)] = (unsigned short)(2 * (id0 + (j >> 1) * DK) + (j & 1));
          off += __popc(m[j]);
        }
      }
    }
    __syncthreads();
    {  // unit-ball projection of the queued pairs
      const int n = ctr[it & 1];
      if (tid == 0) ctr[(it + 1) & 1] = 0;
      for (int e = tid; e < n; e += NT) project(qidx[e]);
    }
    __syncthreads();
    // ---- p edges: publish right column / bottom row, receive left / upper
    if (!kNoSync) {
      if (warp == 0) {
        if (hasR && lane < TH) E[tile].r[lane] = sPX[(lane + 1) * SP + TW];
        if (hasD) {
          E[tile].d[lane] = sPY[TH * SP + lane + 1];
          E[tile].d[lane + 32] = sPY[TH * SP + lane + 33];
        }
        __syncwarp();
        if (lane == 0) st_release(&F[2 * tile], it + 1);
      } else if (warp == 1 && hasL) {
        wait_flag(&F[2 * tL], it + 1, a.err);
        if (lane < TH) sPX[(lane + 1) * SP] = __ldcg(&E[tL].r[lane]);
      } else if (warp == 2 && hasU) {
        wait_flag(&F[2 * tU], it + 1, a.err);
        sPY[lane + 1] = __ldcg(&E[tU].d[lane]);
        sPY[lane + 33] = __ldcg(&E[tU].d[lane + 32]);
      }
      __syncthreads();
    }
    // ---- primal descent + TV-L1 shrinkage
#pragma unroll
    for (int k = 0; k < PY; ++k) {
      const unsigned f = fl >> (8 * k);
      if (IN || (f & FL_IN))
        primal_px<P2, IN>(id0 + k * DK, (rg + RG * k) * TW + col, f, u1[k], u2[k], gx[k], gy[k],
                          tau, tl);
    }
    if (it + 1 == a.iters) break;  // the last u-bar is not read
    __syncthreads();
    // ---- u-bar edges: publish left column / top row, receive right / lower
    if (!kNoSync) {
      if (warp == 0) {
        if (hasL && lane < TH) E[tile].l[lane] = sB[(lane + 1) * SP + 1];
        if (hasU) {
          E[tile].u[lane] = sB[SP + lane + 1];
          E[tile].u[lane + 32] = sB[SP + lane + 33];
        }
        __syncwarp();
        if (lane == 0) st_release(&F[2 * tile + 1], it + 1);
      } else if (warp == 1 && hasR) {
        wait_flag(&F[2 * tR + 1], it + 1, a.err);
        if (lane < TH) sB[(lane + 1) * SP + TW + 1] = __ldcg(&E[tR].l[lane]);
      } else if (warp == 2 && hasD) {
        wait_flag(&F[2 * tD + 1], it + 1, a.err);
        sB[(TH + 1) * SP + lane + 1] = __ldcg(&E[tD].u[lane]);
        sB[(TH + 1) * SP + lane + 33] = __ldcg(&E[tD].u[lane + 32]);
      }
      __syncthreads();
    }
  }
  // ---- epilogue: u of the warp's last iteration
#pragma unroll
  for (int k = 0; k < PY; ++k) {
    const int gc = ox + col, gr = oy + rg + RG * k;
    if (!IN && !((fl >> (8 * k)) & FL_IN)) continue;
    const int64_t o = so + (int64_t)gr * W + gc;
    a.out1[o] = u1[k];
    a.out2[o] = u2[k];
  }
}

template <bool P2>
__global__ void __launch_bounds__(NT, 2) k_pd_level(const LevelPDArgs a) {
  const int ox = blockIdx.x * TW, oy = blockIdx.y * TH;
  if (ox >= 1 && oy >= 1 && ox + TW <= a.w - 1 && oy + TH <= a.h - 1)
    level_body<P2, true>(a);
  else
    level_body<P2, false>(a);
}

}  // namespace

size_t level_pd_edges_bytes(int tiles) { return (size_t)tiles * sizeof(Edges); }

int level_pd_capacity(int device, int *max_ctas) {
  int sms = 0, per_sm = 0, coop = 0;
  FT_CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
  FT_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  FT_CUDA_TRY(cudaFuncSetAttribute(k_pd_level<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kSmem));
  FT_CUDA_TRY(cudaFuncSetAttribute(k_pd_level<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kSmem));
  FT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pd_level<true>, NT, kSmem));
  int per_sm2 = 0;
  FT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm2, k_pd_level<false>, NT, kSmem));
  *max_ctas = coop ? sms * std::min(per_sm, per_sm2) : 0;
  return FT_OK;
}

int launch_level_pd(const LevelPDArgs &a, int nb, int pow2, cudaStream_t s) {
  const int tx = (a.w + TW - 1) / TW, ty = (a.h + TH - 1) / TH;
  FT_CUDA_TRY(cudaMemsetAsync(a.flags, 0, (size_t)2 * tx * ty * nb * sizeof(unsigned), s));
  void (*fn)(LevelPDArgs) = pow2 ? k_pd_level<true> : k_pd_level<false>;
  FT_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(tx, ty, nb);
  cfg.blockDim = dim3(NT);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  FT_CUDA_TRY(cudaLaunchKernelEx(&cfg, fn, a));
  count_launch();
  return FT_OK;
}

}  // namespace ft

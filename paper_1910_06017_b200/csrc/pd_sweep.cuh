// Row-sweep primal-dual kernel (k_pd_sweep) -- included inside the anonymous
// namespace of k_flow.cu, after PDArgs / cp_async8 / madx.
//
// Same arithmetic, operation order and half-step launch schedule as k_pd_tile
// (reference optflow.py:178-208), organised without block barriers:
//
// * One warp owns a strip of 32 columns (lane = column) and a segment of
//   output rows, and streams down the rows.  The launch's NH half-steps are
//   pipelined stages: at sweep step s, stage j works on row s - j.  A stage
//   consumes only what its predecessors produced at earlier steps (P stages
//   run before D stages within a step), so every stage of a step is
//   independent of the others -- NH-way instruction-level parallelism.
// * x-neighbours come from warp shuffles (u-bar at x+1 in a dual step, p at
//   x-1 in a primal step); y-neighbours are the previous rows of the same
//   lane, carried in registers (each stage output lives for two steps).
// * The strip keeps K = 4 halo columns on each side (the x dependency cone
//   of <= 8 half-steps); rows are clipped per stage to the cone of the segment
//   (host-computed offsets SweepArgs::cA/cB), so there is no y halo waste.
// * Inputs (u, p, gx, gy, rho0) stream into a per-warp shared-memory ring
//   with cp.async, PF rows ahead; the per-row constants (gx, gy, rho0, the
//   threshold tau*lam*|grad|^2 and 1/|grad|^2) go to a second ring read by
//   the primal stages at their lag.  Every lane touches only its own column
//   there, so no synchronisation is needed.
// * The unit-ball projection (hypot + two divisions, ~9 % of pairs at C2) is
//   batched over all dual stages of a step: saturated pairs are compacted
//   into a per-warp queue (ballot/popc), projected by the first lanes, and
//   read back.
// Launch boundaries follow k_pd_tile's half-step schedule: a launch ends
// after a dual step (state u, p), or after a primal step in the warp's last
// launch (u only).

struct SweepArgs {
  StatePtrs in, out;
  const double *gx, *gy, *r0;
  int w, h;
  int64_t cap;
  int seg;      // output rows per warp segment
  int nstrips;  // strips per image row
  // stage j computes rows [y0 - cA[j], y1 + cB[j]) clipped to the image
  signed char cA[16], cB[16];
  double tau, tl, sigma, shrink;
};

// C = columns per lane (1 or 2): a warp covers 32*C columns, of which the
// outer K on each side are halo.
template <int NH, int C>
__host__ __device__ constexpr int sweep_halo() {
  return C == 1 ? (NH + 1) / 2 : ((NH + 1) / 2 + 1) / 2 * 2;  // even for C = 2 (16-byte pairs)
}

template <int NH, int NSLOT, int C>
struct SweepGeom {
  static constexpr int NC = 32 * C;               // columns per warp
  static constexpr int CR = NH <= 4 ? 4 : 8;      // constant-ring rows (>= NH)
  static constexpr int RING = NSLOT * 9 * NC;     // doubles: u1 u2 p11 p12 p21 p22 gx gy r0
  static constexpr int CRING = CR * 5 * NC;       // doubles: gx gy r0 thr ig2
  static constexpr int QUEUE = (NH + 1) / 2 * 2 * NC * 2;  // doubles: 2 pairs per dual stage per column
  static constexpr int PER_WARP = RING + CRING + QUEUE;
  static constexpr size_t smem_per_warp = PER_WARP * sizeof(double);
  static_assert(NH <= CR, "constant ring too short for the stage lags");
};

// Stage kinds of a launch: stage j is a dual step iff (j even) == FIRSTD.
template <bool FIRSTD>
__host__ __device__ constexpr bool sweep_is_dual(int j) {
  return ((j & 1) == 0) == FIRSTD;
}

__device__ __forceinline__ void cp_async16(double *dst, const double *src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(n));
}

template <int NH, bool FIRSTD, bool P2, int NSLOT, int MINB, int C>
__global__ void __launch_bounds__(32, MINB) k_pd_sweep(const SweepArgs a) {
  using G = SweepGeom<NH, NSLOT, C>;
  constexpr int NC = G::NC;
  constexpr int K = sweep_halo<NH, C>();  // strip halo: the launch's x dependency cone
  static_assert(NH >= 1 && NH <= 8, "at most 8 half-steps per launch");
  static_assert(C == 1 || C == 2, "one or two columns per lane");
  constexpr int STRIP = NC - 2 * K;
  constexpr int PF = NSLOT - 3;  // rows prefetched beyond s+1
  constexpr int L = NH - 1;      // last stage
  constexpr bool END_D = sweep_is_dual<FIRSTD>(L);
  static_assert(PF >= 1, "ring too short");
  extern __shared__ __align__(16) double sm[];

  const int lane = threadIdx.x;
  const int strip = blockIdx.x;
  double *const ring = sm;
  double *const cring = sm + G::RING;
  double2 *const queue = reinterpret_cast<double2 *>(sm + G::RING + G::CRING);

  const int W = a.w, H = a.h;
  const int x0 = strip * STRIP - K + C * lane;  // this lane's first column
  // 16-byte global pairs: even width and plane capacity (x0 is even for C=2)
  const bool vec = C == 2 && (W & 1) == 0 && (a.cap & 1) == 0;
  bool xin[C], wr[C], fR[C], fL[C], fLC[C];
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int x = x0 + c;
    xin[c] = x >= 0 && x < W;
    wr[c] = xin[c] && C * lane + c >= K && C * lane + c < NC - K;
    fR[c] = x < W - 1;
    fL[c] = x > 0;
    fLC[c] = x == W - 1;
  }
  const int y0 = blockIdx.y * a.seg, y1 = min(y0 + a.seg, H);
  const int64_t so = (int64_t)blockIdx.z * a.cap;
  const unsigned lt_mask = (1u << lane) - 1u;
  const double tau = a.tau, tl = a.tl, sigma = a.sigma, shrink = a.shrink;

  int lo[NH], hi[NH];
  int s1 = 0;
#pragma unroll
  for (int j = 0; j < NH; ++j) {
    lo[j] = max(y0 - (int)a.cA[j], 0);
    hi[j] = min(y1 + (int)a.cB[j], H);
    s1 = max(s1, hi[j] + j);
  }
  const int s0 = lo[0];
  const int lr0 = max(lo[0] - 1, 0), lr1 = min(hi[0] + 1, H);  // input rows to load

  // ---- input ring: row r -> slot r & (NSLOT-1), 9 planes x NC columns
  auto load_row = [&](int r) {
    if (r < lr0 || r >= lr1) return;
    double *dst = ring + (r & (NSLOT - 1)) * 9 * NC + C * lane;
    const int64_t o = so + (int64_t)r * W + x0;
    const double *src[9] = {a.in.p[U1], a.in.p[U2], a.in.p[P11], a.in.p[P12], a.in.p[P21],
                            a.in.p[P22], a.gx, a.gy, a.r0};
#pragma unroll
    for (int f = 0; f < 9; ++f) {
      if (FIRSTD && f >= 2 && f < 6) continue;  // p = 0 at the start of a warp
      if (C == 2 && vec) {
        cp_async16(dst + f * NC, xin[0] ? src[f] + o : src[f], xin[0]);
      } else {
#pragma unroll
        for (int c = 0; c < C; ++c) cp_async8(dst + f * NC + c, xin[c] ? src[f] + o + c : src[f], xin[c]);
      }
    }
  };
  // this lane's C values of plane f in ring row r / constant row r
  auto rd = [&](int r, int f, double *v) {
    const double *q = ring + (r & (NSLOT - 1)) * 9 * NC + f * NC + C * lane;
    if (C == 2) {
      const double2 t = *reinterpret_cast<const double2 *>(q);
      v[0] = t.x;
      v[C - 1] = t.y;
    } else {
      v[0] = q[0];
    }
  };
  auto crd = [&](int r, int f, double *v) {
    const double *q = cring + (r & (G::CR - 1)) * 5 * NC + f * NC + C * lane;
    if (C == 2) {
      const double2 t = *reinterpret_cast<const double2 *>(q);
      v[0] = t.x;
      v[C - 1] = t.y;
    } else {
      v[0] = q[0];
    }
  };

  // prologue: rows s0-1 .. s0+1 as one group, then s0+2 .. s0+PF one group each
  load_row(s0 - 1);
  load_row(s0);
  load_row(s0 + 1);
  cp_async_commit();
#pragma unroll
  for (int k = 2; k <= PF; ++k) {
    load_row(s0 + k);
    cp_async_commit();
  }

  // ---- stage carries (registers).  Slot t of a stage holds the row it
  // produced at a step with (s - s0) & 1 == t: on entry to a step, slot PB is
  // age 1 (previous step) and slot PA age 2; the step's outputs replace slot
  // PA.  Alternating the slot names (two step bodies per loop iteration)
  // keeps the carries in place -- no register moves.
  double pX[NH][2][4][C], uX[NH][2][2][C], bX[NH][2][2][C];
#pragma unroll
  for (int j = 0; j < NH; ++j)
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
      for (int c = 0; c < C; ++c) {
#pragma unroll
        for (int k = 0; k < 4; ++k) pX[j][t][k][c] = 0.0;
#pragma unroll
        for (int k = 0; k < 2; ++k) uX[j][t][k][c] = bX[j][t][k][c] = 0.0;
      }

  auto const_row = [&](int r) {
    double vgx[C], vgy[C], vr0[C];
    rd(r, 6, vgx);
    rd(r, 7, vgy);
    rd(r, 8, vr0);
    double *q = cring + (r & (G::CR - 1)) * 5 * NC + C * lane;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const double g2 = vgx[c] * vgx[c] + vgy[c] * vgy[c];
      const bool ok = g2 > 1e-12;
      q[0 * NC + c] = vgx[c];
      q[1 * NC + c] = vgy[c];
      q[2 * NC + c] = vr0[c];
      q[3 * NC + c] = tl * g2;
      q[4 * NC + c] = ok ? 1.0 / (g2 > 1e-12 ? g2 : 1e-12) : 0.0;
    }
  };

  int s = s0;
  // One sweep step.  Every stage runs every step (straight-line code the
  // scheduler can interleave); a stage whose row is outside its cone or the
  // image computes a value nobody reads -- only its projection requests and
  // the write-back are masked.
  auto step = [&](auto slot) {
    constexpr int PA = decltype(slot)::value, PB = PA ^ 1;
    load_row(s + 1 + PF);
    cp_async_commit();
    asm volatile("cp.async.wait_group %0;\n" ::"n"(PF) : "memory");
    if (s == s0 && s0 < lr1) const_row(s0);

    double pF[NH][4][C], uF[NH][2][C], bF[NH][2][C];
    // ---- primal stages (:194-208): rows s - j
#pragma unroll
    for (int j = 0; j < NH; ++j) {
      if (sweep_is_dual<FIRSTD>(j)) continue;
      const int r = s - j;
      double p11[C], p12[C], p21[C], p22[C], q12[C], q22[C], u1[C], u2[C];
      if (j == 0) {  // input p at rows r, r-1 and u at r
        rd(r, 2, p11); rd(r, 3, p12); rd(r, 4, p21); rd(r, 5, p22);
        rd(r - 1, 3, q12); rd(r - 1, 5, q22);
        rd(r, 0, u1); rd(r, 1, u2);
      } else {
#pragma unroll
        for (int c = 0; c < C; ++c) {
          p11[c] = pX[j - 1][PB][0][c]; p12[c] = pX[j - 1][PB][1][c];
          p21[c] = pX[j - 1][PB][2][c]; p22[c] = pX[j - 1][PB][3][c];
          q12[c] = pX[j - 1][PA][1][c]; q22[c] = pX[j - 1][PA][3][c];
        }
        if (j == 1) { rd(r, 0, u1); rd(r, 1, u2); }
        else {
#pragma unroll
          for (int c = 0; c < C; ++c) u1[c] = uX[j - 2][PA][0][c], u2[c] = uX[j - 2][PA][1][c];
        }
      }
      // p at x-1: the lane's previous column, or lane-1's last one
      double l11[C], l21[C];
      l11[0] = __shfl_up_sync(0xffffffffu, p11[C - 1], 1);
      l21[0] = __shfl_up_sync(0xffffffffu, p21[C - 1], 1);
#pragma unroll
      for (int c = 1; c < C; ++c) l11[c] = p11[c - 1], l21[c] = p21[c - 1];
      double gx[C], gy[C], r0[C], thr[C], ig2[C];
      crd(r, 0, gx); crd(r, 1, gy); crd(r, 2, r0); crd(r, 3, thr); crd(r, 4, ig2);
      const bool U = r > 0, LR = r == H - 1;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        // divergence (imageops.py:41-50) with the reference's border rules
        const double dx1 = fL[c] ? (fLC[c] ? -l11[c] : p11[c] - l11[c]) : p11[c];
        const double dx2 = fL[c] ? (fLC[c] ? -l21[c] : p21[c] - l21[c]) : p21[c];
        const double dy1 = U ? (LR ? -q12[c] : p12[c] - q12[c]) : p12[c];
        const double dy2 = U ? (LR ? -q22[c] : p22[c] - q22[c]) : p22[c];
        const double v1 = madx<P2>(tau, dx1 + dy1, u1[c]);
        const double v2 = madx<P2>(tau, dx2 + dy2, u2[c]);
        const double rho = r0[c] + gx[c] * v1 + gy[c] * v2;
        const bool lo_ = rho < -thr[c];
        const bool hi_ = rho > thr[c];
        double d = lo_ ? tl : (hi_ ? -tl : -rho * ig2[c]);
        d = (ig2[c] != 0.0 || lo_ || hi_) ? d : 0.0;  // ig2 != 0 <=> |grad|^2 > 1e-12
        const double n1 = v1 + d * gx[c];
        const double n2 = v2 + d * gy[c];
        uF[j][0][c] = n1;
        uF[j][1][c] = n2;
        bF[j][0][c] = madx<true>(2.0, n1, -u1[c]);
        bF[j][1][c] = madx<true>(2.0, n2, -u2[c]);
      }
    }
    // constants of row s+1 (optflow.py:163-176) for the next step's primal
    // stages (after this step's reads: the slot it replaces held row s+1-CR)
    if (s + 1 < lr1) const_row(s + 1);

    // ---- dual stages (:180-185), unprojected: rows s - j
    unsigned need = 0;
#pragma unroll
    for (int j = 0; j < NH; ++j) {
      if (!sweep_is_dual<FIRSTD>(j)) continue;
      const int r = s - j;
      double c1[C], c2[C], d1[C], d2[C], o11[C], o12[C], o21[C], o22[C];
      if (j == 0) {  // first launch: u-bar = u, p = 0
        rd(r, 0, c1); rd(r, 1, c2); rd(r + 1, 0, d1); rd(r + 1, 1, d2);
#pragma unroll
        for (int c = 0; c < C; ++c) o11[c] = o12[c] = o21[c] = o22[c] = 0.0;
      } else {
#pragma unroll
        for (int c = 0; c < C; ++c) {
          c1[c] = bX[j - 1][PB][0][c]; c2[c] = bX[j - 1][PB][1][c];
          d1[c] = bF[j - 1][0][c]; d2[c] = bF[j - 1][1][c];
        }
        if (j == 1) { rd(r, 2, o11); rd(r, 3, o12); rd(r, 4, o21); rd(r, 5, o22); }
        else {
#pragma unroll
          for (int c = 0; c < C; ++c) {
            o11[c] = pX[j - 2][PA][0][c]; o12[c] = pX[j - 2][PA][1][c];
            o21[c] = pX[j - 2][PA][2][c]; o22[c] = pX[j - 2][PA][3][c];
          }
        }
      }
      // u-bar at x+1: the lane's next column, or lane+1's first one
      double r1[C], r2[C];
      r1[C - 1] = __shfl_down_sync(0xffffffffu, c1[0], 1);
      r2[C - 1] = __shfl_down_sync(0xffffffffu, c2[0], 1);
#pragma unroll
      for (int c = 0; c + 1 < C; ++c) r1[c] = c1[c + 1], r2[c] = c2[c + 1];
      const bool D = r < H - 1;
      const unsigned valid = (r >= lo[j] && r < hi[j]) ? 3u : 0u;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const double a1x = fR[c] ? r1[c] - c1[c] : 0.0;
        const double a1y = D ? d1[c] - c1[c] : 0.0;
        const double a2x = fR[c] ? r2[c] - c2[c] : 0.0;
        const double a2y = D ? d2[c] - c2[c] : 0.0;
        const double p11 = madx<P2>(sigma, a1x, o11[c]) * shrink;
        const double p12 = madx<P2>(sigma, a1y, o12[c]) * shrink;
        const double p21 = madx<P2>(sigma, a2x, o21[c]) * shrink;
        const double p22 = madx<P2>(sigma, a2y, o22[c]) * shrink;
        pF[j][0][c] = p11; pF[j][1][c] = p12; pF[j][2][c] = p21; pF[j][3][c] = p22;
        // screening test only (not reference arithmetic): fused is fine.
        // Rows outside the stage's cone are never read: no projection.
        const unsigned sat = (fma(p11, p11, p12 * p12) > 0.999999 ? 1u : 0u) |
                             (fma(p21, p21, p22 * p22) > 0.999999 ? 2u : 0u);
        need |= (sat & valid) << (2 * (j * C + c));
      }
    }

    // ---- unit-ball projection n = max(1, hypot(.)); p /= n (:186-191),
    // batched over the dual stages of this step through a per-warp queue.
    // need bit 2*(j*C + c) + k: pair k (0: p11,p12; 1: p21,p22) of column c.
    if (__any_sync(0xffffffffu, need != 0u)) {
      int off[2 * NH * C];
      int total = 0;
#pragma unroll
      for (int k = 0; k < 2 * NH * C; ++k) {
        if (!sweep_is_dual<FIRSTD>(k / (2 * C))) continue;
        const unsigned m = __ballot_sync(0xffffffffu, (need >> k) & 1u);
        off[k] = total + __popc(m & lt_mask);
        total += __popc(m);
      }
#pragma unroll
      for (int k = 0; k < 2 * NH * C; ++k) {
        if (!sweep_is_dual<FIRSTD>(k / (2 * C))) continue;
        if ((need >> k) & 1u) {
          const int j = k / (2 * C), c = (k >> 1) % C, e = (k & 1) * 2;
          queue[off[k]] = make_double2(pF[j][e][c], pF[j][e + 1][c]);
        }
      }
      __syncwarp();
      for (int e = lane; e < total; e += 32) {
        const double2 v = queue[e];
        const double nn = np_max(1.0, glibc_hypot(v.x, v.y));
        queue[e] = make_double2(v.x / nn, v.y / nn);
      }
      __syncwarp();
#pragma unroll
      for (int k = 0; k < 2 * NH * C; ++k) {
        if (!sweep_is_dual<FIRSTD>(k / (2 * C))) continue;
        if ((need >> k) & 1u) {
          const int j = k / (2 * C), c = (k >> 1) % C, e = (k & 1) * 2;
          const double2 v = queue[off[k]];
          pF[j][e][c] = v.x;
          pF[j][e + 1][c] = v.y;
        }
      }
      __syncwarp();
    }

    // ---- write back the segment's rows of the last stage (interior columns)
    {
      const int r = s - L;
      if (r >= y0 && r < y1) {
        const int64_t o = so + (int64_t)r * W + x0;
        auto put = [&](int plane, const double *v) {
          if (C == 2 && vec) {
            if (wr[0]) *reinterpret_cast<double2 *>(a.out.p[plane] + o) = make_double2(v[0], v[C - 1]);
          } else {
#pragma unroll
            for (int c = 0; c < C; ++c)
              if (wr[c]) a.out.p[plane][o + c] = v[c];
          }
        };
        if (END_D) {
          put(U1, uX[L - 1][PB][0]);
          put(U2, uX[L - 1][PB][1]);
          put(P11, pF[L][0]);
          put(P12, pF[L][1]);
          put(P21, pF[L][2]);
          put(P22, pF[L][3]);
        } else {
          put(U1, uF[L][0]);
          put(U2, uF[L][1]);
        }
      }
    }

    // ---- this step's outputs replace the age-2 slot
#pragma unroll
    for (int j = 0; j < NH; ++j)
#pragma unroll
      for (int c = 0; c < C; ++c) {
        if (sweep_is_dual<FIRSTD>(j)) {
#pragma unroll
          for (int k = 0; k < 4; ++k) pX[j][PA][k][c] = pF[j][k][c];
        } else {
#pragma unroll
          for (int k = 0; k < 2; ++k) {
            uX[j][PA][k][c] = uF[j][k][c];
            bX[j][PA][k][c] = bF[j][k][c];
          }
        }
      }
    ++s;
  };
  while (s + 1 < s1) {
    step(std::integral_constant<int, 0>{});
    step(std::integral_constant<int, 1>{});
  }
  if (s < s1) step(std::integral_constant<int, 0>{});
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

// Rows each stage must compute, as offsets from the written segment
// [y0, y1): stage j covers [y0 - cA[j], y1 + cB[j]).  Propagated backwards
// from the launch's outputs: a dual step at row r reads u-bar at r, r+1 and
// the previous p at r; a primal step reads p at r, r-1 and the previous u at
// r.
inline void sweep_cone(bool firstd, int nh, signed char *cA, signed char *cB) {
  const int kNone = -1000;
  int A[16], B[16];
  for (int j = 0; j < 16; ++j) A[j] = B[j] = kNone;
  const int L = nh - 1;
  auto isd = [&](int j) { return ((j & 1) == 0) == firstd; };
  auto cover = [&](int j, int a, int b) {
    if (j < 0) return;
    A[j] = std::max(A[j], a);
    B[j] = std::max(B[j], b);
  };
  cover(L, 0, 0);
  if (isd(L)) cover(L - 1, 0, 0);  // u of the segment comes from the last primal
  for (int j = L; j >= 0; --j) {
    if (A[j] == kNone) continue;
    if (isd(j)) {
      cover(j - 1, A[j], B[j] + 1);
      cover(j - 2, A[j], B[j]);
    } else {
      cover(j - 1, A[j] + 1, B[j]);
      cover(j - 2, A[j], B[j]);
    }
  }
  for (int j = 0; j < 16; ++j) {
    cA[j] = (signed char)(j < nh ? std::max(A[j], 0) : 0);
    cB[j] = (signed char)(j < nh ? std::max(B[j], 0) : 0);
  }
}

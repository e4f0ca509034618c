// Standalone GPU check of k_pd_sweep against k_pd_tile, one launch of each
// half-step schedule on a random state (bit-exact compare).  Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 \
//     --expt-relaxed-constexpr -I include -o /tmp/sweep_test tools/sweep_test.cu \
//     -L paper_1910_06017_b200 -lomnitrack -Xlinker -rpath=$PWD/paper_1910_06017_b200
#include "../paper_1910_06017_b200/csrc/k_flow.cu"
#include <cstdio>
#include <random>
#include <vector>

using namespace ft;

int flow_check(int W, int H, int iters, int warps);

int main(int argc, char **argv) {
  if (argc > 3) return flow_check(atoi(argv[1]), atoi(argv[2]), atoi(argv[3]), atoi(argv[4]));
  const int W = argc > 1 ? atoi(argv[1]) : 53, H = argc > 2 ? atoi(argv[2]) : 45, nb = 2;
  const int64_t cap = (int64_t)W * H;
  std::mt19937_64 rng(7);
  std::normal_distribution<double> nd(0.0, 1.0);
  std::uniform_real_distribution<double> ud(-0.7, 0.7);
  const size_t plane = nb * cap;
  std::vector<double> hin(NST * plane), hc(3 * plane);
  for (size_t i = 0; i < NST * plane; ++i) hin[i] = (i / plane) >= P11 ? ud(rng) : nd(rng);
  for (size_t i = 0; i < 3 * plane; ++i) hc[i] = nd(rng) * (i < 2 * plane ? 1.0 : 0.3);
  double *din, *dt, *ds, *dc;
  cudaMalloc(&din, NST * plane * 8);
  cudaMalloc(&dt, NST * plane * 8);
  cudaMalloc(&ds, NST * plane * 8);
  cudaMalloc(&dc, 3 * plane * 8);
  cudaMemcpy(din, hin.data(), NST * plane * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dc, hc.data(), 3 * plane * 8, cudaMemcpyHostToDevice);
  struct Case { bool first; int nh; };
  const Case cases[] = {{true, 7}, {false, 8}, {false, 5}, {false, 1}, {true, 4}, {false, 3}, {true, 2}};
  int bad = 0;
  for (const Case &c : cases) {
    const bool endd = ((((c.nh - 1) & 1) == 0) == c.first);
    PDArgs a{};
    a.in = state_ptrs(din, nb, cap);
    a.gx = dc;
    a.gy = dc + plane;
    a.r0 = dc + 2 * plane;
    a.w = W;
    a.h = H;
    a.cap = cap;
    a.halo = 4;
    a.iters = c.nh;
    a.nb = nb;
    a.pow2 = 1;
    a.cone = 1;
    a.cq = 1;
    a.async_ld = 1;
    a.tau = 0.25;
    a.lam = 0.15;
    a.sigma = 0.5;
    a.shrink = 1.0 / (1.0 + 0.5 * 0.01);
    halfstep_schedule(a, c.first, c.nh, !endd, 4, 32);
    cudaMemset(dt, 0xff, NST * plane * 8);
    cudaMemset(ds, 0xff, NST * plane * 8);
    a.out = state_ptrs(dt, nb, cap);
    int rc1 = pd_launch(pd_config(1), a, nb, 0);
    a.out = state_ptrs(ds, nb, cap);
    int rc2 = sweep_launch(a, c.nh, c.first, nb, 0);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<double> ht(NST * plane), hs(NST * plane);
    cudaMemcpy(ht.data(), dt, NST * plane * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hs.data(), ds, NST * plane * 8, cudaMemcpyDeviceToHost);
    long nmis = 0;
    double mx = 0;
    int fr = -1, fc = -1, fp = -1, fb = -1;
    for (int pl : {U1, U2, P11, P12, P21, P22}) {
      if (!endd && pl >= P11) continue;
      for (int b = 0; b < nb; ++b)
        for (int y = 0; y < H; ++y)
          for (int x = 0; x < W; ++x) {
            const size_t i = pl * plane + b * cap + (size_t)y * W + x;
            if (memcmp(&ht[i], &hs[i], 8) != 0) {
              if (nmis == 0) fr = y, fc = x, fp = pl, fb = b;
              ++nmis;
              mx = std::max(mx, std::fabs(ht[i] - hs[i]));
            }
          }
    }
    printf("first=%d nh=%d rc=%d/%d err=%s mismatches=%ld maxdiff=%g first(b=%d plane=%d y=%d x=%d)\n",
           c.first, c.nh, rc1, rc2, cudaGetErrorString(e), nmis, mx, fb, fp, fr, fc);
    if (nmis) {
      const size_t i = fp * plane + fb * cap + (size_t)fr * W + fc;
      printf("   tile=%.17g sweep=%.17g\n", ht[i], hs[i]);
      ++bad;
    }
  }
  printf(bad ? "SWEEP MISMATCH\n" : "SWEEP OK\n");
  return bad ? 1 : 0;
}

// whole-flow check: run_flow with FT_PD_SWEEP=0 and =1 on random pyramids
int flow_check(int W, int H, int iters, int warps) {
  const int S = 2;
  int lw[2] = {W, W / 2}, lh[2] = {H, H / 2};
  int64_t loff[2] = {0, (int64_t)W * H};
  const int64_t tot = (int64_t)W * H + (int64_t)(W / 2) * (H / 2);
  std::vector<double> h0(tot), h1(tot);
  std::mt19937_64 rng(3);
  std::uniform_real_distribution<double> ud(0.0, 255.0);
  for (auto &v : h0) v = ud(rng);
  for (int64_t i = 0; i < tot; ++i) h1[i] = 0.7 * h0[i] + 0.3 * ud(rng);
  double *p0, *p1, *dx, *dy;
  cudaMalloc(&p0, tot * 8);
  cudaMalloc(&p1, tot * 8);
  cudaMalloc(&dx, (size_t)W * H * 8 * 2);
  dy = dx + (size_t)W * H;
  cudaMemcpy(p0, h0.data(), tot * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(p1, h1.data(), tot * 8, cudaMemcpyHostToDevice);
  FlowWork fw;
  flow_work_alloc(fw, 1, (int64_t)W * H);
  FlowParamsD p{0.15, 0.25, 0.01, warps, iters};
  cudaStream_t s;
  cudaStreamCreate(&s);
  std::vector<double> out[2];
  for (int v = 0; v < 2; ++v) {
    setenv("FT_PD_SWEEP", v ? "1" : "0", 1);
    cudaMemset(dx, 0, (size_t)W * H * 16);
    int rc = run_flow(p0, p1, 0, lw, lh, loff, S, p, fw, dx, dy, 0, 1, s, nullptr);
    cudaStreamSynchronize(s);
    out[v].resize((size_t)W * H * 2);
    cudaMemcpy(out[v].data(), dx, (size_t)W * H * 16, cudaMemcpyDeviceToHost);
    printf("  run_flow sweep=%d rc=%d err=%s\n", v, rc, cudaGetErrorString(cudaGetLastError()));
  }
  long nm = 0;
  double mx = 0;
  for (size_t i = 0; i < out[0].size(); ++i)
    if (memcmp(&out[0][i], &out[1][i], 8)) ++nm, mx = std::max(mx, std::fabs(out[0][i] - out[1][i]));
  printf("flow %dx%d iters=%d warps=%d: mismatches=%ld maxdiff=%g\n", W, H, iters, warps, nm, mx);
  return nm != 0;
}

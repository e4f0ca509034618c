// Microbenchmark: inter-CTA signalling latency through L2 on this GPU
// (calibrates the tile-edge exchange of k_pd_level.cu).  Two CTAs (on
// different SMs) bounce a counter N times; reports ns per one-way hop for
// several publish / poll idioms, and the cost of a gpu-scope fence.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pingpong tools/pingpong.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_relaxed(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed(unsigned *p, unsigned v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// MODE 0: st.release / ld.acquire
// MODE 1: data store + __threadfence + st.release / ld.acquire + ld.cg data
// MODE 2: st.relaxed / ld.relaxed (no ordering: latency floor)
// MODE 3: 32 lanes store data, __syncwarp, lane 0 st.release; all lanes ld.acquire + ld.cg
template <int MODE>
__global__ void pingpong(unsigned *flags, double2 *data, int n, long long *out) {
  const int me = blockIdx.x, other = 1 - me;
  const int lane = threadIdx.x;
  long long t0 = clock64();
  double2 acc = make_double2(0, 0);
  for (int i = 1; i <= n; ++i) {
    if ((i & 1) == me) {  // my turn to send value i
      if (MODE == 1 || MODE == 3) data[me * 32 + lane] = make_double2(i, lane);
      if (MODE == 1) __threadfence();
      if (MODE == 3 || MODE == 1) __syncwarp();
      if (lane == 0) {
        if (MODE == 2) st_relaxed(&flags[me * 32], i);
        else st_release(&flags[me * 32], i);
      }
    } else {
      if (MODE == 2) {
        while (ld_relaxed(&flags[other * 32]) < (unsigned)i) {}
      } else {
        while (ld_acquire(&flags[other * 32]) < (unsigned)i) {}
      }
      if (MODE == 1 || MODE == 3) {
        const double2 v = __ldcg(&data[other * 32 + lane]);
        acc.x += v.x;
        acc.y += v.y;
      }
    }
  }
  long long t1 = clock64();
  if (lane == 0) out[me] = t1 - t0;
  if (acc.x == -1) out[2] = 1;
}

__global__ void fence_cost(long long *out, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __threadfence();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main() {
  unsigned *flags;
  double2 *data;
  long long *out;
  cudaMalloc(&flags, 4096);
  cudaMalloc(&data, 4096);
  cudaMallocManaged(&out, 64);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int n = 20000;
  const char *names[4] = {"release/acquire", "data+fence+release / acquire+ld.cg",
                          "relaxed/relaxed", "warp data+syncwarp+release / acquire+ld.cg"};
  for (int m = 0; m < 4; ++m) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(flags, 0, 4096);
      if (m == 0) pingpong<0><<<2, 32>>>(flags, data, n, out);
      if (m == 1) pingpong<1><<<2, 32>>>(flags, data, n, out);
      if (m == 2) pingpong<2><<<2, 32>>>(flags, data, n, out);
      if (m == 3) pingpong<3><<<2, 32>>>(flags, data, n, out);
      cudaDeviceSynchronize();
    }
    const double cyc = (double)out[0] / n;
    printf("%-48s %7.1f cycles/hop  %6.1f ns/hop\n", names[m], cyc, cyc / (clk * 1e-6));
  }
  fence_cost<<<148, 32>>>(out, 1000);
  cudaDeviceSynchronize();
  printf("__threadfence (no outstanding stores): %.1f cycles\n", (double)out[0] / 1000);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

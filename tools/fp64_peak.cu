// Microbenchmark: sustained fp64 DFMA / DADD / DMUL issue rate on this GPU
// (the fp64 pipe bounds the TV-L1 iteration once data is on chip).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double *out, int iters, double a, double b) {
  double x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) x[i] = fma(x[i], a, b);
      else if (OP == 1) x[i] = __dadd_rn(x[i], b);
      else x[i] = __dmul_rn(x[i], a);
    }
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}
int main() {
  double *d; cudaMalloc(&d, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const char *names[3] = {"DFMA", "DADD", "DMUL"};
  for (int op = 0; op < 3; ++op) {
    int iters = 4096, blocks = sms * 8, threads = 256;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (op == 0) k<0><<<blocks, threads>>>(d, iters, 0.999, 1e-3);
      if (op == 1) k<1><<<blocks, threads>>>(d, iters, 0.999, 1e-3);
      if (op == 2) k<2><<<blocks, threads>>>(d, iters, 0.999, 1e-3);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
    }
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)blocks * threads * iters * 8;
    printf("%s: %.2f Tops/s  (%.1f ops/clk/SM at 1965 MHz)\n", names[op], ops / ms / 1e9,
           ops / (ms * 1e-3) / sms / 1.965e9);
  }
  return 0;
}

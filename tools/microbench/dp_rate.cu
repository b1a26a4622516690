// Measured fp64 issue rates on this GPU: independent DADD / DMUL / DFMA chains.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dp_rate dp_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(double* out, double s, int iters) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (OP == 0) a[j] = a[j] + s;
      if (OP == 1) a[j] = a[j] * s;
      if (OP == 2) a[j] = fma(a[j], s, s);
    }
  }
  double t = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) t += a[j];
  if (t == 12345.678) out[0] = t;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const char* names[3] = {"DADD", "DMUL", "DFMA"};
  for (int threads : {256, 512, 1024}) {
    for (int op = 0; op < 3; ++op) {
      const int iters = 4096;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto launch = [&] {
        if (op == 0) k<0><<<nsm, threads>>>(out, 1.0000001, iters);
        if (op == 1) k<1><<<nsm, threads>>>(out, 1.0000001, iters);
        if (op == 2) k<2><<<nsm, threads>>>(out, 1.0000001, iters);
      };
      launch();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)nsm * threads * iters * 8;
      int clk;
      cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
      printf("%s threads/SM %4d: %.3f ms  %.2f Tops/s  %.1f lane-ops/clk/SM (at %d MHz)\n", names[op], threads, ms,
             ops / ms / 1e9, ops / (ms * 1e-3) / nsm / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}

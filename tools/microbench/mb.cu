// Microbenchmarks used to size the B200 design: HBM / L2-resident streaming bandwidth,
// fp64 DFMA issue rate, shared-memory 16-byte bandwidth.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e){printf("CUDA %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__global__ void copyk(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x, st = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += st) b[i] = a[i];
}
__global__ void fmak(double* out, int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4=a0+4,a5=a0+5,a6=a0+6,a7=a0+7;
  const double b = 0.999999, c = 1e-9;
  for (int i = 0; i < iters; ++i) {
    a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
    a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}
__global__ void smemk(double* out, int iters) {
  __shared__ double2 s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_double2(i, i);
  __syncthreads();
  double2 acc = make_double2(0, 0);
  int idx = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    double2 v = s[(idx + i * 32) & 2047];
    acc.x += v.x; acc.y += v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
}
int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("%s SMs=%d L2=%d MB smemPerBlockOptin=%zu clock=%d kHz memclk=%d kHz bus=%d\n", p.name, p.multiProcessorCount,
         p.l2CacheSize >> 20, p.sharedMemPerBlockOptin, p.clockRate, p.memoryClockRate, p.memoryBusWidth);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  size_t sizes_mb[] = {4, 8, 16, 32, 48, 64, 96, 2048};
  for (size_t mb : sizes_mb) {
    size_t bytes = mb << 20, n = bytes / 16;
    double2 *a, *b; CK(cudaMalloc(&a, bytes)); CK(cudaMalloc(&b, bytes));
    cudaMemset(a, 0, bytes); cudaMemset(b, 0, bytes);
    int reps = mb >= 1024 ? 10 : 200;
    for (int grid : {148 * 4, 148 * 8}) {
      copyk<<<grid, 512>>>(a, b, n);
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) copyk<<<grid, 512>>>(a, b, n);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      printf("copy %5zu MB grid %d: %.1f GB/s (r+w)\n", mb, grid, 2.0 * bytes * reps / (ms * 1e-3) / 1e9);
    }
    cudaFree(a); cudaFree(b);
  }
  double* o; CK(cudaMalloc(&o, 148 * 64 * 1024 * 8));
  for (int bs : {256, 512, 1024}) {
    int iters = 20000;
    fmak<<<148 * 2, bs>>>(o, 100);
    cudaEventRecord(e0); fmak<<<148 * 2, bs>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * 148.0 * 2 * bs;
    printf("DFMA bs=%d: %.2f TFLOP/s\n", bs, fl / (ms * 1e-3) / 1e12);
  }
  {
    int iters = 20000, bs = 512;
    smemk<<<148 * 2, bs>>>(o, 100);
    cudaEventRecord(e0); smemk<<<148 * 2, bs>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double by = 16.0 * iters * 148.0 * 2 * bs;
    printf("smem LDS.128: %.1f TB/s chip, %.1f B/clk/SM at %d MHz\n", by / (ms * 1e-3) / 1e12,
           by / (ms * 1e-3) / 148 / (p.clockRate * 1e3), p.clockRate / 1000);
  }
  return 0;
}

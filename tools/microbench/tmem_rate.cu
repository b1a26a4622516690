// tcgen05.ld / tcgen05.st throughput per SM (32x32b shapes), 4..16 warps per CTA, one CTA per SM.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void ld32(unsigned a, unsigned* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
               : "r"(a));
}
__device__ __forceinline__ void st32(unsigned a, const unsigned* v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};"
               :: "r"(a), "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
               : "memory");
}

template <int MODE>  // 0 = ld, 1 = st, 2 = ld+st
__global__ void k(unsigned* out, int iters) {
  __shared__ unsigned base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (unsigned)__cvta_generic_to_shared(&base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const unsigned ta = base + ((unsigned)(32 * (warp & 3)) << 16) + 32u * (unsigned)((warp >> 2) & 15);
  unsigned v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = threadIdx.x + i;
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
      ld32(ta, v);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) acc += v[i];
    }
    if (MODE != 0) {
      v[it & 31] += 1;
      st32(ta, v);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
  }
  if (acc == 0xdeadbeef) out[0] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

int main() {
  unsigned* out;
  cudaMalloc(&out, 4);
  int nsm, clk;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const char* nm[3] = {"ld32", "st32", "ld32+st32"};
  for (int warps : {4, 8, 16}) {
    for (int mode = 0; mode < 3; ++mode) {
      const int iters = 20000;
      auto launch = [&] {
        if (mode == 0) k<0><<<nsm, warps * 32>>>(out, iters);
        if (mode == 1) k<1><<<nsm, warps * 32>>>(out, iters);
        if (mode == 2) k<2><<<nsm, warps * 32>>>(out, iters);
      };
      launch();
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double bytes = (double)warps * 32 * 128 * iters * (mode == 2 ? 2 : 1);
      printf("%-10s warps %2d: %.3f ms  %.1f B/clk/SM  (err %s)\n", nm[mode], warps, ms,
             bytes / (ms * 1e-3) / (clk * 1e3), cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}

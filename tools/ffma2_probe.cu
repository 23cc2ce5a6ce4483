// Development probe: FFMA2 throughput vs operand pattern (register-file
// operand bandwidth).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ffma2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) { u64 r; asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ void f2(u64& d, u64 a, u64 b) { asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b)); }

template <int MODE>
__global__ void __launch_bounds__(256) k(int iters, float* sink, float seed) {
  float a[8]; u64 b[4]; u64 d[8][4];
  for (int i = 0; i < 8; ++i) a[i] = seed + i * threadIdx.x;
  for (int p = 0; p < 4; ++p) b[p] = pk(seed * p, seed + p);
  for (int i = 0; i < 8; ++i) for (int p = 0; p < 4; ++p) d[i][p] = 0;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {        // p outer, i inner (b reused)
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int i = 0; i < 8; ++i) f2(d[i][p], pk(a[i], a[i]), b[p]);
    } else if (MODE == 1) { // i outer, p inner (a reused)
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) f2(d[i][p], pk(a[i], a[i]), b[p]);
    } else if (MODE == 2) { // pairs for a too (no broadcast)
#pragma unroll
      for (int i = 0; i < 8; i += 2)
#pragma unroll
        for (int p = 0; p < 4; ++p) { f2(d[i][p], pk(a[i], a[i+1]), b[p]); f2(d[i+1][p], pk(a[i+1], a[i]), b[p]); }
    } else {                // same a, same b, 32 accumulators
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) f2(d[i][p], pk(a[0], a[0]), b[0]);
    }
  }
  u64 s = 0;
  for (int i = 0; i < 8; ++i) for (int p = 0; p < 4; ++p) s ^= d[i][p];
  if (s == 42) sink[threadIdx.x] = (float)s;
}

template <int MODE> void run(const char* name, int warps_per_sm) {
  float* sink; cudaMalloc(&sink, 4096);
  int iters = 4000; int blocks = 148 * warps_per_sm / 8;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<blocks, 256>>>(10, sink, 1.0f);
  cudaEventRecord(e0); k<MODE><<<blocks, 256>>>(iters, sink, 1.0f); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = (double)blocks * 256 * iters * 32 * 4;
  printf("%-28s warps/SM=%2d  %.1f TFLOP/s\n", name, warps_per_sm, flops / ms / 1e9);
}
int main() {
  for (int w : {8, 16}) {
    run<0>("p-outer (b reuse)", w); run<1>("i-outer (a reuse)", w); run<2>("paired a, no bcast", w); run<3>("all reuse", w);
  }
}

// Development probe: the FFMA2 outer-product operand pattern of sgemm_tma.cu
// (B pair reused across rows, one fresh broadcast A scalar per instruction)
// as a function of the CTA shape: math warps per SM x accumulator block per
// lane (ROWS x PAIRS).  Register-only loops; answers whether more resident
// warps with a smaller register block lift the pattern's ceiling.
//   outer : d[i][p] = b[p] * {a[i], a[i]} + d[i][p]   (p outer, i inner)
//   acc   : d[i][p] = x * d[i][p] + y                 (accumulator read only)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ffma2_shape_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2(u64& d, u64 a, u64 b) {
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}

template <int WARPS, int CTAS, int ROWS, int PAIRS, int MODE>
__global__ void __launch_bounds__(WARPS * 32, CTAS) k(int iters, float* sink, float seed) {
  u64 b[PAIRS], d[ROWS][PAIRS];
#pragma unroll
  for (int p = 0; p < PAIRS; ++p) b[p] = pk(seed * p + threadIdx.x, seed + p);
#pragma unroll
  for (int i = 0; i < ROWS; ++i)
#pragma unroll
    for (int p = 0; p < PAIRS; ++p) d[i][p] = 0;
  float ar[ROWS];
#pragma unroll
  for (int i = 0; i < ROWS; ++i) ar[i] = seed + i * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    if (MODE == 1) {
#pragma unroll
      for (int i = 0; i < ROWS; ++i)
#pragma unroll
        for (int p = 0; p < PAIRS; ++p) f2(d[i][p], b[0], b[1 % PAIRS]);
    } else {
#pragma unroll
      for (int p = 0; p < PAIRS; ++p)
#pragma unroll
        for (int i = 0; i < ROWS; ++i) f2(d[i][p], b[p], pk(ar[i], ar[i]));
    }
  }
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < ROWS; ++i)
#pragma unroll
    for (int p = 0; p < PAIRS; ++p) s ^= d[i][p];
  if (s == 42) sink[threadIdx.x] = (float)s;
}

template <int WARPS, int CTAS, int ROWS, int PAIRS, int MODE>
void run(float* sink) {
  const int iters = 20000, blocks = 148 * CTAS;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<WARPS, CTAS, ROWS, PAIRS, MODE><<<blocks, WARPS * 32>>>(10, sink, 1.0f);
  cudaEventRecord(e0);
  k<WARPS, CTAS, ROWS, PAIRS, MODE><<<blocks, WARPS * 32>>>(iters, sink, 1.0f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = double(blocks) * WARPS * 32 * iters * ROWS * PAIRS * 4;
  std::printf("%-5s warps/SM %2d  block %dx%d pairs  %.1f TFLOP/s\n", MODE ? "acc" : "outer",
              WARPS * CTAS, ROWS, PAIRS, flops / ms / 1e9);
}

template <int WARPS, int CTAS, int ROWS, int PAIRS>
void both(float* sink) {
  run<WARPS, CTAS, ROWS, PAIRS, 0>(sink);
  run<WARPS, CTAS, ROWS, PAIRS, 1>(sink);
}

int main() {
  float* sink;
  cudaMalloc(&sink, 4096);
  for (int r = 0; r < 2; ++r) {
    both<8, 1, 8, 8>(sink);    // today's kernel shape
    both<8, 1, 16, 4>(sink);   // same warps, taller block
    both<8, 1, 4, 16>(sink);   // same warps, wider block
    both<12, 1, 8, 5>(sink);
    both<16, 1, 8, 4>(sink);   // 16 math warps, half the block
    both<16, 1, 4, 8>(sink);
    both<16, 1, 6, 5>(sink);
    both<8, 2, 8, 4>(sink);    // two CTAs of 8 warps
    both<4, 1, 8, 8>(sink);    // one warp per scheduler
    both<16, 2, 4, 4>(sink);   // 32 warps
    std::printf("\n");
  }
  return cudaGetLastError() != cudaSuccess;
}

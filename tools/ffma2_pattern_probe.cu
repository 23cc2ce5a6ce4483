// Development probe: FFMA2 outer-product operand patterns at the sgemm kernel's
// shape (8 math warps per SM, 64 accumulator pairs per lane).
//   bcast : d[i][p] += {a_i, a_i} * (b_2p, b_2p+1)          (sgemm_tma.cu today)
//   diag  : d[q][p][0] += (a_2q, a_2q+1) * (b_2p, b_2p+1)
//           d[q][p][1] += (a_2q, a_2q+1) * (b_2p+1, b_2p)    (swapped pair held in registers)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ffma2_pattern_probe.cu
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

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(int iters, float* sink, float seed) {
  float a[8], bf[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + i * threadIdx.x;
#pragma unroll
  for (int j = 0; j < 16; ++j) bf[j] = seed * j + threadIdx.x;
  u64 d[64];
#pragma unroll
  for (int i = 0; i < 64; ++i) d[i] = 0;
  u64 b[8], bs[8], ap[4];
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    b[p] = pk(bf[2 * p], bf[2 * p + 1]);
    bs[p] = pk(bf[2 * p + 1], bf[2 * p]);
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) ap[q] = pk(a[2 * q], a[2 * q + 1]);
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 8; ++p) f2(d[i * 8 + p], pk(a[i], a[i]), b[p]);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int p = 0; p < 8; ++p) {
          f2(d[q * 16 + 2 * p], ap[q], b[p]);
          f2(d[q * 16 + 2 * p + 1], ap[q], bs[p]);
        }
    }
  }
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < 64; ++i) s ^= d[i];
  if (s == 42) sink[threadIdx.x] = (float)s;
}

template <int MODE>
void run(const char* name) {
  float* sink;
  cudaMalloc(&sink, 4096);
  const int iters = 20000, blocks = 148;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<MODE><<<blocks, 256>>>(10, sink, 1.0f);
  cudaEventRecord(e0);
  k<MODE><<<blocks, 256>>>(iters, sink, 1.0f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = double(blocks) * 256 * iters * 64 * 4;
  std::printf("%-8s %.1f TFLOP/s\n", name, flops / ms / 1e9);
}
int main() {
  for (int r = 0; r < 2; ++r) {
    run<0>("bcast");
    run<1>("diag");
  }
}

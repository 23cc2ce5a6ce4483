// Development probe: does taking the broadcast A scalar of the FFMA2 outer
// product from a uniform register (FFMA2 Rd, Rb.F32x2, URa.F32, Rd) lift the
// register-file-bound rate of the sgemm kernel's operand pattern?  Register-
// only loops at the kernel's shape (8 warps per SM, 64 accumulator pairs per
// lane, B pair outer / A scalar inner):
//   rscalar : A scalar in a regular register (sgemm_tma.cu today)
//   uconst  : A scalar from constant memory (LDCU -> uniform register)
//   uredux  : A scalar loaded from shared memory, made uniform by redux.sync
//   peak    : FFMA2 d = x*d + y (only the accumulator read from the RF)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ffma2_uniform_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__constant__ float ca[4096];
__device__ __forceinline__ u64 pk(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2(u64& d, u64 a, u64 b) {
  asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
__device__ __forceinline__ float uni(float x) {
  unsigned r;
  asm volatile("redux.sync.or.b32 %0, %1, 0xffffffff;" : "=r"(r) : "r"(__float_as_uint(x)));
  return __uint_as_float(r);
}

template <int MODE>
__global__ void __launch_bounds__(256, 1) k(int iters, float* sink, float seed, const float* g) {
  __shared__ float sa[8][1024];
  for (int i = threadIdx.x; i < 8 * 1024; i += 256) (&sa[0][0])[i] = g[i & 4095];
  __syncthreads();
  const int w = threadIdx.x >> 5;
  u64 b[8], d[8][8];
#pragma unroll
  for (int p = 0; p < 8; ++p) b[p] = pk(seed * p + threadIdx.x, seed + p);
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int p = 0; p < 8; ++p) d[i][p] = 0;
  float ar[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) ar[i] = seed + i * threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    float av[8];
    if (MODE == 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i) av[i] = ar[i];
    } else if (MODE == 1) {
      const float* a = ca + (it & 511) * 8;
#pragma unroll
      for (int i = 0; i < 8; ++i) av[i] = a[i];
    } else if (MODE == 2) {
      const float* a = &sa[w][(it & 127) * 8];
#pragma unroll
      for (int i = 0; i < 8; ++i) av[i] = uni(a[i]);
    }
    if (MODE == 3) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 8; ++p) f2(d[i][p], b[0], b[1]);
    } else {
#pragma unroll
      for (int p = 0; p < 8; ++p)
#pragma unroll
        for (int i = 0; i < 8; ++i) f2(d[i][p], b[p], pk(av[i], av[i]));
    }
  }
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int p = 0; p < 8; ++p) s ^= d[i][p];
  if (s == 42) sink[threadIdx.x] = (float)s;
}

template <int MODE>
void run(const char* name, const float* g, float* sink) {
  const int iters = 20000, blocks = 148;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<MODE><<<blocks, 256>>>(10, sink, 1.0f, g);
  cudaEventRecord(e0);
  k<MODE><<<blocks, 256>>>(iters, sink, 1.0f, g);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = double(blocks) * 256 * iters * 64 * 4;
  std::printf("%-8s %.1f TFLOP/s\n", name, flops / ms / 1e9);
}

int main() {
  float *g, *sink;
  cudaMalloc(&g, 4096 * 4);
  cudaMemset(g, 0, 4096 * 4);
  cudaMalloc(&sink, 4096);
  for (int r = 0; r < 2; ++r) {
    run<0>("rscalar", g, sink);
    run<1>("uconst", g, sink);
    run<2>("uredux", g, sink);
    run<3>("peak", g, sink);
  }
  return cudaGetLastError() != cudaSuccess;
}

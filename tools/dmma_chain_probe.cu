// dmma_chain_probe.cu -- DMMA.8x8x4 throughput per SM against the number of
// resident warps and independent accumulator chains per warp (registers
// only).  Tells how many chains the small-tile DMMA plans need in flight to
// fill the FP64 tensor pipe, and the latency of one dependent DMMA.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/dmma_chain_probe \
//        tools/dmma_chain_probe.cu && tools/dmma_chain_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

template <int CH>
__global__ void chain_kernel(int iters, double* sink, long long* cycles) {
  const double x = 1.0 + threadIdx.x * 1e-9, y = 1.0 - threadIdx.x * 1e-9;
  double d[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = 0.0;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], x, y);
  __syncthreads();
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.0) sink[threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int CH>
void run(int warps, double* sink, long long* cyc, int sms) {
  const int iters = 4096;
  chain_kernel<CH><<<sms, 32 * warps>>>(iters, sink, cyc);
  cudaDeviceSynchronize();
  long long h[1024];
  cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double dmma_per_clk = static_cast<double>(warps) * CH * iters / mx;
  printf("warps/SM %2d chains/warp %2d: %.3f DMMA/clk/SM (%.0f%% of 0.25), %.1f clk per dependent DMMA per warp\n",
         warps, CH, dmma_per_clk, dmma_per_clk / 0.25 * 100, static_cast<double>(mx) / iters);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink;
  long long* cyc;
  cudaMalloc(&sink, 1 << 16);
  cudaMalloc(&cyc, sizeof(long long) * 1024);
  for (int w : {1, 2, 4, 8, 16, 24, 32}) {
    run<1>(w, sink, cyc, sms);
    run<2>(w, sink, cyc, sms);
    run<4>(w, sink, cyc, sms);
    run<8>(w, sink, cyc, sms);
    run<16>(w, sink, cyc, sms);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}

// fp64_copipe_probe.cu -- do the FP64 tensor path (DMMA.8x8x4) and the FP64
// vector pipe (DFMA / DADD / DMUL) run concurrently on one SM, or do they
// share issue capacity?  Warps 0..3 of every CTA run a DMMA chain loop, warps
// 4..7 a vector loop; each half alone, then both together.  If the mixed
// run takes ~max of the halves the pipes are separate; ~sum means shared.
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/fp64_copipe_probe \
//        tools/fp64_copipe_probe.cu && tools/fp64_copipe_probe
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// VEC: 0 DFMA, 1 DADD, 2 DMUL+DADD, 3 FFMA2
template <int VEC>
__global__ void __launch_bounds__(256) mix_kernel(int it_mma, int it_vec, double* sink) {
  const int w = threadIdx.x >> 5;
  const double x = 1.0 + threadIdx.x * 1e-9, y = 1.0 - threadIdx.x * 1e-9;
  double s = 0;
  if (w < 4) {
    double d[8][2];
#pragma unroll
    for (int c = 0; c < 8; ++c) d[c][0] = d[c][1] = 0.0;
    for (int it = 0; it < it_mma; ++it)
#pragma unroll
      for (int c = 0; c < 8; ++c) dmma(d[c][0], d[c][1], x, y);
#pragma unroll
    for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
  } else if (VEC == 3) {
    unsigned long long d[8];
    const float xf = static_cast<float>(x), yf = static_cast<float>(y);
    unsigned long long xx, yy;
    asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(xf));
    asm("mov.b64 %0, {%1, %1};" : "=l"(yy) : "f"(yf));
#pragma unroll
    for (int c = 0; c < 8; ++c) d[c] = static_cast<unsigned long long>(c);
    for (int it = 0; it < it_vec; ++it)
#pragma unroll
      for (int c = 0; c < 8; ++c)
        asm volatile("fma.rn.f32x2 %0, %1, %0, %2;" : "+l"(d[c]) : "l"(xx), "l"(yy));
    unsigned long long t = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) t ^= d[c];
    s = static_cast<double>(t);
  } else {
    double d[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) d[c] = c;
    for (int it = 0; it < it_vec; ++it)
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        if (VEC == 0) d[c] = fma(x, d[c], y);
        else if (VEC == 1) d[c] = __dadd_rn(d[c], y);
        else d[c] = __dadd_rn(__dmul_rn(x, d[c]), y);
      }
#pragma unroll
    for (int c = 0; c < 8; ++c) s += d[c];
  }
  if (s == 12345.0) sink[threadIdx.x] = s;
}

template <int VEC>
float run(int it_mma, int it_vec, double* sink, int sms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  mix_kernel<VEC><<<sms * 4, 256>>>(it_mma, it_vec, sink);  // warm-up
  cudaEventRecord(e0);
  mix_kernel<VEC><<<sms * 4, 256>>>(it_mma, it_vec, sink);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

template <int VEC>
void trial(const char* name, int it_mma, int sms, double* sink) {
  // pick it_vec so that the vector half alone takes as long as the DMMA half
  const float tm = run<VEC>(it_mma, 0, sink, sms);
  const float tv1 = run<VEC>(0, it_mma, sink, sms);
  int it_vec = static_cast<int>(it_mma * (tm / tv1));
  const float tv = run<VEC>(0, it_vec, sink, sms);
  const float tb = run<VEC>(it_mma, it_vec, sink, sms);
  // flops: DMMA 8 per warp-iter x 512; vector per thread-iter 8 x (2 or 1 or 2 or 4)
  const double warps = sms * 4.0 * 4;
  const double f_mma = warps * it_mma * 8 * 512.0;
  const double per = VEC == 0 ? 2 : VEC == 1 ? 1 : VEC == 2 ? 2 : 4;
  const double f_vec = warps * 32 * static_cast<double>(it_vec) * 8 * per;
  printf("%-10s dmma alone %.3f ms (%.1f TF)  vec alone %.3f ms (%.1f TF)  both %.3f ms "
         "(%.1f TF total)  both/max(alone) = %.2f\n",
         name, tm, f_mma / tm / 1e9, tv, f_vec / tv / 1e9, tb, (f_mma + f_vec) / tb / 1e9,
         tb / (tm > tv ? tm : tv));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* sink;
  cudaMalloc(&sink, 4096);
  const int it = 20000;
  trial<0>("DFMA", it, sms, sink);
  trial<1>("DADD", it, sms, sink);
  trial<2>("DMUL+DADD", it, sms, sink);
  trial<3>("FFMA2", it, sms, sink);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}

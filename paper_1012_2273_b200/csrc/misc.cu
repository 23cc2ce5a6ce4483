// misc.cu -- device-side helpers: input generators, padded packing, and the
// FP64/FP32 pipe peak probes used as roofline denominators.
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace mmws_impl {
namespace {

// ---------------------------------------------------------------- generators
// Element i (row-major flat index over the logical rows x cols matrix, plus
// `first`) is splitmix64's (i+1)-th output for `seed` -- the reference's
// random_matrix stream (include/mmws/matrix.hpp:23-33, 101-107) evaluated
// counter-style.  dist 0..2 are integer-exact and bit-identical to the host
// oracle; dist 3 (normal, Box-Muller in double) uses device libm and is
// therefore generated once on the device and copied to the host when the
// oracle needs it.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t draw(uint64_t seed, uint64_t i) {
  return mix64(seed + (i + 1) * 0x9E3779B97F4A7C15ULL);
}

__global__ void fill_kernel(int dist, uint64_t seed, void* dst, int64_t rows, int64_t cols,
                            int64_t ld, int is_f32, uint64_t first) {
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / cols, c = e % cols;
    const uint64_t i = first + static_cast<uint64_t>(e);
    double x;
    if (dist == 3) {
      const double u1 = static_cast<double>(draw(seed, 2 * i) >> 11) * 0x1.0p-53;
      const double u2 = static_cast<double>(draw(seed, 2 * i + 1) >> 11) * 0x1.0p-53;
      x = sqrt(-2.0 * log(1.0 - u1)) * cos(6.283185307179586 * u2);
    } else {
      const uint64_t m = draw(seed, i) >> 11;
      if (dist == 0) x = static_cast<double>(m) * 0x1.0p-53;
      else if (dist == 1) x = 2.0 * (static_cast<double>(m) * 0x1.0p-53) - 1.0;
      else x = static_cast<double>(static_cast<int64_t>((m * 17ULL) >> 53) - 8);
    }
    if (is_f32) static_cast<float*>(dst)[r * ld + c] = static_cast<float>(x);
    else static_cast<double*>(dst)[r * ld + c] = x;
  }
}

// ---------------------------------------------------------------- progress board
// One progress word of the row-block failure detector (rowblock.cu), stored
// from this GPU into rank 0's board -- local memory on rank 0, a CUDA IPC
// mapping over NVLink on the workers -- in stream order.
__global__ void board_mark_kernel(volatile unsigned* word, unsigned value) {
  *word = value;
  __threadfence_system();
}

// ---------------------------------------------------------------- packing
// One CTA row-strip per (row, 1024-column chunk): no 64-bit division per
// element, coalesced reads and writes.
template <class T>
__global__ void pack_kernel(const T* __restrict__ src, int64_t rows, int64_t cols, int64_t ld_src,
                            T* __restrict__ dst, int64_t rows_p, int64_t cols_p, int64_t ld_dst) {
  for (int64_t r = blockIdx.y; r < rows_p; r += gridDim.y) {
    const T* s = src + r * ld_src;
    T* d = dst + r * ld_dst;
    for (int64_t c = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; c < cols_p;
         c += static_cast<int64_t>(gridDim.x) * blockDim.x)
      d[c] = (r < rows && c < cols) ? s[c] : T(0);
  }
}

template <class T>
cudaError_t launch_pack(const Launch& L, const T* src, int64_t rows, int64_t cols, int64_t ld_src,
                        T* dst, int64_t rows_p, int64_t cols_p, int64_t ld_dst) {
  const dim3 grid(static_cast<unsigned>((cols_p + 255) / 256 < 8 ? (cols_p + 255) / 256 : 8),
                  static_cast<unsigned>(rows_p < 65535 ? rows_p : 65535));
  pack_kernel<T><<<grid, 256, 0, L.stream>>>(src, rows, cols, ld_src, dst, rows_p, cols_p, ld_dst);
  L.count();
  return cudaGetLastError();
}

// ---------------------------------------------------------------- FFMA2 outer-product probe
// The fp32 GEMM kernel's operand pattern in registers only (sgemm_tma.cu):
// 8 warps per SM, 64 accumulator pairs per lane, B pairs reused across 8
// consecutive FFMA2, the broadcast A scalar fresh from the register file each
// time.  One loop of that pattern, not a ceiling: such loops measure 56-71
// TFLOP/s depending on block shape and register assignment, and the kernel
// with A staged k-major runs above this one.
__global__ void __launch_bounds__(256, 1) ffma2_outer_probe_kernel(int iters, double* sink) {
  typedef unsigned long long u64;
  auto pk = [](float a, float b) {
    u64 r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
  };
  const float seed = 1.0f + threadIdx.x * 1e-7f;
  u64 b[8], d[8][8];
  float ar[8];
#pragma unroll
  for (int p = 0; p < 8; ++p) b[p] = pk(seed * (0.5f + p), seed * (1.25f + p) + 0.375f);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    ar[i] = seed * (2.0625f + 0.1875f * i) - 3.0f;  // distinct from every B element
#pragma unroll
    for (int p = 0; p < 8; ++p) d[i][p] = 0;
  }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int p = 0; p < 8; ++p)
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d[i][p]) : "l"(b[p]), "l"(pk(ar[i], ar[i])));
  u64 x = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int p = 0; p < 8; ++p) x ^= d[i][p];
  if (x == 12345ull) sink[threadIdx.x] = static_cast<double>(x);
}

// ---------------------------------------------------------------- peak probes
// 0: DMMA.8x8x4 (FP64 tensor)  1: DFMA  2: DMUL+DADD  3: FFMA (fp32)  4: FFMA2 (fp32x2)
template <int WHICH>
__global__ void __launch_bounds__(256) probe_kernel(int iters, double* sink) {
  const double x = 1.0 + threadIdx.x * 1e-9, y = 1.0 - threadIdx.x * 1e-9;
  if (WHICH == 0) {
    double d[8][2];
#pragma unroll
    for (int c = 0; c < 8; ++c) d[c][0] = d[c][1] = 0.0;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int c = 0; c < 8; ++c) mmws_dev::dmma_8x8x4(d[c][0], d[c][1], x, y);
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += d[c][0] + d[c][1];
    if (s == 12345.0) sink[threadIdx.x] = s;
  } else if (WHICH == 1 || WHICH == 2) {
    double d[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) d[c] = c;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int c = 0; c < 8; ++c)
        d[c] = WHICH == 1 ? fma(x, d[c], y) : __dadd_rn(__dmul_rn(x, d[c]), y);
    double s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s += d[c];
    if (s == 12345.0) sink[threadIdx.x] = s;
  } else if (WHICH == 4) {
    unsigned long long d[8];
    const float xf = static_cast<float>(x), yf = static_cast<float>(y);
    unsigned long long xx, yy;
    asm("mov.b64 %0, {%1, %1};" : "=l"(xx) : "f"(xf));
    asm("mov.b64 %0, {%1, %1};" : "=l"(yy) : "f"(yf));
#pragma unroll
    for (int c = 0; c < 8; ++c) d[c] = static_cast<unsigned long long>(c);
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int c = 0; c < 8; ++c) asm volatile("fma.rn.f32x2 %0, %1, %0, %2;" : "+l"(d[c]) : "l"(xx), "l"(yy));
    unsigned long long s = 0;
#pragma unroll
    for (int c = 0; c < 8; ++c) s ^= d[c];
    if (s == 12345ull) sink[threadIdx.x] = static_cast<double>(s);
  } else {
    float d[16];
    const float xf = static_cast<float>(x), yf = static_cast<float>(y);
#pragma unroll
    for (int c = 0; c < 16; ++c) d[c] = c;
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int c = 0; c < 16; ++c) d[c] = fmaf(xf, d[c], yf);
    float s = 0;
#pragma unroll
    for (int c = 0; c < 16; ++c) s += d[c];
    if (s == 12345.f) sink[threadIdx.x] = s;
  }
}

int grid_for(const Launch& L, int64_t total) {
  const int64_t want = (total + 255) / 256;
  const int64_t cap = static_cast<int64_t>(L.num_sms) * 16;
  return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

}  // namespace

cudaError_t launch_fill(const Launch& L, int dist, uint64_t seed, void* dst, int64_t rows,
                        int64_t cols, int64_t ld, int is_f32, uint64_t first) {
  fill_kernel<<<grid_for(L, rows * cols), 256, 0, L.stream>>>(dist, seed, dst, rows, cols, ld,
                                                               is_f32, first);
  L.count();
  return cudaGetLastError();
}

cudaError_t launch_pack_f64(const Launch& L, const double* src, int64_t rows, int64_t cols,
                            int64_t ld_src, double* dst, int64_t rows_p, int64_t cols_p,
                            int64_t ld_dst) {
  return launch_pack(L, src, rows, cols, ld_src, dst, rows_p, cols_p, ld_dst);
}

cudaError_t launch_pack_f32(const Launch& L, const float* src, int64_t rows, int64_t cols,
                            int64_t ld_src, float* dst, int64_t rows_p, int64_t cols_p,
                            int64_t ld_dst) {
  return launch_pack(L, src, rows, cols, ld_src, dst, rows_p, cols_p, ld_dst);
}

cudaError_t launch_peak_probe(const Launch& L, int which, int iters, double* sink,
                              double* flops) {
  const int blocks = L.num_sms * 8, threads = 256;
  const double thr = static_cast<double>(blocks) * threads;
  switch (which) {
    case 0:
      probe_kernel<0><<<blocks, threads, 0, L.stream>>>(iters, sink);
      *flops = thr / 32.0 * 8.0 * iters * 512.0;  // 8 DMMA (256 FMA) per warp-iter
      break;
    case 1:
      probe_kernel<1><<<blocks, threads, 0, L.stream>>>(iters, sink);
      *flops = thr * 8.0 * iters * 2.0;
      break;
    case 2:
      probe_kernel<2><<<blocks, threads, 0, L.stream>>>(iters, sink);
      *flops = thr * 8.0 * iters * 2.0;
      break;
    case 3:
      probe_kernel<3><<<blocks, threads, 0, L.stream>>>(iters, sink);
      *flops = thr * 16.0 * iters * 2.0;
      break;
    case 4:
      probe_kernel<4><<<blocks, threads, 0, L.stream>>>(iters, sink);
      *flops = thr * 8.0 * iters * 4.0;  // 8 chains x 2 lanes x 2 flops
      break;
    default:  // 5: the fp32 GEMM's FFMA2 operand pattern, one 8-warp CTA per SM
      ffma2_outer_probe_kernel<<<L.num_sms, 256, 0, L.stream>>>(iters, sink);
      *flops = static_cast<double>(L.num_sms) * 256 * 64.0 * iters * 4.0;
      break;
  }
  L.count();
  return cudaGetLastError();
}

cudaError_t launch_board_mark(const Launch& L, unsigned* word, unsigned value) {
  board_mark_kernel<<<1, 1, 0, L.stream>>>(word, value);
  L.count();
  return cudaGetLastError();
}

cudaError_t preload_misc() {
  return preload_kernels(fill_kernel, pack_kernel<double>, pack_kernel<float>, board_mark_kernel,
                         ffma2_outer_probe_kernel, probe_kernel<0>, probe_kernel<1>,
                         probe_kernel<2>, probe_kernel<3>, probe_kernel<4>);
}

}  // namespace mmws_impl

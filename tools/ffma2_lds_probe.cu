// Development probe: the sgemm_tma.cu math loop (FFMA2 outer product fed by
// LDS.128 from a 4-stage [128x16] A / [16x256] B shared-memory ring) without
// TMA or barriers, for the per-lane blocks 8x8 pairs (RI = 8) and 4x16 pairs
// (RI = 4).  FEED: 0 registers only, 1 B from shared memory, 2 A from shared
// memory, 3 both (the kernel's loop), 7 both with A staged k-major ([16 k][128
// rows]: one LDS.128 = four rows at one k, so a row's A scalar sits in the same
// register bank for every k).  Shows which operand feed costs what
// against the register-only rate of the same block.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/ffma2_lds_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1,%2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void f2(u64& d, u64 a, u64 b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
constexpr int BM = 128, BN = 256, BK = 16, STAGES = 4;
constexpr int STAGE_FLOATS = BM * BK + BK * BN;

template <int RI, int FEED>
__global__ void __launch_bounds__(256, 1) k(int iters, float* sink, float seed) {
  extern __shared__ __align__(128) float sm[];
  for (int i = threadIdx.x; i < STAGES * STAGE_FLOATS; i += 256) sm[i] = seed * (i & 15);
  __syncthreads();
  constexpr int NJ = 32 / RI, CG = 64 / NJ, RG = 32 / CG, CSTR = 4 * CG;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane / CG, c = lane % CG;
  const int row_base = warp * 16 + g;
  u64 part[RI][2 * NJ];
#pragma unroll
  for (int i = 0; i < RI; ++i)
#pragma unroll
    for (int p = 0; p < 2 * NJ; ++p) part[i][p] = 0;
  float4 areg[RI];
  u64 breg[2 * NJ];
#pragma unroll
  for (int i = 0; i < RI; ++i) areg[i] = make_float4(seed + i, seed * i, seed - i, seed + 2 * i);
#pragma unroll
  for (int p = 0; p < 2 * NJ; ++p) breg[p] = pk(seed * p + threadIdx.x, seed + p);
  for (int kt = 0; kt < iters; ++kt) {
    const float* as = sm + (kt % STAGES) * STAGE_FLOATS;
    const float* bs = as + BM * BK;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      float4 a4[RI];
#pragma unroll
      for (int i = 0; i < RI; ++i)
        a4[i] = (FEED & 2) ? *reinterpret_cast<const float4*>(as + (row_base + i * RG) * BK + k4)
                           : areg[i];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        float4 at[RI / 4];  // k-major A: rows warp*16 + g*RI + 4q .. +3 at k = k4 + kk
        if (FEED & 4) {
#pragma unroll
          for (int q = 0; q < RI / 4; ++q)
            at[q] = *reinterpret_cast<const float4*>(as + (k4 + kk) * BM + warp * 16 + g * RI + 4 * q);
        }
        u64 b2[2 * NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          if (FEED & 1) {
            const float4 b =
                *reinterpret_cast<const float4*>(bs + (k4 + kk) * BN + c * 4 + CSTR * j);
            b2[2 * j] = pk(b.x, b.y);
            b2[2 * j + 1] = pk(b.z, b.w);
          } else {
            b2[2 * j] = breg[2 * j];
            b2[2 * j + 1] = breg[2 * j + 1];
          }
        }
#pragma unroll
        for (int p = 0; p < 2 * NJ; ++p)
#pragma unroll
          for (int i = 0; i < RI; ++i) {
            float a = kk == 0 ? a4[i].x : kk == 1 ? a4[i].y : kk == 2 ? a4[i].z : a4[i].w;
            if (FEED & 4) {
              const float4 t = at[i / 4];
              a = (i & 3) == 0 ? t.x : (i & 3) == 1 ? t.y : (i & 3) == 2 ? t.z : t.w;
            }
            f2(part[i][p], b2[p], pk(a, a));
          }
      }
    }
  }
  u64 s = 0;
#pragma unroll
  for (int i = 0; i < RI; ++i)
#pragma unroll
    for (int p = 0; p < 2 * NJ; ++p) s ^= part[i][p];
  if (s == 42) sink[threadIdx.x] = (float)s;
}

template <int RI, int FEED>
void run(float* sink) {
  const int iters = 4000, blocks = 148, smem = STAGES * STAGE_FLOATS * 4;
  cudaFuncSetAttribute(k<RI, FEED>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<RI, FEED><<<blocks, 256, smem>>>(10, sink, 1.0f);
  cudaEventRecord(e0);
  k<RI, FEED><<<blocks, 256, smem>>>(iters, sink, 1.0f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = double(blocks) * 256 * iters * BK * 64 * 4;
  std::printf("block %dx%d pairs  feed %s  %.1f TFLOP/s\n", RI, 64 / RI,
              FEED == 0 ? "registers" : FEED == 1 ? "B from smem" : FEED == 2 ? "A from smem"
              : FEED == 3 ? "A and B from smem" : FEED == 4 ? "A k-major from smem"
                                                              : "A k-major and B from smem",
              flops / ms / 1e9);
}

int main() {
  float* sink;
  cudaMalloc(&sink, 4096);
  for (int r = 0; r < 2; ++r) {
    run<8, 0>(sink);
    run<8, 1>(sink);
    run<8, 2>(sink);
    run<8, 3>(sink);
    run<8, 4>(sink);
    run<8, 5>(sink);
    run<4, 0>(sink);
    run<4, 1>(sink);
    run<4, 2>(sink);
    run<4, 3>(sink);
    run<4, 4>(sink);
    run<4, 5>(sink);
    std::printf("\n");
  }
  return cudaGetLastError() != cudaSuccess;
}

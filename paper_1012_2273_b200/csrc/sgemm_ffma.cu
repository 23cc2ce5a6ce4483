// sgemm_ffma.cu -- register-blocked FP32 GEMM on the FFMA pipe.
//
// The fp32 configuration (BASELINE.json configs[4], N=32768 normal(0,1)) has
// no counterpart in the reference (its Matrix is fp64 only, matrix.hpp:39-91);
// this is the same C = A.B contraction in fp32, checked normwise against the
// fp64 oracle of the widened inputs (tolerance 1e-5, tests/test_gpu_parity.py).
//
// 192x128 CTA tile, 384 threads (12 warps, 1 CTA/SM, <= 168 registers each),
// 8x8 outputs per thread (rows 4*ty + 96v + h, cols 4*tx + 64v + h) held as
// packed fp32 pairs and updated with Blackwell's FFMA2 (two multiply-adds per
// instruction; the A value is the instruction's broadcast operand).  A and B
// k-tiles (16 wide) stream through a 3-stage cp.async ring in natural layout;
// a lane fetches A as (k, k+1) pairs of one row (broadcast LDS.64) and B as
// 4-column vectors (conflict-free LDS.128).
//
// Accuracy: a single fp32 chain over K = 32768 terms has an expected normwise
// error of ~5e-6, uncomfortably close to the 1e-5 bound.  The
// kernel therefore sums each KC-long k-chunk into a fresh register partial and
// adds the partial into a running total kept in shared memory (96 KB: 64
// floats per thread) once per chunk -- two-level (blocked) summation, error
// growth ~sqrt(KC) + sqrt(K / KC) instead of ~sqrt(K), for ~1% extra
// instructions and without doubling the accumulator registers.
#include "common.cuh"
#include "kernels.h"

namespace mmws_impl {
namespace {

using namespace mmws_dev;

// Packed fp32 pairs (FFMA2): ptxas folds a {x, x} pair of a scalar into the
// instruction's broadcast operand, so no MOV is emitted.
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 pack2(float lo, float hi) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 unpack2(f32x2 v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ void ffma2(f32x2& d, f32x2 a, f32x2 b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}

constexpr int BM = 192, BN = 128, BK = 16, THREADS = 384, STAGES = 3;
constexpr int RSTEP = BM / 2;  // row stride between a thread's two 4-row groups
constexpr int KC_TILES = 64;  // partial-sum chunk = 64 k-tiles = 1024 k (as sgemm_tma.cu)
constexpr int SLA = BK + 4;   // A row pitch (floats)
constexpr int SLB = BN;       // B row pitch
constexpr int A_ELEMS = BM * SLA, B_ELEMS = BK * SLB;
constexpr int TOT_FLOATS = THREADS * 64;
constexpr int SMEM = (STAGES * (A_ELEMS + B_ELEMS) + TOT_FLOATS) * sizeof(float);

template <bool VA, bool VB>
__global__ void __launch_bounds__(THREADS, 1)
    sgemm_ffma_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ B,
                      int64_t ldb, float* __restrict__ C, int64_t ldc, int M, int N, int K,
                      int tiles_m, int tiles_n, int vec_c) {
  extern __shared__ __align__(16) float smem_f[];
  float* As = smem_f;                               // [STAGES][BM][SLA]
  float* Bs = smem_f + STAGES * A_ELEMS;            // [STAGES][BK][SLB]
  float4* tot = reinterpret_cast<float4*>(Bs + STAGES * B_ELEMS);  // [16][THREADS]

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  // grouped rasterisation over 8 tile-rows (L2 reuse of the B panels)
  constexpr int GROUP = 8;
  const int tile = blockIdx.x;
  const int per_group = GROUP * tiles_n;
  const int first_m = (tile / per_group) * GROUP;
  const int gm = min(tiles_m - first_m, GROUP);
  const int tm = first_m + (tile % per_group) % gm;
  const int tn = (tile % per_group) / gm;
  const int row0 = tm * BM, col0 = tn * BN;
  const int KT = (K + BK - 1) / BK;

  auto load_stage = [&](int kt) {
    const int s = kt % STAGES;
    load_tile_async<float, BM, BK, SLA, THREADS, VA>(As + s * A_ELEMS, A, lda, row0, kt * BK, M, K);
    load_tile_async<float, BK, BN, SLB, THREADS, VB>(Bs + s * B_ELEMS, B, ldb, kt * BK, col0, K, N);
  };

#pragma unroll
  for (int q = 0; q < 16; ++q) tot[q * THREADS + tid] = make_float4(0.f, 0.f, 0.f, 0.f);

  // part[i][p]: columns (2p, 2p+1) of row i of the thread's 8x8 block
  f32x2 part[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int p = 0; p < 4; ++p) part[i][p] = 0ull;

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s);
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    if (kt + STAGES - 1 < KT) load_stage(kt + STAGES - 1);
    cp_async_commit();
    const float* as = As + (kt % STAGES) * A_ELEMS;
    const float* bs = Bs + (kt % STAGES) * B_ELEMS;
#pragma unroll
    for (int k = 0; k < BK; k += 2) {
      float2 a2[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        a2[i] = *reinterpret_cast<const float2*>(as + (ty * 4 + RSTEP * (i >> 2) + (i & 3)) * SLA + k);
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        const float4 b0 = *reinterpret_cast<const float4*>(bs + (k + kk) * SLB + tx * 4);
        const float4 b1 = *reinterpret_cast<const float4*>(bs + (k + kk) * SLB + tx * 4 + 64);
        const f32x2 b2[4] = {pack2(b0.x, b0.y), pack2(b0.z, b0.w), pack2(b1.x, b1.y),
                             pack2(b1.z, b1.w)};
        // p outer / i inner: consecutive FFMA2s share the B pair (operand
        // reuse cache), so each reads only the broadcast A value and the
        // accumulator pair from the register file
#pragma unroll
        for (int p = 0; p < 4; ++p)
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float a = kk ? a2[i].y : a2[i].x;
            ffma2(part[i][p], pack2(a, a), b2[p]);
          }
      }
    }
    if ((kt % KC_TILES) == KC_TILES - 1 || kt + 1 == KT) {
      // fold the chunk partial into the shared-memory running total
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int i = q >> 1, p = (q & 1) * 2;
        float4 t = tot[q * THREADS + tid];
        const float2 lo = unpack2(part[i][p]), hi = unpack2(part[i][p + 1]);
        t.x += lo.x;
        t.y += lo.y;
        t.z += hi.x;
        t.w += hi.y;
        tot[q * THREADS + tid] = t;
        part[i][p] = part[i][p + 1] = 0ull;
      }
    }
  }

#pragma unroll
  for (int q = 0; q < 16; ++q) {
    const int i = q >> 1, h = q & 1;
    const int r = row0 + ty * 4 + RSTEP * (i >> 2) + (i & 3);
    if (r >= M) continue;
    const int c = col0 + tx * 4 + 64 * h;
    const float4 v = tot[q * THREADS + tid];
    float* crow = C + static_cast<int64_t>(r) * ldc;
    if (vec_c && c + 3 < N) {
      *reinterpret_cast<float4*>(crow + c) = v;
    } else {
      const float w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if (c + j < N) crow[c + j] = w[j];
    }
  }
}

}  // namespace

cudaError_t launch_sgemm_ffma(const Launch& L, int64_t M, int64_t N, int64_t K, const float* A,
                              int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc) {
  const int tiles_m = static_cast<int>((M + BM - 1) / BM);
  const int tiles_n = static_cast<int>((N + BN - 1) / BN);
  // 16-byte cp.async when a whole chunk is always in or out of the matrix
  const bool va = lda % 4 == 0 && K % 4 == 0 && reinterpret_cast<uintptr_t>(A) % 16 == 0;
  const bool vb = ldb % 4 == 0 && N % 4 == 0 && reinterpret_cast<uintptr_t>(B) % 16 == 0;
  const int vec_c = (ldc % 4 == 0) && (reinterpret_cast<uintptr_t>(C) % 16 == 0);
  auto kern = va ? (vb ? sgemm_ffma_kernel<true, true> : sgemm_ffma_kernel<true, false>)
                 : (vb ? sgemm_ffma_kernel<false, true> : sgemm_ffma_kernel<false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  if (e != cudaSuccess) return e;
  kern<<<tiles_m * tiles_n, THREADS, SMEM, L.stream>>>(A, lda, B, ldb, C, ldc,
                                                       static_cast<int>(M), static_cast<int>(N),
                                                       static_cast<int>(K), tiles_m, tiles_n,
                                                       vec_c);
  L.count();
  return cudaGetLastError();
}

cudaError_t preload_sgemm() {
  return preload_kernels(sgemm_ffma_kernel<true, true>, sgemm_ffma_kernel<true, false>,
                         sgemm_ffma_kernel<false, true>, sgemm_ffma_kernel<false, false>);
}

}  // namespace mmws_impl

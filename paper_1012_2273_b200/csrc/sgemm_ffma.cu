// sgemm_ffma.cu -- register-blocked FP32 GEMM on the FFMA pipe.
//
// The fp32 configuration (BASELINE.json configs[4], N=32768 normal(0,1)) has
// no counterpart in the reference (its Matrix is fp64 only, matrix.hpp:39-91);
// this is the same C = A.B contraction in fp32, checked normwise against the
// fp64 oracle of the widened inputs (tolerance 1e-5, tests/test_gpu_parity.py).
//
// 128x128 CTA tile, 256 threads, 8x8 outputs per thread (rows 4*ty + 64v + h,
// cols 4*tx + 64v + h so fragment fetches are 128-bit broadcast / conflict-free
// LDS) held as packed fp32 pairs and updated with FFMA2 (the a-value is the
// broadcast operand), A staged k-major (transposed) in shared memory,
// global->register->shared double buffering over 8-wide k-tiles.
//
// Accuracy: a single fp32 chain over K = 32768 terms has an expected normwise
// error of ~5e-6, uncomfortably close to the 1e-5 bound.  The
// kernel therefore sums each KC-long k-chunk into a fresh partial and adds the
// partial into the running total once per chunk (two-level / blocked
// summation), which shrinks the error growth from ~sqrt(K) to
// ~sqrt(KC) + sqrt(K / KC) for one extra FADD per KC FFMAs.
#include "common.cuh"
#include "kernels.h"

// Packed fp32 pairs (Blackwell FFMA2 / FADD2): one instruction does two
// multiply-adds, halving issue pressure; ptxas folds a {x, x} pair of a scalar
// into the instruction's broadcast operand (no MOV).
#define MMWS_F2 unsigned long long
__device__ __forceinline__ MMWS_F2 pack2(float lo, float hi) {
  MMWS_F2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float2 unpack2(MMWS_F2 v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ void ffma2(MMWS_F2& d, MMWS_F2 a, MMWS_F2 b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
__device__ __forceinline__ void fadd2(MMWS_F2& d, MMWS_F2 a) {
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(d) : "l"(a));
}

namespace mmws_impl {
namespace {

constexpr int BM = 128, BN = 128, BK = 8, THREADS = 256;
constexpr int KC_TILES = 16;  // partial-sum chunk = 16 k-tiles = 128 k
constexpr int LDA_S = BM + 4;

__global__ void __launch_bounds__(THREADS, 1)
    sgemm_ffma_kernel(const float* __restrict__ A, int64_t lda, const float* __restrict__ B,
                      int64_t ldb, float* __restrict__ C, int64_t ldc, int M, int N, int K,
                      int tiles_m, int tiles_n, int vec_a, int vec_b, int vec_c) {
  __shared__ __align__(16) float As[2][BK][LDA_S];
  __shared__ __align__(16) float Bs[2][BK][BN];

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

  const int a_r = tid >> 1, a_k = (tid & 1) * 4;   // A: row a_r, k a_k .. a_k+3
  const int b_k = tid >> 5, b_c = (tid & 31) * 4;  // B: k-row b_k, cols b_c .. b_c+3
  const bool a_row_ok = row0 + a_r < M;
  const float* a_src = A + static_cast<int64_t>(row0 + a_r) * lda;

  float ra[4], rb[4];
  auto load_tile = [&](int kt) {
    const int k0 = kt * BK;
    const int ka = k0 + a_k;
    if (vec_a && a_row_ok && ka + 3 < K) {
      const float4 v = *reinterpret_cast<const float4*>(a_src + ka);
      ra[0] = v.x; ra[1] = v.y; ra[2] = v.z; ra[3] = v.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) ra[j] = (a_row_ok && ka + j < K) ? a_src[ka + j] : 0.f;
    }
    const int kb = k0 + b_k;
    const float* b_src = B + static_cast<int64_t>(kb) * ldb + col0 + b_c;
    if (vec_b && kb < K && col0 + b_c + 3 < N) {
      const float4 v = *reinterpret_cast<const float4*>(b_src);
      rb[0] = v.x; rb[1] = v.y; rb[2] = v.z; rb[3] = v.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) rb[j] = (kb < K && col0 + b_c + j < N) ? b_src[j] : 0.f;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int j = 0; j < 4; ++j) As[buf][a_k + j][a_r] = ra[j];
    *reinterpret_cast<float4*>(&Bs[buf][b_k][b_c]) = make_float4(rb[0], rb[1], rb[2], rb[3]);
  };

  // acc[i][p] holds columns (2p, 2p+1) of row i of the thread's 8x8 block
  MMWS_F2 acc[8][4], part[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int p = 0; p < 4; ++p) acc[i][p] = part[i][p] = 0ull;

  const int KT = (K + BK - 1) / BK;
  load_tile(0);
  store_tile(0);
  __syncthreads();

  for (int kt = 0; kt < KT; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < KT) load_tile(kt + 1);
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4 + 64]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4 + 64]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      const MMWS_F2 b2[4] = {pack2(b0.x, b0.y), pack2(b0.z, b0.w), pack2(b1.x, b1.y),
                             pack2(b1.z, b1.w)};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const MMWS_F2 aa = pack2(a[i], a[i]);
#pragma unroll
        for (int p = 0; p < 4; ++p) ffma2(part[i][p], aa, b2[p]);
      }
    }
    if ((kt % KC_TILES) == KC_TILES - 1 || kt + 1 == KT) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int p = 0; p < 4; ++p) {
          fadd2(acc[i][p], part[i][p]);
          part[i][p] = 0ull;
        }
    }
    if (kt + 1 < KT) store_tile(buf ^ 1);
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = row0 + ty * 4 + 64 * (i >> 2) + (i & 3);
    if (r >= M) continue;
    float* crow = C + static_cast<int64_t>(r) * ldc;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = col0 + tx * 4 + 64 * h;
      const float2 lo = unpack2(acc[i][2 * h]), hi = unpack2(acc[i][2 * h + 1]);
      const float v[4] = {lo.x, lo.y, hi.x, hi.y};
      if (vec_c && c + 3 < N) {
        *reinterpret_cast<float4*>(crow + c) = make_float4(v[0], v[1], v[2], v[3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (c + j < N) crow[c + j] = v[j];
      }
    }
  }
}

}  // namespace

cudaError_t launch_sgemm_ffma(const Launch& L, int64_t M, int64_t N, int64_t K, const float* A,
                              int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc) {
  const int tiles_m = static_cast<int>((M + BM - 1) / BM);
  const int tiles_n = static_cast<int>((N + BN - 1) / BN);
  const int vec_a = (lda % 4 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0);
  const int vec_b = (ldb % 4 == 0) && (reinterpret_cast<uintptr_t>(B) % 16 == 0);
  const int vec_c = (ldc % 4 == 0) && (reinterpret_cast<uintptr_t>(C) % 16 == 0);
  sgemm_ffma_kernel<<<tiles_m * tiles_n, THREADS, 0, L.stream>>>(
      A, lda, B, ldb, C, ldc, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K),
      tiles_m, tiles_n, vec_a, vec_b, vec_c);
  L.count();
  return cudaGetLastError();
}

}  // namespace mmws_impl

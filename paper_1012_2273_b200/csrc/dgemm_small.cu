// dgemm_small.cu -- latency path for small fp64 problems (the paper's N = 10 ..
// ~250 range, and the exact mode up to N ~ 1500).
//
// At these sizes the multiply is a few microseconds of work spread over a
// handful of SMs: what matters is how fast one CTA gets its first operands and
// how many SMs share the work, not tensor-pipe throughput (a 128x128 DMMA or
// exact-order tile would leave >90% of the 148 SMs idle and pays TMA
// descriptor / mbarrier set-up).  One CTA per 32x32 output tile, 256 threads
// with a 2x2 register block each, plain coalesced loads double-buffered
// through registers into shared memory, no TMA, no dynamic shared memory.
//
// EXACT: acc = +0.0; acc = RN(acc + RN(a*b)) for k ascending -- bitwise the
// reference's matmul_seq chain (matrix.hpp:118-124), like dgemm_exact.cu.
// !EXACT: the same chain with a fused multiply-add (one rounding per step);
// normwise error far below the 1e-12 bound.  Either way each output element's
// arithmetic depends only on its row of A and column of B, never on the tile
// or grid shape.
#include "common.cuh"
#include "kernels.h"

namespace mmws_impl {
namespace {

constexpr int T = 32, BK = 32, THREADS = 256;

template <bool EXACT>
__global__ void __launch_bounds__(THREADS)
    dgemm_small_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                       int64_t ldb, double* C, int64_t ldc, int M, int N, int K,
                       int tiles_n, const double* cin, int64_t ldcin) {
  __shared__ __align__(16) double As[2][T][BK + 1];  // [row][k], +1 spreads the row starts
  __shared__ __align__(16) double Bs[2][BK][T];      // [k][col]

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int row0 = (blockIdx.x / tiles_n) * T, col0 = (blockIdx.x % tiles_n) * T;
  // staging: 4 consecutive elements of one row per thread for each operand
  const int lr = tid >> 3, lc = (tid & 7) * 4;

  double ra[4], rb[4];
  auto load = [&](int k0) {
    const int ar = row0 + lr;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int k = k0 + lc + j;
      ra[j] = (ar < M && k < K) ? A[static_cast<int64_t>(ar) * lda + k] : 0.0;
    }
    const int bk = k0 + lr;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = col0 + lc + j;
      rb[j] = (bk < K && c < N) ? B[static_cast<int64_t>(bk) * ldb + c] : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int j = 0; j < 4; ++j) As[buf][lr][lc + j] = ra[j];
#pragma unroll
    for (int j = 0; j < 4; ++j) Bs[buf][lr][lc + j] = rb[j];
  };

  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  if (cin) {  // accumulate: continue Cin's chains (Cin may alias C)
#pragma unroll
    for (int h = 0; h < 2; ++h)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = row0 + ty * 2 + h, c = col0 + tx * 2 + e;
        if (r < M && c < N) acc[h][e] = cin[static_cast<int64_t>(r) * ldcin + c];
      }
  }
  const int KT = (K + BK - 1) / BK;
  load(0);
  store(0);
  __syncthreads();
  for (int kt = 0; kt < KT; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < KT) load((kt + 1) * BK);
#pragma unroll 8
    for (int k = 0; k < BK; ++k) {
      const double a0 = As[buf][ty * 2][k], a1 = As[buf][ty * 2 + 1][k];
      const double2 b = *reinterpret_cast<const double2*>(&Bs[buf][k][tx * 2]);
      if constexpr (EXACT) {
        acc[0][0] = __dadd_rn(acc[0][0], __dmul_rn(a0, b.x));
        acc[0][1] = __dadd_rn(acc[0][1], __dmul_rn(a0, b.y));
        acc[1][0] = __dadd_rn(acc[1][0], __dmul_rn(a1, b.x));
        acc[1][1] = __dadd_rn(acc[1][1], __dmul_rn(a1, b.y));
      } else {
        acc[0][0] = fma(a0, b.x, acc[0][0]);
        acc[0][1] = fma(a0, b.y, acc[0][1]);
        acc[1][0] = fma(a1, b.x, acc[1][0]);
        acc[1][1] = fma(a1, b.y, acc[1][1]);
      }
    }
    if (kt + 1 < KT) store(buf ^ 1);
    __syncthreads();
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int r = row0 + ty * 2 + h;
    if (r >= M) continue;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int c = col0 + tx * 2 + e;
      if (c < N) C[static_cast<int64_t>(r) * ldc + c] = acc[h][e];
    }
  }
}

// 16x16 tiles, one output per thread (256 threads): four times the CTAs of
// the 32x32 kernel for the smallest problems; same per-element chain.
template <bool EXACT>
__global__ void __launch_bounds__(THREADS)
    dgemm_small16_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                         int64_t ldb, double* C, int64_t ldc, int M, int N, int K, int tiles_n,
                         const double* cin, int64_t ldcin) {
  constexpr int T16 = 16;
  __shared__ __align__(16) double As[2][T16][BK + 1];  // [row][k]
  __shared__ __align__(16) double Bs[2][BK][T16 + 1];  // [k][col]
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int row0 = (blockIdx.x / tiles_n) * T16, col0 = (blockIdx.x % tiles_n) * T16;
  // staging: A as 16 rows x 32 k (2 per thread), B as 32 k x 16 columns (2 per thread)
  const int ar = tid >> 4, ak = (tid & 15) * 2;
  const int bk = tid >> 3, bc = (tid & 7) * 2;
  double ra[2], rb[2];
  auto load = [&](int k0) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int r = row0 + ar, k = k0 + ak + j;
      ra[j] = (r < M && k < K) ? A[static_cast<int64_t>(r) * lda + k] : 0.0;
      const int kk = k0 + bk, c = col0 + bc + j;
      rb[j] = (kk < K && c < N) ? B[static_cast<int64_t>(kk) * ldb + c] : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      As[buf][ar][ak + j] = ra[j];
      Bs[buf][bk][bc + j] = rb[j];
    }
  };
  const int r = row0 + ty, c = col0 + tx;
  double acc = 0.0;
  if (cin && r < M && c < N) acc = cin[static_cast<int64_t>(r) * ldcin + c];
  const int KT = (K + BK - 1) / BK;
  load(0);
  store(0);
  __syncthreads();
  for (int kt = 0; kt < KT; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < KT) load((kt + 1) * BK);
#pragma unroll 8
    for (int k = 0; k < BK; ++k) {
      const double a = As[buf][ty][k], b = Bs[buf][k][tx];
      if constexpr (EXACT) acc = __dadd_rn(acc, __dmul_rn(a, b));
      else acc = fma(a, b, acc);
    }
    if (kt + 1 < KT) store(buf ^ 1);
    __syncthreads();
  }
  if (r < M && c < N) C[static_cast<int64_t>(r) * ldc + c] = acc;
}

}  // namespace

cudaError_t launch_dgemm_small16(const Launch& L, bool exact, int64_t M, int64_t N, int64_t K,
                                 const double* A, int64_t lda, const double* B, int64_t ldb,
                                 double* C, int64_t ldc, const double* cin, int64_t ldcin) {
  const int tiles_m = static_cast<int>((M + 15) / 16);
  const int tiles_n = static_cast<int>((N + 15) / 16);
  auto kern = exact ? dgemm_small16_kernel<true> : dgemm_small16_kernel<false>;
  kern<<<tiles_m * tiles_n, THREADS, 0, L.stream>>>(A, lda, B, ldb, C, ldc, static_cast<int>(M),
                                                    static_cast<int>(N), static_cast<int>(K),
                                                    tiles_n, cin, ldcin);
  L.count();
  return cudaGetLastError();
}

cudaError_t launch_dgemm_small(const Launch& L, bool exact, int64_t M, int64_t N, int64_t K,
                               const double* A, int64_t lda, const double* B, int64_t ldb,
                               double* C, int64_t ldc, const double* cin, int64_t ldcin) {
  const int tiles_m = static_cast<int>((M + T - 1) / T);
  const int tiles_n = static_cast<int>((N + T - 1) / T);
  auto kern = exact ? dgemm_small_kernel<true> : dgemm_small_kernel<false>;
  kern<<<tiles_m * tiles_n, THREADS, 0, L.stream>>>(A, lda, B, ldb, C, ldc, static_cast<int>(M),
                                                    static_cast<int>(N), static_cast<int>(K),
                                                    tiles_n, cin, ldcin);
  L.count();
  return cudaGetLastError();
}

cudaError_t preload_dgemm_small() {
  return preload_kernels(dgemm_small_kernel<true>, dgemm_small_kernel<false>,
                         dgemm_small16_kernel<true>, dgemm_small16_kernel<false>);
}

}  // namespace mmws_impl

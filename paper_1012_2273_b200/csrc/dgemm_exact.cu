// dgemm_exact.cu -- exact-order FP64 GEMM: bitwise equal to matmul_seq.
//
// The reference's bitwise contract (include/mmws/matrix.hpp:112-126, built
// with -ffp-contract=off, proj/CMakeLists.txt:12-15) is, per output element:
//     acc = +0.0;  for j = 0 .. K-1 ascending:  acc = RN(acc + RN(a(i,j)*b(j,k)))
// This kernel keeps exactly that chain per thread-owned element: DMUL then
// DADD (__dmul_rn / __dadd_rn are never contracted into DFMA), k ascending
// through the smem k-tiles, accumulator initialised to +0.0 and stored as is.
// Out-of-range k is zero-filled in BOTH operands, which appends (+0)*(+0) = +0
// terms; acc is never -0 (it starts at +0 and RN(x + -x) = +0), so acc + +0 ==
// acc bit-for-bit.  Hence C is bitwise matmul_seq(A, B) for every input
// without NaNs (NaN payload propagation is hardware-specific on both sides).
//
// Layout: 128x128 CTA tile, 256 threads, 8x8 register block per thread with
// rows {2*ty + 32v + h} and cols {2*tx + 32v + h} (v < 4, h < 2) so every
// fragment fetch is a conflict-free / broadcast 128-bit LDS; A is staged
// transposed (k-major) in shared memory, B as is; global->register->shared
// double buffering over 8-wide k-tiles.  Bound: FP64 pipe at one DMUL + one
// DADD per multiply-add, i.e. half of the DFMA peak.
#include "common.cuh"
#include "kernels.h"

namespace mmws_impl {
namespace {

constexpr int BM = 128, BN = 128, BK = 8, THREADS = 256;
constexpr int AV = BM * BK / THREADS;  // A elements staged per thread (4)
constexpr int BV = BN * BK / THREADS;  // B elements staged per thread (4)
constexpr int LDA_S = BM + 2;  // padded k-major A rows (keeps 16-byte alignment)

__global__ void __launch_bounds__(THREADS, 1)
    dgemm_exact_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                       int64_t ldb, double* __restrict__ C, int64_t ldc, int M, int N, int K,
                       int tiles_n) {
  __shared__ __align__(16) double As[2][BK][LDA_S];
  __shared__ __align__(16) double Bs[2][BK][BN];

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x % tiles_n;
  const int row0 = tm * BM, col0 = tn * BN;

  // global staging coordinates
  const int a_r = tid / (BK / AV), a_k = (tid % (BK / AV)) * AV;  // A: row a_r, k a_k..+AV
  const int b_k = tid / (BN / BV), b_c = (tid % (BN / BV)) * BV;  // B: k-row b_k, cols b_c..+BV
  const bool a_row_ok = row0 + a_r < M;
  const double* a_src = A + static_cast<int64_t>(row0 + a_r) * lda;

  double ra[AV], rb[BV];
  auto load_tile = [&](int kt) {
    const int k0 = kt * BK;
#pragma unroll
    for (int j = 0; j < AV; ++j) {
      const int k = k0 + a_k + j;
      ra[j] = (a_row_ok && k < K) ? a_src[k] : 0.0;
    }
    const int kb = k0 + b_k;
    const double* b_src = B + static_cast<int64_t>(kb) * ldb + col0 + b_c;
#pragma unroll
    for (int j = 0; j < BV; ++j) rb[j] = (kb < K && col0 + b_c + j < N) ? b_src[j] : 0.0;
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int j = 0; j < AV; ++j) As[buf][a_k + j][a_r] = ra[j];
#pragma unroll
    for (int j = 0; j < BV; j += 2)
      *reinterpret_cast<double2*>(&Bs[buf][b_k][b_c + j]) = make_double2(rb[j], rb[j + 1]);
  };

  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;

  const int KT = (K + BK - 1) / BK;
  load_tile(0);
  store_tile(0);
  __syncthreads();

  for (int kt = 0; kt < KT; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < KT) load_tile(kt + 1);
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      double a[8], b[8];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const double2 av = *reinterpret_cast<const double2*>(&As[buf][k][ty * 2 + 32 * v]);
        const double2 bv = *reinterpret_cast<const double2*>(&Bs[buf][k][tx * 2 + 32 * v]);
        a[2 * v] = av.x;
        a[2 * v + 1] = av.y;
        b[2 * v] = bv.x;
        b[2 * v + 1] = bv.y;
      }
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a[i], b[j]));
    }
    if (kt + 1 < KT) store_tile(buf ^ 1);
    __syncthreads();
  }

#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int r = row0 + ty * 2 + 32 * (i >> 1) + (i & 1);
    if (r >= M) continue;
    double* crow = C + static_cast<int64_t>(r) * ldc;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = col0 + tx * 2 + 32 * (j >> 1) + (j & 1);
      if (c < N) crow[c] = acc[i][j];
    }
  }
}

}  // namespace

cudaError_t launch_dgemm_exact(const Launch& L, int64_t M, int64_t N, int64_t K, const double* A,
                               int64_t lda, const double* B, int64_t ldb, double* C,
                               int64_t ldc) {
  const int tiles_m = static_cast<int>((M + BM - 1) / BM);
  const int tiles_n = static_cast<int>((N + BN - 1) / BN);
  dgemm_exact_kernel<<<tiles_m * tiles_n, THREADS, 0, L.stream>>>(
      A, lda, B, ldb, C, ldc, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K),
      tiles_n);
  L.count();
  return cudaGetLastError();
}

}  // namespace mmws_impl

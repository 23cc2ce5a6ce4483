// sgemm_tma.cu -- FP32 GEMM on the FFMA2 pipe, TMA-fed and warp-specialised.
//
// The fp32 configuration (BASELINE.json configs[4], N=32768 normal(0,1)) has
// no counterpart in the reference (its Matrix is fp64 only, matrix.hpp:39-91);
// this is the same C = A.B contraction as the reference's threaded body
// (workshare.hpp:98-113) in fp32, checked normwise against the fp64 oracle of
// the widened inputs (tolerance 1e-5, tests/test_gpu_parity.py).
//
// Accuracy: a single fp32 chain over K = 32768 terms has an expected normwise
// error of ~5e-6, uncomfortably close to the 1e-5 bound.  Each 1024-long
// k-chunk is therefore summed into a fresh register partial that is added
// into a running total kept in shared memory once per chunk -- two-level
// (blocked) summation, error growth ~sqrt(KC) + sqrt(K / KC) instead of
// ~sqrt(K), without doubling the accumulator registers.
//
// Structure (like the DMMA kernel, so the math warps do nothing but LDS +
// FFMA2):
//   * a producer warpgroup (one elected lane) streams A[128 x 16] and
//     B[16 x 256] k-slices with TMA into a 3-stage mbarrier ring and gives its
//     registers to the math warps (setmaxnreg 40 / 232);
//   * 8 math warps, each lane owning 8 rows x 16 columns (64 packed fp32 pairs)
//     -- 64 FFMA2 per k against 6 LDS.128 (A as 4-k vectors of one row,
//     broadcast; B as 4-column vectors 64 columns apart, conflict-free);
//   * stages are released one iteration late (after the next stage's full
//     barrier), the ptxas-proof ordering dgemm_dmma.cu documents.
// Operand pattern: every FFMA2 reads its accumulator pair and the broadcast A
// scalar from the register file (the B pair comes from the operand reuse
// cache).  How fast that issues depends on where the operands sit in the
// register file: register-only loops of this outer product measure 56-71
// TFLOP/s on B200 depending on the block shape and ptxas' assignment
// (tools/ffma2_shape_probe.cu), and with the operands fed by LDS.128 the
// row-major A stage -- a float4 holds four k of one row, so a row's scalar
// changes register bank with k -- costs 64.3 against 68.6 TFLOP/s for a
// k-major stage, where a float4 holds four rows of one k and each row's scalar
// keeps its register (tools/ffma2_lds_probe.cu, profiles/r02_ffma2_lds_probe.txt).
// Hence the AT instance: wide problems transpose A once (transpose_f32_kernel,
// HBM-bound, 0.17 % of the multiply at N=32768) and TMA stages A^T tiles;
// N=16384 65.0 vs 62.3 TFLOP/s, same bits (profiles/r02_sgemm_k_major.txt);
// 66.4 with the 3-stage ring.
// Layouts TMA cannot read are packed by the caller (mmws_gpu.cu), so every
// layout takes this kernel.
#include "common.cuh"
#include "kernels.h"

namespace mmws_impl {
namespace {

using namespace mmws_dev;

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

// k per stage and ring depth (build-time, for tuning runs: make EXTRA=-D...).
// The ring depth is not a limit (2, 3 and 4 stages of 16 k: 66.0 / 67.2 / 66.0
// TFLOP/s at N=32768; 8-k stages lose 8 %: profiles/r02_sgemm_ring_geometry.txt);
// 3 stages is the instance ptxas schedules best.
#ifndef MMWS_SGEMM_GROUP
#define MMWS_SGEMM_GROUP 8
#endif
#ifndef MMWS_SGEMM_BK
#define MMWS_SGEMM_BK 16
#endif
#ifndef MMWS_SGEMM_STAGES
#define MMWS_SGEMM_STAGES 3
#endif
constexpr int BM = 128, BN = 256, BK = MMWS_SGEMM_BK, STAGES = MMWS_SGEMM_STAGES, CONSUMERS = 8;
constexpr int THREADS = (CONSUMERS + 4) * 32;
constexpr int KC_STAGES = 1024 / BK;  // partial-sum chunk = 1024 k
constexpr int A_BYTES = BM * BK * 4, B_BYTES = BK * BN * 4;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TOT_BYTES = CONSUMERS * 32 * 128 * 4;  // 128 floats per math lane
constexpr int SMEM = STAGES * STAGE_BYTES + TOT_BYTES + 2 * STAGES * 8 + 128;

// AT: tmA describes A transposed ([K][M], made by transpose_f32_kernel), so a
// stage holds A k-major ([16 k][128 rows]) and one LDS.128 brings four rows of
// one k -- a row's A scalar then sits in the same register bank for every k
// (see the header); otherwise A is staged as it lies ([128 rows][16 k]).
template <bool AT>
__global__ void __launch_bounds__(THREADS, 1)
    sgemm_tma_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB, float* C, int64_t ldc,
                     int M, int N, int K, int tiles_m, int tiles_n, int vec_c, const float* cin,
                     int64_t ldcin) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  float4* tot = reinterpret_cast<float4*>(smem + STAGES * STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES + TOT_BYTES);
  uint64_t* empty = full + STAGES;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int GROUP = MMWS_SGEMM_GROUP;  // tile rows per raster group
  const int tile = blockIdx.x;
  const int per_group = GROUP * tiles_n;
  const int first_m = (tile / per_group) * GROUP;
  const int gm = min(tiles_m - first_m, GROUP);
  const int tm = first_m + (tile % per_group) % gm;
  const int tn = (tile % per_group) / gm;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CONSUMERS);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int KT = (K + BK - 1) / BK;

  if (warp >= CONSUMERS) {
    // ---------------- TMA producer ----------------
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if (warp == CONSUMERS && lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        if (kt >= STAGES) mbar_wait(&empty[s], ((kt / STAGES) - 1) & 1);
        uint8_t* sa = smem + s * STAGE_BYTES;
        mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
        if (AT) tma_load_2d(sa, &tmA, &full[s], tm * BM, kt * BK);
        else tma_load_2d(sa, &tmA, &full[s], kt * BK, tm * BM);
        tma_load_2d(sa + A_BYTES, &tmB, &full[s], tn * BN, kt * BK);
      }
    }
    return;
  }

  // ---------------- math warps ----------------
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
  const int g = lane >> 4, c = lane & 15;
  const int row_base = warp * 16 + g * 8;  // rows row_base + i, i < 8
  const int tid = threadIdx.x;             // < 256

#pragma unroll
  for (int q = 0; q < 32; ++q) tot[q * 256 + tid] = make_float4(0.f, 0.f, 0.f, 0.f);
  if (cin) {  // accumulate: the running totals start from Cin (the epilogue's layout)
#pragma unroll 4
    for (int q = 0; q < 32; ++q) {
      const int i = q >> 2, j = q & 3;
      const int r = tm * BM + row_base + i;
      if (r >= M) continue;
      const int col = tn * BN + c * 4 + 64 * j;
      const float* crow = cin + static_cast<int64_t>(r) * ldcin;
      float4 t;
      t.x = col + 0 < N ? crow[col + 0] : 0.f;
      t.y = col + 1 < N ? crow[col + 1] : 0.f;
      t.z = col + 2 < N ? crow[col + 2] : 0.f;
      t.w = col + 3 < N ? crow[col + 3] : 0.f;
      tot[q * 256 + tid] = t;
    }
  }

  f32x2 part[8][8];  // [row i][pair p]: columns c*4 + 64*(p>>1) + 2*(p&1) + {0,1}
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int p = 0; p < 8; ++p) part[i][p] = 0ull;

  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % STAGES;
    mbar_wait(&full[s], (kt / STAGES) & 1);
    if (kt > 0) {  // release the previous stage (see header)
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[(kt - 1) % STAGES]);
    }
    const float* as = reinterpret_cast<const float*>(smem + s * STAGE_BYTES);
    const float* bs = as + BM * BK;
#pragma unroll
    for (int k4 = 0; k4 < BK; k4 += 4) {
      float4 a4[8];
      if (!AT) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
          a4[i] = *reinterpret_cast<const float4*>(as + (row_base + i) * BK + k4);
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        float4 at[2];  // AT: rows row_base .. +7 at k = k4 + kk
        if (AT) {
          at[0] = *reinterpret_cast<const float4*>(as + (k4 + kk) * BM + row_base);
          at[1] = *reinterpret_cast<const float4*>(as + (k4 + kk) * BM + row_base + 4);
        }
        f32x2 b2[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 b = *reinterpret_cast<const float4*>(bs + (k4 + kk) * BN + c * 4 + 64 * j);
          b2[2 * j] = pack2(b.x, b.y);
          b2[2 * j + 1] = pack2(b.z, b.w);
        }
        f32x2 aa[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          float a;
          if (AT) {
            const float4 t = at[i >> 2];
            a = (i & 3) == 0 ? t.x : (i & 3) == 1 ? t.y : (i & 3) == 2 ? t.z : t.w;
          } else {
            a = kk == 0 ? a4[i].x : kk == 1 ? a4[i].y : kk == 2 ? a4[i].z : a4[i].w;
          }
          aa[i] = pack2(a, a);
        }
        // B pair outer, A inner: consecutive FFMA2s share the B pair (operand
        // reuse cache) and read one fresh scalar A register each
#pragma unroll
        for (int p = 0; p < 8; ++p)
#pragma unroll
          for (int i = 0; i < 8; ++i) ffma2(part[i][p], b2[p], aa[i]);
      }
    }
    if ((kt % KC_STAGES) == KC_STAGES - 1 || kt + 1 == KT) {
#pragma unroll
      for (int q = 0; q < 32; ++q) {  // q = i*4 + j: row i, column group j
        const int i = q >> 2, j = q & 3;
        float4 t = tot[q * 256 + tid];
        const float2 lo = unpack2(part[i][2 * j]), hi = unpack2(part[i][2 * j + 1]);
        t.x += lo.x;
        t.y += lo.y;
        t.z += hi.x;
        t.w += hi.y;
        tot[q * 256 + tid] = t;
        part[i][2 * j] = part[i][2 * j + 1] = 0ull;
      }
    }
  }

#pragma unroll
  for (int q = 0; q < 32; ++q) {
    const int i = q >> 2, j = q & 3;
    const int r = tm * BM + row_base + i;
    if (r >= M) continue;
    const int col = tn * BN + c * 4 + 64 * j;
    const float4 v = tot[q * 256 + tid];
    float* crow = C + static_cast<int64_t>(r) * ldc;
    if (vec_c && col + 3 < N) {
      *reinterpret_cast<float4*>(crow + col) = v;
    } else {
      const float w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (col + e < N) crow[col + e] = w[e];
    }
  }
}

// A [rows][cols] (pitch ld_src, any alignment) -> dst [cols][rows] (pitch
// ld_dst): one HBM-bound pass, 32x32 tiles through shared memory so both sides
// are coalesced.
__global__ void __launch_bounds__(256)
    transpose_f32_kernel(const float* __restrict__ src, int64_t rows, int64_t cols, int64_t ld_src,
                         float* __restrict__ dst, int64_t ld_dst) {
  __shared__ float tile[32][33];
  // 1-D grid (no 65535 limit on either dimension), column tiles fastest
  const int64_t tiles_c = (cols + 31) / 32;
  const int64_t c0 = (blockIdx.x % tiles_c) * 32, r0 = (blockIdx.x / tiles_c) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    const int64_t r = r0 + ty + j, c = c0 + tx;
    tile[ty + j][tx] = r < rows && c < cols ? src[r * ld_src + c] : 0.f;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 32; j += 8) {
    const int64_t c = c0 + ty + j, r = r0 + tx;
    if (c < cols && r < rows) dst[c * ld_dst + r] = tile[tx][ty + j];
  }
}

bool make_map_f32(const Launch& L, CUtensorMap* map, const float* base, int64_t inner,
                  int64_t outer, int64_t ld, int box_inner, int box_outer) {
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(float)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner),
                             static_cast<cuuint32_t>(box_outer)};
  const cuuint32_t estr[2] = {1, 1};
  return L.encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

bool sgemm_tma_supported(int64_t lda, int64_t ldb, const float* A, const float* B) {
  return lda % 4 == 0 && ldb % 4 == 0 && reinterpret_cast<uintptr_t>(A) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(B) % 16 == 0;
}

cudaError_t launch_transpose_f32(const Launch& L, const float* src, int64_t rows, int64_t cols,
                                 int64_t ld_src, float* dst, int64_t ld_dst) {
  const int64_t tiles = ((cols + 31) / 32) * ((rows + 31) / 32);
  if (tiles > 0x7fffffffLL) return cudaErrorInvalidValue;
  transpose_f32_kernel<<<static_cast<unsigned>(tiles), 256, 0, L.stream>>>(src, rows, cols, ld_src,
                                                                          dst, ld_dst);
  L.count();
  return cudaGetLastError();
}

// a_transposed: A points at A transposed ([K][M], pitch lda >= M)
cudaError_t launch_sgemm_tma(const Launch& L, int64_t M, int64_t N, int64_t K, const float* A,
                             int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                             const float* cin, int64_t ldcin, bool a_transposed) {
  CUtensorMap ta, tb;
  if (a_transposed ? !make_map_f32(L, &ta, A, M, K, lda, BM, BK)
                   : !make_map_f32(L, &ta, A, K, M, lda, BK, BM))
    return cudaErrorInvalidValue;
  if (!make_map_f32(L, &tb, B, N, K, ldb, BN, BK)) return cudaErrorInvalidValue;
  auto kern = a_transposed ? sgemm_tma_kernel<true> : sgemm_tma_kernel<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  if (e != cudaSuccess) return e;
  const int tiles_m = static_cast<int>((M + BM - 1) / BM);
  const int tiles_n = static_cast<int>((N + BN - 1) / BN);
  const int vec_c = (ldc % 4 == 0) && (reinterpret_cast<uintptr_t>(C) % 16 == 0);
  kern<<<tiles_m * tiles_n, THREADS, SMEM, L.stream>>>(
      ta, tb, C, ldc, static_cast<int>(M), static_cast<int>(N), static_cast<int>(K), tiles_m,
      tiles_n, vec_c, cin, ldcin);
  L.count();
  return cudaGetLastError();
}

cudaError_t preload_sgemm_tma() {
  return preload_kernels(sgemm_tma_kernel<false>, sgemm_tma_kernel<true>, transpose_f32_kernel);
}

}  // namespace mmws_impl

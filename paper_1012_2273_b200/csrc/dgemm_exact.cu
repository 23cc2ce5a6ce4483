// dgemm_exact.cu -- exact-order FP64 GEMM: bitwise equal to matmul_seq.
//
// The reference's bitwise contract (include/mmws/matrix.hpp:112-126, built
// with -ffp-contract=off, proj/CMakeLists.txt:12-15) is, per output element:
//     acc = +0.0;  for j = 0 .. K-1 ascending:  acc = RN(acc + RN(a(i,j)*b(j,k)))
// This kernel keeps exactly that chain per thread-owned element: DMUL then
// DADD (__dmul_rn / __dadd_rn are never contracted into DFMA), k ascending
// through the shared-memory k-tiles, accumulator initialised to +0.0 and
// stored as is.  Out-of-range k is zero-filled in BOTH operands, which appends
// (+0)*(+0) = +0 terms; acc is never -0 (it starts at +0 and RN(x + -x) = +0),
// so acc + +0 == acc bit-for-bit.  Hence C is bitwise matmul_seq(A, B) for
// every input without NaNs (NaN payload propagation is hardware-specific on
// both sides).
//
// Layout: 128x128 CTA tile, 256 threads, 8x8 register block per thread with
// rows {2*ty + 32v + h} and cols {2*tx + 32v + h} (v < 4, h < 2).  A and B
// k-tiles (16 wide) stream through a 3-stage cp.async ring in their natural
// row-major layout; a lane fetches A as (k, k+1) pairs of one row (broadcast
// LDS.128) and B as column pairs (conflict-free LDS.128).  Bound: FP64 pipe
// at one DMUL + one DADD per multiply-add, i.e. half of the DFMA peak.
#include "common.cuh"
#include "kernels.h"

namespace mmws_impl {
namespace {

using namespace mmws_dev;

constexpr int BM = 128, BN = 128, BK = 16, THREADS = 256, STAGES = 3;
constexpr int SLA = BK + 2;   // A row pitch (doubles): keeps 16-byte alignment, spreads banks
constexpr int SLB = BN;       // B row pitch
constexpr int A_ELEMS = BM * SLA, B_ELEMS = BK * SLB;
constexpr int SMEM = STAGES * (A_ELEMS + B_ELEMS) * sizeof(double);

template <bool VA, bool VB>
__global__ void __launch_bounds__(THREADS, 1)
    dgemm_exact_kernel(const double* __restrict__ A, int64_t lda, const double* __restrict__ B,
                       int64_t ldb, double* C, int64_t ldc, int M, int N, int K,
                       int tiles_m, int tiles_n, const double* cin, int64_t ldcin) {
  extern __shared__ __align__(16) double smem_d[];
  double* As = smem_d;                       // [STAGES][BM][SLA]
  double* Bs = smem_d + STAGES * A_ELEMS;    // [STAGES][BK][SLB]

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
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
    load_tile_async<double, BM, BK, SLA, THREADS, VA>(As + s * A_ELEMS, A, lda, row0, kt * BK, M, K);
    load_tile_async<double, BK, BN, SLB, THREADS, VB>(Bs + s * B_ELEMS, B, ldb, kt * BK, col0, K, N);
  };

  double acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0;
  if (cin) {  // accumulate: continue Cin's chains (the epilogue's layout; Cin may alias C)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = row0 + ty * 2 + 32 * (i >> 1) + (i & 1);
      if (r >= M) continue;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = col0 + tx * 2 + 32 * (j >> 1) + (j & 1);
        if (c < N) acc[i][j] = cin[static_cast<int64_t>(r) * ldcin + c];
      }
    }
  }

#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_stage(s);
    cp_async_commit();
  }

  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();  // stage kt landed for everyone; stage kt-1 fully consumed
    if (kt + STAGES - 1 < KT) load_stage(kt + STAGES - 1);
    cp_async_commit();
    const double* as = As + (kt % STAGES) * A_ELEMS;
    const double* bs = Bs + (kt % STAGES) * B_ELEMS;
#pragma unroll
    for (int k = 0; k < BK; k += 2) {
      double2 a2[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        a2[i] = *reinterpret_cast<const double2*>(as + (ty * 2 + 32 * (i >> 1) + (i & 1)) * SLA + k);
#pragma unroll
      for (int kk = 0; kk < 2; ++kk) {
        double b[8];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const double2 bv = *reinterpret_cast<const double2*>(bs + (k + kk) * SLB + tx * 2 + 32 * v);
          b[2 * v] = bv.x;
          b[2 * v + 1] = bv.y;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const double a = kk ? a2[i].y : a2[i].x;
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a, b[j]));
        }
      }
    }
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

// ---------------------------------------------------------------------------
// TMA-fed, warp-specialised variant (same per-thread arithmetic and layout):
// a producer warpgroup streams A[128 x 16] and B[16 x 128] k-slices with TMA
// into a 4-stage mbarrier ring and donates its registers to the 8 math warps
// (setmaxnreg 40 / 232), so the math warps issue nothing but LDS, DMUL and
// DADD -- no cp.async address arithmetic, no __syncthreads per k-tile.  Stages
// are released one iteration late (see dgemm_dmma.cu).  Zero-filled TMA
// out-of-bounds boxes are the (+0)*(+0) padding discussed above.
// TBM x TBN tiles (128x128, or 64x64 / 32x32 for problems that would leave
// SMs idle);
// each of the 256 math threads owns (TBM/16) x (TBN/16) outputs at rows
// 2*ty + 32v + h and columns 2*tx + 32v + h.
// CONS math warps (8, or 4 for the 32x32 tile): 16 x (2*CONS) math threads,
// rows 2*ty + RP*v + h with the row period RP = 4*CONS.  The 32x32 tile
// runs 4 math warps with 4 x 2 outputs per thread (64 registers, 4 CTAs/SM):
// fewer LDS per DMUL+DADD than 8 warps with 2 x 2 -- device time per call
// (round 2, tools/exact_plan_probe.py) N=256 12.4 -> 10.4 us, 300 14.4 ->
// 12.4, 400 24.7 -> 21.3, 500 32.1 -> 26.8; on the 64x64 tile 4 warps lose
// (N=640 52.7 vs 55.1, 1000 stream-K 140.1 vs 148.4).
#ifndef MMWS_EXACT_STAGES  // ring depth of the TMA variant (build-time, for tuning runs)
#define MMWS_EXACT_STAGES 4
#endif
constexpr int T_STAGES = MMWS_EXACT_STAGES;
template <int TBM, int TBN, int CONS = 8>
struct ExactTma {
  static constexpr int A_BYTES = TBM * BK * 8, B_BYTES = BK * TBN * 8;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int SMEM = T_STAGES * STAGE + 2 * T_STAGES * 8 + 128;
  static constexpr int RP = 4 * CONS;                        // row period
  static constexpr int TM = 2 * TBM / RP, TN = TBN / 16;     // outputs per thread
  static constexpr int THREADS = (CONS + 4) * 32;
  static constexpr int MINB = TBM == 128 ? 1 : TBM == 64 ? 2 : 4;
  static_assert(TBM % RP == 0, "row period");
};

// SK = true: stream-K with in-order fix-up, exactly as dgemm_dmma.cu's MODE 2
// (one persistent CTA per SM, equal k-iteration ranges walked top-down, a cut
// tile's accumulators parked by the lower CTA and continued by the upper one)
// -- each element keeps its single ascending-k DMUL+DADD chain, so the result
// is still bitwise matmul_seq.
MMWS_DEVICE uint64_t exact_global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
MMWS_DEVICE void exact_wait_flag(const int* f) {
  const uint64_t t0 = exact_global_ns();
  for (;;) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if (v) return;
    __nanosleep(200);
    if (exact_global_ns() - t0 > 60ull * 1000000000ull) __trap();
  }
}

template <int TBM, int TBN, bool SK = false, int CONS = 8>
__global__ void __launch_bounds__(ExactTma<TBM, TBN, CONS>::THREADS, ExactTma<TBM, TBN, CONS>::MINB)
    dgemm_exact_tma_kernel(const __grid_constant__ CUtensorMap tmA,
                           const __grid_constant__ CUtensorMap tmB, double* C,
                           int64_t ldc, int M, int N, int K, int tiles_m, int tiles_n,
                           double* partial = nullptr, int* flags = nullptr,
                           const double* cin = nullptr, int64_t ldcin = 0) {
  using X = ExactTma<TBM, TBN, CONS>;
  constexpr int T_A_BYTES = X::A_BYTES, T_STAGE = X::STAGE, TM = X::TM, TN = X::TN;
  constexpr int RP = X::RP, T_CONSUMERS = CONS;
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + T_STAGES * T_STAGE);
  uint64_t* empty = full + T_STAGES;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int GROUP = 8;
  auto raster = [&](int tile, int& tm, int& tn) {
    const int per_group = GROUP * tiles_n;
    const int first_m = (tile / per_group) * GROUP;
    const int gm = min(tiles_m - first_m, GROUP);
    tm = first_m + (tile % per_group) % gm;
    tn = (tile % per_group) / gm;
  };
  if (threadIdx.x == 0) {
    for (int s = 0; s < T_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], T_CONSUMERS);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const int KT = (K + BK - 1) / BK;
  // work units (tile, k-iterations [k0, k1)): the CTA's tile, or (SK) its
  // iteration range top-down
  const long long w = static_cast<long long>(tiles_m) * tiles_n * KT;
  const long long lo = SK ? w * blockIdx.x / gridDim.x : 0;
  const long long hi0 = SK ? w * (blockIdx.x + 1) / gridDim.x : 1;
  auto next_unit = [&](long long& pos, int& tile, int& k0, int& k1) -> bool {
    if constexpr (SK) {
      if (pos <= lo) return false;
      tile = static_cast<int>((pos - 1) / KT);
      const long long base = static_cast<long long>(tile) * KT;
      k0 = static_cast<int>((lo > base ? lo : base) - base);
      k1 = static_cast<int>(pos - base);
      pos = base + k0;
    } else {
      if (pos == 0) return false;
      pos = 0;
      tile = blockIdx.x;
      k0 = 0;
      k1 = KT;
    }
    return true;
  };

  if (warp >= T_CONSUMERS) {
    if constexpr (TBM == 128) asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if (warp == T_CONSUMERS && lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      long long pos = hi0;
      int tile, k0, k1, kg = 0;  // kg: stage counter, continuous across units
      while (next_unit(pos, tile, k0, k1)) {
        int tm, tn;
        raster(tile, tm, tn);
        for (int kt = k0; kt < k1; ++kt, ++kg) {
          const int s = kg % T_STAGES;
          if (kg >= T_STAGES) mbar_wait(&empty[s], ((kg / T_STAGES) - 1) & 1);
          uint8_t* sa = smem + s * T_STAGE;
          mbar_arrive_expect_tx(&full[s], T_STAGE);
          tma_load_2d(sa, &tmA, &full[s], kt * BK, tm * TBM);
          tma_load_2d(sa + T_A_BYTES, &tmB, &full[s], tn * TBN, kt * BK);
        }
      }
    }
    return;
  }
  if constexpr (TBM == 128) asm volatile("setmaxnreg.inc.sync.aligned.u32 232;");
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  constexpr int MATH_THREADS = T_CONSUMERS * 32;
  long long pos = hi0;
  int tile, k0, k1, kg = 0;
  while (next_unit(pos, tile, k0, k1)) {
    int tm, tn;
    raster(tile, tm, tn);
    double acc[TM][TN];
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;
    if (!SK && cin) {  // accumulate: continue Cin's chains (epilogue layout)
#pragma unroll
      for (int i = 0; i < TM; ++i) {
        const int r = tm * TBM + ty * 2 + RP * (i >> 1) + (i & 1);
        if (r >= M) continue;
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          const int c = tn * TBN + tx * 2 + 32 * (j >> 1) + (j & 1);
          if (c < N) acc[i][j] = cin[static_cast<int64_t>(r) * ldcin + c];
        }
      }
    }
    if constexpr (SK) {
      if (k0 > 0) {  // continue the lower CTA's chains for this tile
        if (tid == 0) exact_wait_flag(flags + blockIdx.x);
        asm volatile("bar.sync 1, %0;" ::"n"(MATH_THREADS) : "memory");
        const double* src = partial + static_cast<size_t>(blockIdx.x) * TM * TN * MATH_THREADS;
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = __ldcg(src + (i * TN + j) * MATH_THREADS + tid);
        if (tid == 0) flags[blockIdx.x] = 0;
      }
    }

    for (int kt = k0; kt < k1; ++kt, ++kg) {
      const int s = kg % T_STAGES;
      mbar_wait(&full[s], (kg / T_STAGES) & 1);
      if (kg > 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[(kg - 1) % T_STAGES]);
      }
      const double* as = reinterpret_cast<const double*>(smem + s * T_STAGE);  // [TBM][BK]
      const double* bs = as + TBM * BK;                                         // [BK][TBN]
#pragma unroll
      for (int k = 0; k < BK; k += 2) {
        double2 a2[TM];
#pragma unroll
        for (int i = 0; i < TM; ++i)
          a2[i] =
              *reinterpret_cast<const double2*>(as + (ty * 2 + RP * (i >> 1) + (i & 1)) * BK + k);
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          double b[TN];
#pragma unroll
          for (int v = 0; v < TN / 2; ++v) {
            const double2 bv =
                *reinterpret_cast<const double2*>(bs + (k + kk) * TBN + tx * 2 + 32 * v);
            b[2 * v] = bv.x;
            b[2 * v + 1] = bv.y;
          }
#pragma unroll
          for (int i = 0; i < TM; ++i) {
            const double a = kk ? a2[i].y : a2[i].x;
#pragma unroll
            for (int j = 0; j < TN; ++j) acc[i][j] = __dadd_rn(acc[i][j], __dmul_rn(a, b[j]));
          }
        }
      }
    }
    if constexpr (SK) {
      if (k1 < KT) {  // first part of a tile the upper CTA finishes: park it
        double* dst = partial + static_cast<size_t>(blockIdx.x + 1) * TM * TN * MATH_THREADS;
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) __stcg(dst + (i * TN + j) * MATH_THREADS + tid, acc[i][j]);
        asm volatile("bar.sync 1, %0;" ::"n"(MATH_THREADS) : "memory");
        if (tid == 0) {
          __threadfence();
          asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flags + blockIdx.x + 1), "r"(1)
                       : "memory");
        }
        continue;
      }
    }
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      const int r = tm * TBM + ty * 2 + RP * (i >> 1) + (i & 1);
      if (r >= M) continue;
      double* crow = C + static_cast<int64_t>(r) * ldc;
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int c = tn * TBN + tx * 2 + 32 * (j >> 1) + (j & 1);
        if (c < N) crow[c] = acc[i][j];
      }
    }
  }
}

bool make_map_f64(const Launch& L, CUtensorMap* map, const double* base, int64_t inner,
                  int64_t outer, int64_t ld, int box_inner, int box_outer) {
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(double)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner),
                             static_cast<cuuint32_t>(box_outer)};
  const cuuint32_t estr[2] = {1, 1};
  return L.encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int TBM, int TBN, bool SK = false, int CONS = 8>
cudaError_t run_exact_tma(const Launch& L, int64_t M, int64_t N, int64_t K, const double* A,
                          int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                          double* partial = nullptr, int* flags = nullptr, int grid = 0,
                          const double* cin = nullptr, int64_t ldcin = 0) {
  using X = ExactTma<TBM, TBN, CONS>;
  CUtensorMap ta, tb;
  if (!make_map_f64(L, &ta, A, K, M, lda, BK, TBM) || !make_map_f64(L, &tb, B, N, K, ldb, TBN, BK))
    return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(dgemm_exact_tma_kernel<TBM, TBN, SK, CONS>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, X::SMEM);
  if (e != cudaSuccess) return e;
  const int tiles_m = static_cast<int>((M + TBM - 1) / TBM);
  const int tiles_n = static_cast<int>((N + TBN - 1) / TBN);
  dgemm_exact_tma_kernel<TBM, TBN, SK, CONS><<<SK ? grid : tiles_m * tiles_n, X::THREADS,
                                               X::SMEM, L.stream>>>(ta, tb, C, ldc, static_cast<int>(M),
                                                     static_cast<int>(N), static_cast<int>(K),
                                                     tiles_m, tiles_n, partial, flags, cin,
                                                     ldcin);
  L.count();
  return cudaGetLastError();
}

}  // namespace

bool exact_tma_ok(int64_t lda, int64_t ldb, const double* A, const double* B) {
  return lda % 2 == 0 && ldb % 2 == 0 && reinterpret_cast<uintptr_t>(A) % 16 == 0 &&
         reinterpret_cast<uintptr_t>(B) % 16 == 0;
}

cudaError_t launch_dgemm_exact_sk(const Launch& L, int tile, int64_t M, int64_t N, int64_t K,
                                  const double* A, int64_t lda, const double* B, int64_t ldb,
                                  double* C, int64_t ldc, double* partial, int* flags, int grid) {
  return tile == 64
             ? run_exact_tma<64, 64, true>(L, M, N, K, A, lda, B, ldb, C, ldc, partial, flags, grid)
             : run_exact_tma<128, 128, true>(L, M, N, K, A, lda, B, ldb, C, ldc, partial, flags,
                                             grid);
}

const char* exact_oneshot_plan(const Launch& L, int64_t M, int64_t N, const double* A,
                               int64_t lda, const double* B, int64_t ldb) {
  if (!exact_tma_ok(lda, ldb, A, B)) return "dgemm_exact_kernel<128x128, cp.async>";
  const int64_t tiles64 = ((M + 63) / 64) * ((N + 63) / 64);
  const int64_t tiles128 = ((M + 127) / 128) * ((N + 127) / 128);
  if (2 * tiles64 <= L.num_sms) return "dgemm_exact_tma_kernel<32x32>";  // 4 math warps
  return tiles128 < 2 * L.num_sms ? "dgemm_exact_tma_kernel<64x64>"
                                  : "dgemm_exact_tma_kernel<128x128>";
}

cudaError_t launch_dgemm_exact(const Launch& L, int64_t M, int64_t N, int64_t K, const double* A,
                               int64_t lda, const double* B, int64_t ldb, double* C,
                               int64_t ldc, const double* cin, int64_t ldcin) {
  const int tiles_m = static_cast<int>((M + BM - 1) / BM);
  const int tiles_n = static_cast<int>((N + BN - 1) / BN);
  if (exact_tma_ok(lda, ldb, A, B)) {  // TMA can describe both operands
    // 32x32 tiles while 64x64 ones would not give half the SMs one (device
    // time per call, 64x64 vs 32x32, round 2, tools/exact_plan_probe.py:
    // N=400 33.7 vs 24.8 us, 500 42.8 vs 32.0, 128x500x500 41.1 vs 20.6,
    // 128x1000x1000 78.0 vs 38.6, 256x1000x1000 78.7 vs 58.2; from ~100
    // 64x64 tiles on the bigger tile wins: N=640 52.7 vs 55.4, 700 58.2 vs
    // 78.7, 256x2000x2000 153.9 vs 211.8), then 64x64 tiles while 128x128
    // ones would not give every SM two CTAs
    const int64_t tiles64 = ((M + 63) / 64) * ((N + 63) / 64);
    if (2 * tiles64 <= L.num_sms)  // 4 math warps, 4 x 2 outputs each (see ExactTma)
      return run_exact_tma<32, 32, false, 4>(L, M, N, K, A, lda, B, ldb, C, ldc, nullptr, nullptr,
                                             0, cin, ldcin);
    return tiles_m * tiles_n < 2 * L.num_sms
               ? run_exact_tma<64, 64>(L, M, N, K, A, lda, B, ldb, C, ldc, nullptr, nullptr, 0,
                                       cin, ldcin)
               : run_exact_tma<128, 128>(L, M, N, K, A, lda, B, ldb, C, ldc, nullptr, nullptr, 0,
                                         cin, ldcin);
  }
  // 16-byte cp.async when a whole chunk is always in or out of the matrix
  const bool va = lda % 2 == 0 && K % 2 == 0 && reinterpret_cast<uintptr_t>(A) % 16 == 0;
  const bool vb = ldb % 2 == 0 && N % 2 == 0 && reinterpret_cast<uintptr_t>(B) % 16 == 0;
  auto kern = va ? (vb ? dgemm_exact_kernel<true, true> : dgemm_exact_kernel<true, false>)
                 : (vb ? dgemm_exact_kernel<false, true> : dgemm_exact_kernel<false, false>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  if (e != cudaSuccess) return e;
  kern<<<tiles_m * tiles_n, THREADS, SMEM, L.stream>>>(A, lda, B, ldb, C, ldc,
                                                       static_cast<int>(M), static_cast<int>(N),
                                                       static_cast<int>(K), tiles_m, tiles_n,
                                                       cin, ldcin);
  L.count();
  return cudaGetLastError();
}

cudaError_t preload_dgemm_exact() {
  return preload_kernels(dgemm_exact_tma_kernel<32, 32, false, 4>, dgemm_exact_tma_kernel<64, 64>,
                         dgemm_exact_tma_kernel<128, 128>,
                         dgemm_exact_tma_kernel<128, 128, true>, dgemm_exact_tma_kernel<64, 64, true>,
                         dgemm_exact_kernel<true, true>, dgemm_exact_kernel<true, false>,
                         dgemm_exact_kernel<false, true>, dgemm_exact_kernel<false, false>);
}

}  // namespace mmws_impl

// dgemm_dmma.cu -- FP64 GEMM on the sm_100a FP64 tensor path (DMMA.8x8x4).
//
// Replaces the inner triple loop of matmul_seq / matmul_threads / worker_run
// (reference include/mmws/matrix.hpp:118-124, workshare.hpp:105-111,
// protocol.hpp:132-141) for real-valued fp64 inputs.  Blackwell has no
// tcgen05 .kind::f64, so the FP64 tensor instruction is warp-level
// mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4.
//
// Structure (one CTA per BMxBN output tile, 1 CTA/SM for the big config):
//   * warp CONSUMERS (the last warp) is the TMA producer: one elected lane
//     streams A[BM x 16] and B[16 x BN] k-slices into a STAGES-deep ring of
//     128B-swizzled shared-memory stages, completion via mbarrier tx-counts;
//   * CONSUMERS math warps each own a WM x WN sub-tile held as DMMA
//     accumulator fragments in registers (acc = +0.0 at start; the epilogue
//     stores the accumulator directly -- no beta*C read);
//   * fragments are fetched with conflict-free 128-bit LDS thanks to two
//     index permutations that the 8x8x4 MMA does not care about:
//       - k: within each 8-wide k-group the lane with k-slot t holds the pair
//         (2t, 2t+1) and feeds element q to MMA #q (q = 0, 1);
//       - m: row slot g of an 8-row subtile is physical row sigma(g) =
//         (g>>1) + 4(g&1), so the two rows a quarter-warp touches sit in
//         opposite halves of the 128-byte swizzle row;
//       - n: lane slot g of 16-column box b holds columns (2g, 2g+1) and feeds
//         element e to MMA (b, e); each lane ends up owning 4 consecutive
//         output columns, stored as two 16-byte vectors.
//   * integer-valued inputs (|partial sums| < 2^53) come out bit-exact in any
//     accumulation order, which is what the N=4099 exactness config checks.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace mmws_impl {
namespace {

using namespace mmws_dev;

constexpr int isqrt_round(int x) {
  int r = 0;
  while ((r + 1) * (r + 1) <= x) ++r;
  return (x - r * r > r) ? r + 1 : r;
}
static_assert(isqrt_round(148) == 12 && isqrt_round(444) == 21, "raster groups");

template <int BM_, int BN_, int WM_, int WN_, int STAGES_, int MINB_>
struct Cfg {
  static constexpr int BM = BM_, BN = BN_, WM = WM_, WN = WN_, STAGES = STAGES_, MINB = MINB_;
  static constexpr int BK = 16;  // 16 doubles = one 128-byte swizzle row
  static constexpr int WARPS_M = BM / WM, WARPS_N = BN / WN;
  static constexpr int CONSUMERS = WARPS_M * WARPS_N;
  // With 8 math warps the producer is a whole warpgroup so setmaxnreg can move
  // its registers to the math warpgroups (register budgets are per 4-warp
  // group); smaller configurations need no register shuffle and use one
  // producer warp, which leaves registers for more resident CTAs.
  static constexpr int MATH_REGS = CONSUMERS == 8 ? 232 : 0;  // 0: no setmaxnreg
  static constexpr int PRODUCERS = MATH_REGS > 0 ? 4 : 1;
  static constexpr int THREADS = (CONSUMERS + PRODUCERS) * 32;
  static constexpr int MI = WM / 8;   // 8-row subtiles per warp
  static constexpr int NB = WN / 16;  // 16-column boxes per warp
  static constexpr int A_BYTES = BM * BK * 8;
  static constexpr int B_BYTES = BN * BK * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 2 * STAGES * 8 + 1024;
  static_assert(BM % WM == 0 && BN % WN == 0 && WM % 8 == 0 && WN % 16 == 0, "tile");
  static_assert(BM <= 256, "TMA box");
  // Raster group (tile rows advancing together).  Default: a wave of 148 x
  // MINB resident tiles covers a square of C, the fewest distinct A and B
  // panels per wave (128x128: 12; measured at N=16384: 48.6 GB DRAM reads vs
  // 52.2 with 8 and 78.3 with 4, same time).  64x64 with 3 CTAs/SM: 10
  // (N=16384: 116 GB vs 180 GB with the square 21, 133 with 6, 364 with 42;
  // N=8192: 12.1 vs 14.0 GB; the time does not move, the kernel is bound by
  // the FP64 tensor pipe either way).
  static constexpr int GROUP = (BM == 64 && BN == 64 && MINB == 3)
                                   ? 10
                                   : isqrt_round(148 * MINB * BN / BM);
};

using Big = Cfg<128, 128, 64, 32, 6, 1>;   // 8 math warps, 192 KB ring, 1 CTA/SM
using Small = Cfg<64, 64, 32, 32, 4, 3>;   // 4 math warps, 64 KB ring, 3 CTAs/SM
using Mid = Cfg<128, 64, 32, 32, 5, 1>;    // 8 math warps, 160 KB ring
using Small8 = Cfg<64, 64, 32, 16, 6, 1>;  // 8 math warps on a 64x64 tile (stream-K, 1 CTA/SM)
using Tiny = Cfg<32, 32, 16, 16, 4, 6>;    // 4 math warps, 32 KB ring, 6 CTAs/SM
using Slim = Cfg<32, 64, 16, 32, 4, 4>;    // 4 math warps, 48 KB ring, 4 CTAs/SM
// Few-tile grids (small N): the K loop of a lone tile is bound by TMA round
// trips, not the tensor pipe, so these keep most of K in flight at once.
using TinyDeep = Cfg<32, 32, 16, 16, 12, 2>;  // 4 math warps, 96 KB ring, 2 CTAs/SM
using Micro = Cfg<16, 16, 8, 16, 12, 4>;      // 2 math warps, 48 KB ring, 4 CTAs/SM

// Poll an arrival flag (written by a cuStreamWriteValue32 behind an H2D copy).
// A flag that never arrives is a host-side bug; trap after 60 s so the
// context fails loudly instead of hanging the device.
MMWS_DEVICE uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
MMWS_DEVICE void wait_flag(const int* f) {
  const uint64_t t0 = global_ns();
  for (;;) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
    if (v) return;
    __nanosleep(200);
    if (global_ns() - t0 > 60ull * 1000000000ull) __trap();
  }
}
MMWS_DEVICE void set_flag(int* f, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(f), "r"(v) : "memory");
}

// MODE 0 (one-shot): one CTA per tile, grouped rasterisation (the
// device-pointer path).
// MODE 1 (streamed): persistent CTAs walk a host-ordered tile list (CTA b
// takes entries b, b + grid, ...), the producer waits for the A row band and
// B column band of each tile to have arrived (flags), and the math warps
// count finished tiles per tile row so a copy stream can ship C rows back
// while the rest computes (host_pipeline.cu).
// MODE 2 (stream-K, in-order fix-up): one persistent CTA per SM; CTA b owns
// the global k-iterations [W*b/G, W*(b+1)/G) of the W = tiles*KT iteration
// space, so every SM gets the same work whatever the tile count (no
// partial last wave).  A tile cut by a range boundary is finished by the
// upper CTA *continuing* the lower CTA's accumulators: the lower CTA walks
// its range top-down, so the tile's first k-iterations are its first unit;
// it parks the fp64 accumulators in a workspace slot and raises a flag; the
// upper CTA's last unit waits for the flag, reloads them and carries on with
// the next k.  Every element still sees one DMMA chain in ascending k from
// +0.0, so the result is bitwise the one-shot kernel's.  Needs each range to
// hold at least one tile's K (W/G >= KT), so a tile spans at most two CTAs.
// The per-element arithmetic is the same in all modes.
template <class K, int MODE>
__global__ void __launch_bounds__(K::THREADS, K::MINB)
    dgemm_dmma_kernel(const __grid_constant__ CUtensorMap tmA,
                      const __grid_constant__ CUtensorMap tmB, double* __restrict__ C,
                      int64_t ldc, int M, int N, int K_, int tiles_m, int tiles_n, int vec_ok,
                      int group, DmmaStream st) {
  // (MODE 3 reads st.cin -- possibly C itself -- only before the K loop and
  // writes C only after it, behind the pipeline's barriers)
  // MODE 3 = MODE 0 + accumulate (tiles start from st.cin); a separate
  // instantiation so the plain one-shot kernel's code is untouched
  constexpr bool STREAM = MODE == 1, SK = MODE == 2, ACC = MODE == 3;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // 1024-byte aligned ring (128B-swizzle atoms); offsetting the __shared__
  // array itself keeps the shared address space visible, so fragment fetches
  // compile to LDS rather than generic loads.
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + K::STAGES * K::STAGE_BYTES);
  uint64_t* empty = full + K::STAGES;

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  // Tile coordinates.  One-shot: grouped rasterisation (GROUP tile-rows advance
  // together so the A and B panels of one wave are shared through L2).
  // Streamed: the host's arrival-ordered list.
  auto raster = [&](int tile, int& tm, int& tn) {
    const int per_group = group * tiles_n;
    const int first_m = (tile / per_group) * group;
    const int gm = min(tiles_m - first_m, group);
    tm = first_m + (tile % per_group) % gm;
    tn = (tile % per_group) / gm;
  };
  auto tile_at = [&](int idx, int& tm, int& tn) {
    if constexpr (STREAM) {
      const int t = st.order[idx];
      tm = t / tiles_n;
      tn = t % tiles_n;
    } else {
      raster(SK ? idx : static_cast<int>(blockIdx.x), tm, tn);
    }
  };
  const int idx0 = STREAM ? static_cast<int>(blockIdx.x) : 0;
  const int n_idx = STREAM ? st.count : 1;
  const int idx_step = STREAM ? static_cast<int>(gridDim.x) : 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < K::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], K::CONSUMERS);
    }
    fence_barrier_init();
  }
  __syncthreads();

  const int KT = (K_ + K::BK - 1) / K::BK;

  // Work units: (tile, k-iterations [k0, k1)).  Modes 0/1: whole tiles in
  // list order.  Mode 2: this CTA's iteration range, top-down.
  const long long sk_w = static_cast<long long>(tiles_m) * tiles_n * KT;
  const long long sk_lo = SK ? sk_w * blockIdx.x / gridDim.x : 0;
  struct Cursor {
    int idx;
    long long pos;
  };
  auto next_unit = [&](Cursor& cur, int& tile, int& k0, int& k1) -> bool {
    if constexpr (SK) {
      if (cur.pos <= sk_lo) return false;
      tile = static_cast<int>((cur.pos - 1) / KT);
      const long long base = static_cast<long long>(tile) * KT;
      k0 = static_cast<int>((sk_lo > base ? sk_lo : base) - base);
      k1 = static_cast<int>(cur.pos - base);
      cur.pos = base + k0;
      return true;
    } else {
      if (cur.idx >= n_idx) return false;
      tile = cur.idx;
      cur.idx += idx_step;
      k0 = 0;
      k1 = KT;
      return true;
    }
  };
  const Cursor cur0{idx0, SK ? sk_w * (blockIdx.x + 1) / gridDim.x : 0};

  if (warp >= K::CONSUMERS) {
    // ---------------- TMA producer ----------------
    if constexpr (K::MATH_REGS > 0)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 40;");
    if (warp == K::CONSUMERS && lane == 0) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      int kg = 0;  // stage counter, continuous across tiles
      Cursor cur = cur0;
      int idx, k0, k1;
      while (next_unit(cur, idx, k0, k1)) {
        int tm, tn;
        tile_at(idx, tm, tn);
        if constexpr (STREAM) {
          wait_flag(st.ready_a + tm / st.band_a);
          wait_flag(st.ready_b + tn / st.band_b);
          asm volatile("fence.proxy.async.global;" ::: "memory");
        }
        for (int kt = k0; kt < k1; ++kt, ++kg) {
          const int s = kg % K::STAGES;
          if (kg >= K::STAGES) mbar_wait(&empty[s], ((kg / K::STAGES) - 1) & 1);
          uint8_t* sa = smem + s * K::STAGE_BYTES;
          uint8_t* sb = sa + K::A_BYTES;
          mbar_arrive_expect_tx(&full[s], K::STAGE_BYTES);
          tma_load_2d(sa, &tmA, &full[s], kt * K::BK, tm * K::BM);
#pragma unroll
          for (int b = 0; b < K::BN / 16; ++b)
            tma_load_2d(sb + b * 2048, &tmB, &full[s], tn * K::BN + b * 16, kt * K::BK);
        }
      }
    }
    return;
  }

  // ---------------- math warps ----------------
  if constexpr (K::MATH_REGS > 0)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(K::MATH_REGS));
  const int wm = warp % K::WARPS_M;
  const int wn = warp / K::WARPS_M;
  const int gid = lane >> 2, tig = lane & 3;
  const int sig = (gid >> 1) + ((gid & 1) << 2);

  // Per-lane byte offsets inside a stage.
  uint32_t a_off[K::MI];
#pragma unroll
  for (int i = 0; i < K::MI; ++i) a_off[i] = (wm * K::WM + i * 8 + sig) * 128;
  uint32_t a_chunk[2];
#pragma unroll
  for (int g8 = 0; g8 < 2; ++g8) a_chunk[g8] = ((g8 * 4 + tig) ^ sig) << 4;
  uint32_t b_off[2][2];  // [g8][q]: row (k) byte offset + swizzled chunk
#pragma unroll
  for (int g8 = 0; g8 < 2; ++g8)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      const int k = g8 * 8 + 2 * tig + q;
      b_off[g8][q] = k * 128 + ((gid ^ (k & 7)) << 4);
    }

  int kg = 0;  // stage counter, continuous across tiles
  Cursor cur = cur0;
  int idx, k0, k1;
  // stream-K workspace slot of this thread's accumulators (slot s holds the
  // tile cut by the boundary between CTAs s-1 and s)
  constexpr int ACC_PER_THREAD = K::MI * K::NB * 4;
  constexpr int MATH_THREADS = K::CONSUMERS * 32;
  while (next_unit(cur, idx, k0, k1)) {
    int tm, tn;
    tile_at(idx, tm, tn);
    double acc[K::MI][K::NB][2][2];
  #pragma unroll
    for (int i = 0; i < K::MI; ++i)
  #pragma unroll
      for (int b = 0; b < K::NB; ++b)
  #pragma unroll
        for (int e = 0; e < 2; ++e) acc[i][b][e][0] = acc[i][b][e][1] = 0.0;
    if constexpr (ACC) {
      {  // accumulate: continue Cin's chains (the epilogue's layout)
  #pragma unroll
        for (int i = 0; i < K::MI; ++i) {
          const int row = tm * K::BM + wm * K::WM + i * 8 + sig;
          if (row >= M) continue;
          const double* crow = st.cin + static_cast<int64_t>(row) * st.ldcin;
  #pragma unroll
          for (int b = 0; b < K::NB; ++b) {
            const int col = tn * K::BN + (wn * K::NB + b) * 16 + 4 * tig;
            if (vec_ok && col + 3 < N && (st.ldcin & 1) == 0 &&
                (reinterpret_cast<uintptr_t>(st.cin) & 15) == 0) {
              const double2 lo = __ldcg(reinterpret_cast<const double2*>(crow + col));
              const double2 hi = __ldcg(reinterpret_cast<const double2*>(crow + col) + 1);
              acc[i][b][0][0] = lo.x;
              acc[i][b][1][0] = lo.y;
              acc[i][b][0][1] = hi.x;
              acc[i][b][1][1] = hi.y;
            } else {
              acc[i][b][0][0] = col + 0 < N ? crow[col + 0] : 0.0;
              acc[i][b][1][0] = col + 1 < N ? crow[col + 1] : 0.0;
              acc[i][b][0][1] = col + 2 < N ? crow[col + 2] : 0.0;
              acc[i][b][1][1] = col + 3 < N ? crow[col + 3] : 0.0;
            }
          }
        }
      }
    }
    if constexpr (SK) {
      if (k0 > 0) {  // continue the lower CTA's accumulators for this tile
        if (threadIdx.x == 0) wait_flag(st.flags + blockIdx.x);
        asm volatile("bar.sync 1, %0;" ::"n"(MATH_THREADS) : "memory");
        const double* src = st.partial + static_cast<size_t>(blockIdx.x) * ACC_PER_THREAD * MATH_THREADS;
        double* a = &acc[0][0][0][0];
  #pragma unroll
        for (int j = 0; j < ACC_PER_THREAD; ++j) a[j] = __ldcg(src + j * MATH_THREADS + threadIdx.x);
        if (threadIdx.x == 0) st.flags[blockIdx.x] = 0;  // consumed: ready for the next launch
      }
    }

    for (int kt = k0; kt < k1; ++kt, ++kg) {
      const int s = kg % K::STAGES;
      mbar_wait(&full[s], (kg / K::STAGES) & 1);
      // Release the PREVIOUS stage here, not at the end of its own iteration:
      // ptxas sinks DMMAs below an arrive placed right after them, so the arrive
      // could retire while LDS of that stage are still in flight and the next
      // TMA would overwrite data being read.  Every DMMA of stage kt-1 sits in
      // the basic block before this wait loop and has issued -- so all of its
      // LDS have returned -- by the time we get here.
      if (kg > 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[(kg - 1) % K::STAGES]);
      }
      const uint8_t* sa = smem + s * K::STAGE_BYTES;
      const uint8_t* sb = sa + K::A_BYTES + (wn * K::NB) * 2048;
  #pragma unroll
      for (int g8 = 0; g8 < 2; ++g8) {
        double2 af[K::MI];
        double2 bf[K::NB][2];
  #pragma unroll
        for (int i = 0; i < K::MI; ++i)
          af[i] = *reinterpret_cast<const double2*>(sa + a_off[i] + a_chunk[g8]);
  #pragma unroll
        for (int b = 0; b < K::NB; ++b)
  #pragma unroll
          for (int q = 0; q < 2; ++q)
            bf[b][q] = *reinterpret_cast<const double2*>(sb + b * 2048 + b_off[g8][q]);
  #pragma unroll
        for (int q = 0; q < 2; ++q)
  #pragma unroll
          for (int i = 0; i < K::MI; ++i)
  #pragma unroll
            for (int b = 0; b < K::NB; ++b) {
              const double a = q ? af[i].y : af[i].x;
              dmma_8x8x4(acc[i][b][0][0], acc[i][b][0][1], a, q ? bf[b][1].x : bf[b][0].x);
              dmma_8x8x4(acc[i][b][1][0], acc[i][b][1][1], a, q ? bf[b][1].y : bf[b][0].y);
            }
      }

    }

    if constexpr (SK) {
      if (k1 < KT) {  // first part of a tile the upper CTA finishes: park it
        double* dst =
            st.partial + static_cast<size_t>(blockIdx.x + 1) * ACC_PER_THREAD * MATH_THREADS;
        const double* a = &acc[0][0][0][0];
  #pragma unroll
        for (int j = 0; j < ACC_PER_THREAD; ++j) __stcg(dst + j * MATH_THREADS + threadIdx.x, a[j]);
        asm volatile("bar.sync 1, %0;" ::"n"(MATH_THREADS) : "memory");
        if (threadIdx.x == 0) {
          __threadfence();
          set_flag(st.flags + blockIdx.x + 1, 1);
        }
        continue;
      }
    }

    // ---------------- epilogue: registers -> global ----------------
    // Lane owns row (.., sigma(gid)) and columns 4*tig .. 4*tig+3 of each box.
  #pragma unroll
    for (int i = 0; i < K::MI; ++i) {
      const int row = tm * K::BM + wm * K::WM + i * 8 + sig;
      if (row >= M) continue;
      double* crow = C + static_cast<int64_t>(row) * ldc;
  #pragma unroll
      for (int b = 0; b < K::NB; ++b) {
        const int col = tn * K::BN + (wn * K::NB + b) * 16 + 4 * tig;
        const double v0 = acc[i][b][0][0], v1 = acc[i][b][1][0];
        const double v2 = acc[i][b][0][1], v3 = acc[i][b][1][1];
        if (vec_ok && col + 3 < N) {
          reinterpret_cast<double2*>(crow + col)[0] = make_double2(v0, v1);
          reinterpret_cast<double2*>(crow + col)[1] = make_double2(v2, v3);
        } else {
          if (col + 0 < N) crow[col + 0] = v0;
          if (col + 1 < N) crow[col + 1] = v1;
          if (col + 2 < N) crow[col + 2] = v2;
          if (col + 3 < N) crow[col + 3] = v3;
        }
      }
    }
    if constexpr (STREAM) {
      // all math warps' stores of this tile are issued -> count the tile
      asm volatile("bar.sync 1, %0;" ::"n"(K::CONSUMERS * 32) : "memory");
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(st.done + tm, 1);
      }
    }
  }
}

// Raster group of configuration K; MMWS_GPU_RASTER_GROUP (read at init into
// Launch::raster_group) overrides it (tuning).
template <class K>
int raster_group(const Launch& L) {
  return L.raster_group > 0 ? L.raster_group : K::GROUP;
}

bool make_map(const Launch& L, CUtensorMap* map, const double* base, int64_t inner, int64_t outer,
              int64_t ld, int box_inner, int box_outer) {
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(double)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(box_inner),
                             static_cast<cuuint32_t>(box_outer)};
  const cuuint32_t estr[2] = {1, 1};
  return L.encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                  strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <class K>
cudaError_t run(const Launch& L, int64_t M, int64_t N, int64_t Kd, const double* A, int64_t lda,
                const double* B, int64_t ldb, double* C, int64_t ldc, const double* cin,
                int64_t ldcin) {
  CUtensorMap ta, tb;
  if (!make_map(L, &ta, A, Kd, M, lda, 16, K::BM)) return cudaErrorInvalidValue;
  if (!make_map(L, &tb, B, N, Kd, ldb, 16, 16)) return cudaErrorInvalidValue;
  const int smem = K::SMEM;
  const int tiles_m = static_cast<int>((M + K::BM - 1) / K::BM);
  const int tiles_n = static_cast<int>((N + K::BN - 1) / K::BN);
  cudaError_t e = cudaFuncSetAttribute(dgemm_dmma_kernel<K, 0>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int vec_ok = (ldc % 2 == 0) && (reinterpret_cast<uintptr_t>(C) % 16 == 0);
  DmmaStream st;
  st.cin = cin;
  st.ldcin = ldcin;
  auto kern = dgemm_dmma_kernel<K, 0>;
  if constexpr (K::MATH_REGS == 0) {  // accumulate: small-register plans only (below)
    if (cin) kern = dgemm_dmma_kernel<K, 3>;
  }
  if (cin && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)) !=
                 cudaSuccess)
    return e;
  kern<<<tiles_m * tiles_n, K::THREADS, smem, L.stream>>>(
      ta, tb, C, ldc, static_cast<int>(M), static_cast<int>(N), static_cast<int>(Kd), tiles_m,
      tiles_n, vec_ok, raster_group<K>(L), st);
  L.count();
  return cudaGetLastError();
}

template <class K>
cudaError_t run_sk(const Launch& L, int64_t M, int64_t N, int64_t Kd, const double* A, int64_t lda,
                   const double* B, int64_t ldb, double* C, int64_t ldc, double* partial,
                   int* flags, int grid) {
  CUtensorMap ta, tb;
  if (!make_map(L, &ta, A, Kd, M, lda, 16, K::BM)) return cudaErrorInvalidValue;
  if (!make_map(L, &tb, B, N, Kd, ldb, 16, 16)) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(dgemm_dmma_kernel<K, 2>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM);
  if (e != cudaSuccess) return e;
  const int tiles_m = static_cast<int>((M + K::BM - 1) / K::BM);
  const int tiles_n = static_cast<int>((N + K::BN - 1) / K::BN);
  const int vec_ok = (ldc % 2 == 0) && (reinterpret_cast<uintptr_t>(C) % 16 == 0);
  DmmaStream st;
  st.partial = partial;
  st.flags = flags;
  dgemm_dmma_kernel<K, 2><<<grid, K::THREADS, K::SMEM, L.stream>>>(
      ta, tb, C, ldc, static_cast<int>(M), static_cast<int>(N), static_cast<int>(Kd), tiles_m,
      tiles_n, vec_ok, raster_group<K>(L), st);
  L.count();
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_dgemm_dmma_stream(const Launch& L, int64_t M, int64_t N, int64_t Kd,
                                     const double* A, int64_t lda, const double* B, int64_t ldb,
                                     double* C, int64_t ldc, const DmmaStream& st, int grid) {
  using K = Big;
  CUtensorMap ta, tb;
  if (!make_map(L, &ta, A, Kd, M, lda, 16, K::BM)) return cudaErrorInvalidValue;
  if (!make_map(L, &tb, B, N, Kd, ldb, 16, 16)) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(dgemm_dmma_kernel<K, 1>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, K::SMEM);
  if (e != cudaSuccess) return e;
  const int tiles_m = static_cast<int>((M + K::BM - 1) / K::BM);
  const int tiles_n = static_cast<int>((N + K::BN - 1) / K::BN);
  const int vec_ok = (ldc % 2 == 0) && (reinterpret_cast<uintptr_t>(C) % 16 == 0);
  dgemm_dmma_kernel<K, 1><<<grid, K::THREADS, K::SMEM, L.stream>>>(
      ta, tb, C, ldc, static_cast<int>(M), static_cast<int>(N), static_cast<int>(Kd), tiles_m,
      tiles_n, vec_ok, raster_group<K>(L), st);
  L.count();
  return cudaGetLastError();
}

int dmma_tile_rows(int cfg) {
  switch (cfg) {
    case DMMA_64x64: case DMMA_64x64_W8: return 64;
    case DMMA_32x32: case DMMA_32x64: case DMMA_32x32_DEEP: return 32;
    case DMMA_16x16: return 16;
    default: return 128;
  }
}

int dmma_tile_cols(int cfg) {
  switch (cfg) {
    case DMMA_64x64: case DMMA_64x64_W8: case DMMA_128x64: case DMMA_32x64: return 64;
    case DMMA_32x32: case DMMA_32x32_DEEP: return 32;
    case DMMA_16x16: return 16;
    default: return 128;
  }
}

const char* dmma_plan_name(int cfg, int launch) {
  // [cfg][launch]: one-shot, stream-K
  static const char* const names[8][2] = {
      {"dgemm_dmma_kernel<128x128, 8 math warps, 1 CTA/SM>",
       "dgemm_dmma_kernel<128x128, 8 math warps, stream-K>"},
      {"dgemm_dmma_kernel<64x64, 4 math warps, 3 CTAs/SM>",
       "dgemm_dmma_kernel<64x64, 4 math warps, stream-K>"},
      {"dgemm_dmma_kernel<128x64, 8 math warps, 1 CTA/SM>",
       "dgemm_dmma_kernel<128x64, 8 math warps, stream-K>"},
      {"dgemm_dmma_kernel<64x64, 8 math warps, 1 CTA/SM>",
       "dgemm_dmma_kernel<64x64, 8 math warps, stream-K>"},
      {"dgemm_dmma_kernel<32x32, 4 math warps, 6 CTAs/SM>",
       "dgemm_dmma_kernel<32x32, 4 math warps, stream-K>"},
      {"dgemm_dmma_kernel<32x64, 4 math warps, 4 CTAs/SM>",
       "dgemm_dmma_kernel<32x64, 4 math warps, stream-K>"},
      {"dgemm_dmma_kernel<32x32, 4 math warps, 12 stages, 2 CTAs/SM>",
       "dgemm_dmma_kernel<32x32, 4 math warps, 12 stages, stream-K>"},
      {"dgemm_dmma_kernel<16x16, 2 math warps, 12 stages, 4 CTAs/SM>",
       "dgemm_dmma_kernel<16x16, 2 math warps, 12 stages, stream-K>"}};
  if (cfg < 0 || cfg > DMMA_16x16 || launch < 0 || launch > 1) return "dgemm_dmma_kernel<?>";
  return names[cfg][launch];
}


int dmma_ctas_per_sm(int cfg) {
  switch (cfg) {
    case DMMA_64x64: return Small::MINB;
    case DMMA_128x64: return Mid::MINB;
    case DMMA_64x64_W8: return Small8::MINB;
    case DMMA_32x32: return Tiny::MINB;
    case DMMA_32x64: return Slim::MINB;
    case DMMA_32x32_DEEP: return TinyDeep::MINB;
    case DMMA_16x16: return Micro::MINB;
    default: return Big::MINB;
  }
}

cudaError_t launch_dgemm_dmma_sk(const Launch& L, int cfg, int64_t M, int64_t N, int64_t Kd,
                                 const double* A, int64_t lda, const double* B, int64_t ldb,
                                 double* C, int64_t ldc, double* partial, int* flags, int grid) {
  switch (cfg) {
    case DMMA_64x64: return run_sk<Small>(L, M, N, Kd, A, lda, B, ldb, C, ldc, partial, flags, grid);
    case DMMA_128x64: return run_sk<Mid>(L, M, N, Kd, A, lda, B, ldb, C, ldc, partial, flags, grid);
    case DMMA_64x64_W8:
      return run_sk<Small8>(L, M, N, Kd, A, lda, B, ldb, C, ldc, partial, flags, grid);
    case DMMA_32x32: return run_sk<Tiny>(L, M, N, Kd, A, lda, B, ldb, C, ldc, partial, flags, grid);
    case DMMA_32x64: return run_sk<Slim>(L, M, N, Kd, A, lda, B, ldb, C, ldc, partial, flags, grid);
    case DMMA_32x32_DEEP:
      return run_sk<TinyDeep>(L, M, N, Kd, A, lda, B, ldb, C, ldc, partial, flags, grid);
    case DMMA_16x16: return run_sk<Micro>(L, M, N, Kd, A, lda, B, ldb, C, ldc, partial, flags, grid);
    default: return run_sk<Big>(L, M, N, Kd, A, lda, B, ldb, C, ldc, partial, flags, grid);
  }
}

cudaError_t launch_dgemm_dmma(const Launch& L, int cfg, int64_t M, int64_t N, int64_t K,
                              const double* A, int64_t lda, const double* B, int64_t ldb,
                              double* C, int64_t ldc, const double* cin, int64_t ldcin) {
  // Accumulating launches take the 4-math-warp plans: loading the 8-warp
  // plans' 64 accumulators per lane from Cin would spill (every plan gives the
  // same bits, so the choice is free).
  if (cin && (cfg == DMMA_128x128 || cfg == DMMA_128x64 || cfg == DMMA_64x64_W8)) cfg = DMMA_64x64;
  switch (cfg) {
    case DMMA_64x64: return run<Small>(L, M, N, K, A, lda, B, ldb, C, ldc, cin, ldcin);
    case DMMA_128x64: return run<Mid>(L, M, N, K, A, lda, B, ldb, C, ldc, cin, ldcin);
    case DMMA_64x64_W8: return run<Small8>(L, M, N, K, A, lda, B, ldb, C, ldc, cin, ldcin);
    case DMMA_32x32: return run<Tiny>(L, M, N, K, A, lda, B, ldb, C, ldc, cin, ldcin);
    case DMMA_32x64: return run<Slim>(L, M, N, K, A, lda, B, ldb, C, ldc, cin, ldcin);
    case DMMA_32x32_DEEP: return run<TinyDeep>(L, M, N, K, A, lda, B, ldb, C, ldc, cin, ldcin);
    case DMMA_16x16: return run<Micro>(L, M, N, K, A, lda, B, ldb, C, ldc, cin, ldcin);
    default: return run<Big>(L, M, N, K, A, lda, B, ldb, C, ldc, cin, ldcin);
  }
}

cudaError_t preload_dgemm_dmma() {
  return preload_kernels(dgemm_dmma_kernel<Big, 0>, dgemm_dmma_kernel<Mid, 0>,
                         dgemm_dmma_kernel<Small, 0>, dgemm_dmma_kernel<Big, 1>,
                         dgemm_dmma_kernel<Big, 2>, dgemm_dmma_kernel<Small, 2>,
                         dgemm_dmma_kernel<Mid, 2>,
                         dgemm_dmma_kernel<Small8, 0>, dgemm_dmma_kernel<Small8, 2>,
                         dgemm_dmma_kernel<Tiny, 0>, dgemm_dmma_kernel<Tiny, 2>,
                         dgemm_dmma_kernel<Slim, 0>, dgemm_dmma_kernel<Slim, 2>,
                         dgemm_dmma_kernel<TinyDeep, 0>, dgemm_dmma_kernel<TinyDeep, 2>,
                         dgemm_dmma_kernel<Micro, 0>, dgemm_dmma_kernel<Micro, 2>,
                         dgemm_dmma_kernel<Small, 3>,
                         dgemm_dmma_kernel<Tiny, 3>, dgemm_dmma_kernel<Slim, 3>,
                         dgemm_dmma_kernel<TinyDeep, 3>, dgemm_dmma_kernel<Micro, 3>);
}

}  // namespace mmws_impl

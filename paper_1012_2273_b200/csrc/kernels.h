// kernels.h -- internal (C++) launch interface between the C-ABI layer
// (mmws_gpu.cu) and the kernel translation units.  Not installed, not part of
// the drop-in surface; include/mmws_gpu.h is.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace mmws_impl {

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

struct Launch {
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  EncodeTiledFn encode = nullptr;
  uint64_t* launches = nullptr;  // bumped once per kernel launched
  int raster_group = 0;          // DMMA tile raster group override (0 = the plan's own)
  void count(int n = 1) const {
    if (launches) *launches += static_cast<uint64_t>(n);
  }
};

// DMMA tile configurations (see dgemm_dmma.cu / DESIGN.md s3).
enum DmmaCfg {
  DMMA_128x128 = 0,   // 8 math warps, 1 CTA/SM
  DMMA_64x64 = 1,     // 4 math warps, 3 CTAs/SM
  DMMA_128x64 = 2,    // 8 math warps
  DMMA_64x64_W8 = 3,  // 8 math warps on a 64x64 tile, 1 CTA/SM
  DMMA_32x32 = 4,     // 4 math warps, 6 CTAs/SM
  DMMA_32x64 = 5,     // 4 math warps, 4 CTAs/SM
  DMMA_32x32_DEEP = 6,  // 4 math warps, 12-stage ring, 2 CTAs/SM (few-tile grids)
  DMMA_16x16 = 7,       // 2 math warps, 12-stage ring, 4 CTAs/SM (few-tile grids)
};
// AUTO takes the 32x32 DFMA latency kernel when n and k are both <= this
// (a rule on (n, k) only, so row slices get the whole problem's bits).
constexpr int64_t AUTO_SMALL_MAX = 96;
int dmma_tile_rows(int cfg);
int dmma_tile_cols(int cfg);
int dmma_ctas_per_sm(int cfg);
// launch: 0 one-shot, 1 stream-K
const char* dmma_plan_name(int cfg, int launch);  // resident CTAs per SM the configuration is built for

// Streamed (persistent) DMMA schedule: tile list in arrival order, per-band
// arrival flags, per-tile-row completion counters (see dgemm_dmma.cu).
struct DmmaStream {
  const int* order = nullptr;    // tm * tiles_n + tn, processed in this order
  int count = 0;                 // entries in order
  const int* ready_a = nullptr;  // [tile-row band] != 0 once A's rows have landed
  const int* ready_b = nullptr;  // [tile-col band] != 0 once B's columns have landed
  int band_a = 1;                // tile rows per A band (ready_a granularity)
  int band_b = 1;                // tile columns per B band (ready_b granularity)
  int* done = nullptr;           // [tile row] finished tiles
  // stream-K (launch_dgemm_dmma_sk): accumulator slots and their flags,
  // grid + 1 of each (slot b = the tile cut between CTAs b-1 and b)
  double* partial = nullptr;
  int* flags = nullptr;
  // accumulate (one-shot launches): each tile's accumulators start from
  // Cin instead of +0.0, so C = Cin + A.B continues Cin's DMMA chains
  const double* cin = nullptr;
  int64_t ldcin = 0;
};
// fp64 GEMM emulated on the int8 tensor cores (ozaki.cu): plan (moduli s,
// integer bits t) for inner dimension k, workspace bytes, launch.  `aux` is a
// second stream for the tensor-core GEMMs and `ev` holds at least 5 events
// (timing disabled); the result is ordered on L.stream.
constexpr int OZAKI_EVENTS = 5;
void ozaki_plan(int64_t k, int* s, int* t);
size_t ozaki_workspace_bytes(int64_t m, int64_t n, int64_t k);
cudaError_t launch_dgemm_ozaki(const Launch& L, int64_t M, int64_t N, int64_t K, const double* A,
                               int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                               void* ws, cudaStream_t aux, cudaEvent_t* ev);
// fp32 operands / result through the same scheme (30-bit scaling)
void ozaki_plan_f32(int64_t k, int* s, int* t);
size_t ozaki_workspace_bytes_f32(int64_t m, int64_t n, int64_t k);
cudaError_t launch_sgemm_ozaki(const Launch& L, int64_t M, int64_t N, int64_t K, const float* A,
                               int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                               void* ws, cudaStream_t aux, cudaEvent_t* ev);
// Row-panel form (host pipeline): B's scaling and residues once into `ws`
// (sized by ozaki_workspace_bytes[_f32] for the tallest panel), then any
// number of A row panels against them, in order on one stream.  Each output
// row depends only on its own row of A, so panels give the one-shot bits.
cudaError_t launch_ozaki_prepare_b(const Launch& L, int64_t N, int64_t K, const double* B,
                                   int64_t ldb, void* ws);
cudaError_t launch_ozaki_prepare_b(const Launch& L, int64_t N, int64_t K, const float* B,
                                   int64_t ldb, void* ws);
cudaError_t launch_ozaki_panel(const Launch& L, int64_t M, int64_t N, int64_t K, const double* A,
                               int64_t lda, double* C, int64_t ldc, void* ws);
cudaError_t launch_ozaki_panel(const Launch& L, int64_t M, int64_t N, int64_t K, const float* A,
                               int64_t lda, float* C, int64_t ldc, void* ws);
// Force-load kernels (cudaFuncGetAttributes).  Under CUDA_MODULE_LOADING=LAZY
// the first launch of a kernel loads it with a context-wide synchronisation,
// which would wait forever on the resident latency server (and costs tens of
// ms inside a timed call): mmws_gpu_init preloads every kernel of the library.
template <class... F>
cudaError_t preload_kernels(F... f) {
  cudaFuncAttributes attr;
  cudaError_t e = cudaSuccess;
  ((e == cudaSuccess ? (e = cudaFuncGetAttributes(&attr, reinterpret_cast<const void*>(f))) : e),
   ...);
  return e;
}
cudaError_t preload_dgemm_dmma();
cudaError_t preload_ozaki();
cudaError_t preload_dgemm_exact();
cudaError_t preload_dgemm_small();
cudaError_t preload_sgemm_tma();
cudaError_t preload_misc();

// Stream-K, tiles of configuration cfg, grid persistent CTAs (all resident):
// every CTA gets the same number of k-iterations; bitwise the one-shot
// result.  Needs tiles * ceil(K/16) >= grid * ceil(K/16), i.e. tiles >= grid.
// partial: (grid + 1) * 128 * 128 doubles; flags: grid + 1 ints, zero before
// the first launch (the kernel leaves them zero).  Launches sharing a
// workspace must not overlap.
cudaError_t launch_dgemm_dmma_sk(const Launch& L, int cfg, int64_t M, int64_t N, int64_t K,
                                 const double* A, int64_t lda, const double* B, int64_t ldb,
                                 double* C, int64_t ldc, double* partial, int* flags, int grid);
// 128x128 tiles only; grid = number of persistent CTAs.
cudaError_t launch_dgemm_dmma_stream(const Launch& L, int64_t M, int64_t N, int64_t K,
                                     const double* A, int64_t lda, const double* B, int64_t ldb,
                                     double* C, int64_t ldc, const DmmaStream& st, int grid);

// C[M,N] = A[M,K] . B[K,N], row-major, accumulators from +0.0.  The TMA path
// needs lda, ldb even and A, B 16-byte aligned (the caller packs otherwise).
// cin (optional): accumulate, C = Cin + A.B with every element's chain
// continued from Cin (Cin may alias C); splitting K at multiples of 16 and
// chaining launches gives bitwise the one-launch result.
cudaError_t launch_dgemm_dmma(const Launch& L, int cfg, int64_t M, int64_t N, int64_t K,
                              const double* A, int64_t lda, const double* B, int64_t ldb,
                              double* C, int64_t ldc, const double* cin = nullptr,
                              int64_t ldcin = 0);

// Exact-order SIMT: per element acc = +0.0; for j ascending acc = (acc + a*b)
// with separate roundings -- bitwise equal to matmul_seq for every input.
// Exact-order stream-K (128x128 or 64x64 TMA kernel, `tile`; bitwise
// matmul_seq); same workspace contract as launch_dgemm_dmma_sk, tiles >= grid.
// exact_tma_ok: the layout the TMA kernels (and so this one) accept.
bool exact_tma_ok(int64_t lda, int64_t ldb, const double* A, const double* B);
// the kernel launch_dgemm_exact picks for these arguments (for last_plan)
const char* exact_oneshot_plan(const Launch& L, int64_t M, int64_t N, const double* A,
                               int64_t lda, const double* B, int64_t ldb);
cudaError_t launch_dgemm_exact_sk(const Launch& L, int tile, int64_t M, int64_t N, int64_t K,
                                  const double* A, int64_t lda, const double* B, int64_t ldb,
                                  double* C, int64_t ldc, double* partial, int* flags, int grid);
cudaError_t launch_dgemm_exact(const Launch& L, int64_t M, int64_t N, int64_t K,
                               const double* A, int64_t lda, const double* B, int64_t ldb,
                               double* C, int64_t ldc, const double* cin = nullptr,
                               int64_t ldcin = 0);

// Latency path: 32x32 tiles, plain loads, no TMA.  exact: DMUL+DADD chain
// (bitwise matmul_seq); otherwise one DFMA per step.
cudaError_t launch_dgemm_small(const Launch& L, bool exact, int64_t M, int64_t N, int64_t K,
                               const double* A, int64_t lda, const double* B, int64_t ldb,
                               double* C, int64_t ldc, const double* cin = nullptr,
                               int64_t ldcin = 0);

// Same chain on 16x16 tiles, one output per thread (more CTAs for tiny problems).
cudaError_t launch_dgemm_small16(const Launch& L, bool exact, int64_t M, int64_t N, int64_t K,
                                 const double* A, int64_t lda, const double* B, int64_t ldb,
                                 double* C, int64_t ldc, const double* cin = nullptr,
                                 int64_t ldcin = 0);

// TMA-fed, warp-specialised FFMA2 fp32 GEMM with two-level (chunked)
// accumulation (needs lda, ldb % 4 == 0 and 16-byte aligned A, B; the caller
// packs other layouts).
bool sgemm_tma_supported(int64_t lda, int64_t ldb, const float* A, const float* B);
// cin (optional): accumulate, C = Cin + A.B -- the running totals start from
// Cin; splitting K at multiples of 1024 (the partial-sum chunk) and chaining
// launches gives bitwise the one-launch result.
// a_transposed: A points at A^T ([K][M], pitch lda >= M, lda % 4 == 0) and is
// staged k-major.
cudaError_t launch_sgemm_tma(const Launch& L, int64_t M, int64_t N, int64_t K, const float* A,
                             int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                             const float* cin = nullptr, int64_t ldcin = 0,
                             bool a_transposed = false);
// dst[cols][rows] (pitch ld_dst) = src[rows][cols] (pitch ld_src, any alignment).
cudaError_t launch_transpose_f32(const Launch& L, const float* src, int64_t rows, int64_t cols,
                                 int64_t ld_src, float* dst, int64_t ld_dst);

// Pad/pack src[rows, cols] (ld_src) into dst[rows_p, cols_p] (ld_dst), zero fill.
cudaError_t launch_pack_f64(const Launch& L, const double* src, int64_t rows, int64_t cols,
                            int64_t ld_src, double* dst, int64_t rows_p, int64_t cols_p,
                            int64_t ld_dst);

// Store `value` into one progress word (device or peer-mapped), in stream order.
cudaError_t launch_board_mark(const Launch& L, unsigned* word, unsigned value);

cudaError_t launch_pack_f32(const Launch& L, const float* src, int64_t rows, int64_t cols,
                            int64_t ld_src, float* dst, int64_t rows_p, int64_t cols_p,
                            int64_t ld_dst);

// Counter-based splitmix64 generators (bit-identical to oracle_fill for dist 0..2).
cudaError_t launch_fill(const Launch& L, int dist, uint64_t seed, void* dst, int64_t rows,
                        int64_t cols, int64_t ld, int is_f32, uint64_t first);

// Peak probes: FP64 DMMA / DFMA / DMUL+DADD, FP32 FFMA loops (flops written to
// *flops, elapsed measured by the caller with events on L.stream).
cudaError_t launch_peak_probe(const Launch& L, int which, int iters, double* sink,
                              double* flops);

}  // namespace mmws_impl

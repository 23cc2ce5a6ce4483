// mmws_gpu.cu -- the C ABI (include/mmws_gpu.h): contexts, multiply dispatch,
// host-buffer entry points, CUDA-graph capture, generators, peak probes.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>

#include "../../include/mmws_gpu.h"
#include "ctx.h"
#include "kernels.h"
#include "nccl_dl.h"

namespace {
thread_local std::string g_last_error;
}

namespace mmws_impl {

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  return fail(MMWS_GPU_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
int ok() {
  g_last_error.clear();
  return MMWS_GPU_OK;
}

bool Tuning::set(const char* name, const char* v) {
  if (v && !*v) v = nullptr;
  const Tuning d;
  if (!std::strcmp(name, "MMWS_GPU_NO_STREAMK")) {
    no_streamk = v != nullptr;
  } else if (!std::strcmp(name, "MMWS_GPU_DMMA_PLAN")) {
    dmma_plan = v ? v : "";
  } else if (!std::strcmp(name, "MMWS_GPU_RASTER_GROUP")) {
    raster_group = v ? std::max(0, std::atoi(v)) : d.raster_group;
  } else if (!std::strcmp(name, "MMWS_GPU_PIPELINE_TRACE")) {
    pipeline_trace = v != nullptr;
  } else if (!std::strcmp(name, "MMWS_GPU_ROWBLOCK_RANKS")) {
    rowblock_ranks = !v ? 0 : std::strcmp(v, "all") == 0 ? -1 : std::strcmp(v, "1") == 0 ? 1 : 0;
  } else if (!std::strcmp(name, "MMWS_GPU_SERVER_CTAS")) {
    server_ctas = v ? std::atoi(v) : d.server_ctas;
  } else if (!std::strcmp(name, "MMWS_GPU_COPY_THREADS")) {
    copy_threads = v ? std::clamp(std::atoi(v), 1, 64) : d.copy_threads;
  } else if (!std::strcmp(name, "MMWS_GPU_HOST_PANELS")) {
    host_panels = v ? std::clamp(std::atoi(v), 0, 64) : d.host_panels;
  } else if (!std::strcmp(name, "MMWS_GPU_TIMEOUT_S")) {
    const double s = v ? std::atof(v) : 0.0;
    timeout_s = s > 0 ? s : d.timeout_s;
  } else if (!std::strcmp(name, "MMWS_GPU_NCCL_GATHER")) {
    nccl_gather = v != nullptr;
  } else if (!std::strcmp(name, "MMWS_GPU_SGEMM_AT")) {
    sgemm_at = v ? (std::atoi(v) != 0 ? 1 : 0) : d.sgemm_at;
  } else {
    return false;
  }
  return true;
}

Tuning Tuning::from_env() {
  Tuning t;
  for (const char* name : {"MMWS_GPU_NO_STREAMK", "MMWS_GPU_DMMA_PLAN", "MMWS_GPU_RASTER_GROUP",
                           "MMWS_GPU_PIPELINE_TRACE", "MMWS_GPU_ROWBLOCK_RANKS",
                           "MMWS_GPU_SERVER_CTAS", "MMWS_GPU_COPY_THREADS", "MMWS_GPU_HOST_PANELS",
                           "MMWS_GPU_TIMEOUT_S", "MMWS_GPU_NCCL_GATHER", "MMWS_GPU_SGEMM_AT"})
    if (const char* v = std::getenv(name)) t.set(name, v);
  return t;
}

cudaError_t ensure(mmws_gpu_ctx* ctx, void** buf, size_t* have, size_t bytes) {
  if (*have >= bytes && *buf) return cudaSuccess;
  if (*buf && ctx->server) {
    ctx->deferred_free.push_back(*buf);
    bytes = std::max(bytes, 2 * *have);
    *buf = nullptr;
    *have = 0;
  } else if (*buf) {
    cudaError_t e = cudaFree(*buf);
    if (e != cudaSuccess) return e;
    *buf = nullptr;
    *have = 0;
  }
  cudaError_t e = cudaMalloc(buf, bytes);
  if (e == cudaSuccess) *have = bytes;
  return e;
}

namespace {
inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

int check_dims(int64_t m, int64_t n, int64_t k, int64_t lda, int64_t ldb, int64_t ldc,
               const void* A, const void* B, const void* C) {
  if (m <= 0 || n <= 0 || k <= 0)
    return fail(MMWS_GPU_ERR_DIMENSION, "matmul: dimensions must be positive, got m=" +
                                            std::to_string(m) + " n=" + std::to_string(n) +
                                            " k=" + std::to_string(k));
  if (m > INT32_MAX || n > INT32_MAX || k > INT32_MAX)
    return fail(MMWS_GPU_ERR_DIMENSION, "matmul: dimension exceeds 2^31-1");
  if (lda < k || ldb < n || ldc < n)
    return fail(MMWS_GPU_ERR_DIMENSION, "matmul: leading dimension smaller than row length");
  if (!A || !B || !C) return fail(MMWS_GPU_ERR_DOMAIN, "matmul: null matrix pointer");
  return MMWS_GPU_OK;
}
}  // namespace

// The stream-K workspace of a launch stream: the flags of up to 4 persistent
// CTAs per SM (zeroed once on the stream; every launch leaves them zero), then
// accumulator slots -- (grid + 1) slots of BM x BN doubles, at most
// (num_sms + 1) x 128 x 128.  Allocated on first use and kept while the stream
// is among the 16 most recently used (trim_stream_spaces); fixed size, never
// moved, and graphs never use stream-K, so no replay holds a pointer to it.
int sk_workspace(mmws_gpu_ctx* ctx, cudaStream_t stream, double** partial, int** flags) {
  const size_t flag_bytes = round_up(sizeof(int) * (4 * static_cast<size_t>(ctx->num_sms) + 1), 4096);
  const size_t part_bytes = sizeof(double) * 128 * 128 * (static_cast<size_t>(ctx->num_sms) + 1);
  void* mem = nullptr;
  for (auto& sp : ctx->sk_spaces)
    if (sp.stream == stream) {
      mem = sp.mem;
      sp.last_use = ++ctx->space_clock;
    }
  if (!mem) {
    trim_stream_spaces(ctx, ctx->sk_spaces);
    cudaError_t e;
    if ((e = cudaMalloc(&mem, flag_bytes + part_bytes)) != cudaSuccess)
      return cuda_fail(e, "stream-K workspace");
    if ((e = cudaMemsetAsync(mem, 0, flag_bytes, stream)) != cudaSuccess) {
      cudaFree(mem);
      return cuda_fail(e, "stream-K workspace");
    }
    ctx->sk_spaces.push_back({stream, mem, ++ctx->space_clock});
  }
  *flags = static_cast<int*>(mem);
  *partial = reinterpret_cast<double*>(static_cast<char*>(mem) + flag_bytes);
  return MMWS_GPU_OK;
}

// MODE_OZAKI's second stream and ordering events (created on first use)
int ozaki_streams(mmws_gpu_ctx* ctx) {
  if (ctx->oz_stream) return MMWS_GPU_OK;
  cudaError_t e;
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  if ((e = cudaStreamCreateWithPriority(&ctx->oz_stream, cudaStreamNonBlocking, lo)) != cudaSuccess)
    return cuda_fail(e, "ozaki stream");
  for (int i = 0; i < OZAKI_EVENTS; ++i)
    if ((e = cudaEventCreateWithFlags(&ctx->oz_ev[i], cudaEventDisableTiming)) != cudaSuccess)
      return cuda_fail(e, "ozaki events");
  return MMWS_GPU_OK;
}

int dgemm_dispatch(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                   int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc, int mode,
                   cudaStream_t stream, const double* cin, int64_t ldcin) {
  if (int rc = check_dims(m, n, k, lda, ldb, ldc, A, B, C)) return rc;
  if (cin && ldcin < n)
    return fail(MMWS_GPU_ERR_DIMENSION, "matmul accumulate: leading dimension of Cin smaller than n");
  const Launch L = ctx->launch(stream);
  cudaError_t e;
  const int64_t tiles128 = ((m + 127) / 128) * ((n + 127) / 128);
  // Stream-K (128x128, one persistent CTA per SM, equal k-iterations per SM;
  // bitwise the one-shot result) from one tile per SM up to 32 waves, for
  // MODE_DMMA (128x128 tiles) and the exact mode: it beat the one-shot
  // 128x128 launch at every size measured there (N=1600: 30.0 vs 27.1
  // TFLOP/s, 2000: 32.6 vs 28.6, 2500: 33.3 vs 30.2, 4099: 32.7 vs 30.1,
  // 8192: 36.3 vs 36.0).  AUTO's small-tile plans beat both (below).  Not used
  //   * inside graph capture (the captured launch would share the stream's
  //     workspace with later eager launches),
  //   * while the latency server holds SMs (the grid would not be resident),
  //   * where the caller overlaps NCCL with the multiply (row-block path):
  //     persistent CTAs would keep the communication kernels off the SMs.
  const int64_t G = ctx->num_sms;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(L.stream, &cap);
  const bool sk_ok = cap == cudaStreamCaptureStatusNone && !ctx->server && ctx->allow_streamk &&
                     !ctx->tune.no_streamk && !cin;
  const bool sk = (mode == MMWS_GPU_MODE_DMMA || mode == MMWS_GPU_MODE_EXACT) && tiles128 >= G &&
                  tiles128 < 32 * G && sk_ok;
  // Exact order below one 128x128 tile per SM: stream-K over 64x64 tiles
  // (one CTA of 8 math warps per SM already fills the FP64 pipe) when the
  // one-shot 64x64 launch would leave the SMs unevenly loaded -- tiles per
  // SM rounded up more than ~10 % above the average.  GPU time per call
  // (tools/streamk_probe.py), stream-K vs one-shot: N=800 81.9 vs 122.8 us,
  // 900 115.5 vs 139.2, 1000 141.3 vs 153.5, 1100 192.5 vs 243.7, 1200 229.2
  // vs 262.0, 1400 353.1 vs 405.5; balanced sizes stay one-shot (1300 286.7
  // vs 301.8, 1500 432.1 vs 446.3).
  const int64_t tiles64 = ((m + 63) / 64) * ((n + 63) / 64);
  // latency kernels (plain loads, one chain per element): 16x16 tiles with
  // one output per thread while 32x32 tiles would not give every SM one --
  // 4x the CTAs; device time per call, 32x32 vs 16x16 (round 2): DFMA N=50
  // 6.2 vs 4.2 us, 64 6.2 vs 4.2, 96 7.0 vs 6.2; exact N=96 7.2 vs 6.2, 128
  // 8.2 vs 6.2, 160 10.3 vs 8.2, 256 14.4 vs 12.4; same chain, same bits
  const bool small16 = ((m + 31) / 32) * ((n + 31) / 32) < G;
  const bool sk64 = mode == MMWS_GPU_MODE_EXACT && tiles128 < G && tiles64 >= G && sk_ok &&
                    10 * tiles64 < 9 * (((tiles64 + G - 1) / G) * G);
  // TMA needs 16-byte aligned bases and even row pitches: pack A and/or B into
  // the workspace otherwise (one HBM-bound pass, zero padding never read).
  auto pack_operands = [&]() -> int {
    const bool a_ok = lda % 2 == 0 && reinterpret_cast<uintptr_t>(A) % 16 == 0;
    const bool b_ok = ldb % 2 == 0 && reinterpret_cast<uintptr_t>(B) % 16 == 0;
    if (a_ok && b_ok) return MMWS_GPU_OK;
    const int64_t lda_p = round_up(k, 8), ldb_p = round_up(n, 8);
    const size_t bytes = sizeof(double) * ((a_ok ? 0 : m * lda_p) + (b_ok ? 0 : k * ldb_p));
    void* wsp = nullptr;
    cudaError_t pe = workspace(ctx, bytes, &wsp, L.stream);
    if (pe != cudaSuccess) return cuda_fail(pe, "dgemm pack workspace");
    double* w = static_cast<double*>(wsp);
    if (!a_ok) {
      if ((pe = launch_pack_f64(L, A, m, k, lda, w, m, lda_p, lda_p)) != cudaSuccess)
        return cuda_fail(pe, "dgemm pack A");
      A = w;
      lda = lda_p;
      w += m * lda_p;
    }
    if (!b_ok) {
      if ((pe = launch_pack_f64(L, B, k, n, ldb, w, k, ldb_p, ldb_p)) != cudaSuccess)
        return cuda_fail(pe, "dgemm pack B");
      B = w;
      ldb = ldb_p;
    }
    return MMWS_GPU_OK;
  };
  double* sk_partial = nullptr;
  int* sk_flags = nullptr;
  if (mode == MMWS_GPU_MODE_EXACT) {
    // exact order: the latency kernels for tiny problems -- plain loads, any
    // layout -- up to n, k <= 192 (above that the 32x32 TMA tiles win;
    // device time per call, latency kernel vs 32x32 TMA, round 2: N=128 6.3
    // vs 7.1 us, 160 8.2 vs 8.3, 192 8.3 vs 8.5, 200 12.0 vs 10.3, 300 20.6
    // vs 12.4) and up
    // to 320 for layouts TMA cannot read; the stream-K form of the 128x128
    // TMA kernel (operands packed if needed) from one tile per SM, of the
    // 64x64 one below that where a one-shot launch would load the SMs
    // unevenly; else the 32x32 / 64x64 / 128x128 TMA kernels or the cp.async
    // kernel for layouts TMA cannot read -- every variant gives matmul_seq's
    // bits
    if ((n <= 192 && k <= 192) ||
        (n <= 320 && k <= 320 && !exact_tma_ok(lda, ldb, A, B))) {
      if (small16) {
        e = launch_dgemm_small16(L, true, m, n, k, A, lda, B, ldb, C, ldc, cin, ldcin);
        ctx->last_plan = "dgemm_small_kernel<exact, 16x16>";
      } else {
        e = launch_dgemm_small(L, true, m, n, k, A, lda, B, ldb, C, ldc, cin, ldcin);
        ctx->last_plan = "dgemm_small_kernel<exact, 32x32>";
      }
    } else if (sk || sk64) {
      if (int rc = sk_workspace(ctx, L.stream, &sk_partial, &sk_flags)) return rc;
      if (int rc = pack_operands()) return rc;
      e = launch_dgemm_exact_sk(L, sk ? 128 : 64, m, n, k, A, lda, B, ldb, C, ldc, sk_partial,
                                sk_flags, static_cast<int>(G));
      ctx->last_plan = sk ? "dgemm_exact_tma_kernel<128x128, stream-K>"
                          : "dgemm_exact_tma_kernel<64x64, stream-K>";
    } else {
      e = launch_dgemm_exact(L, m, n, k, A, lda, B, ldb, C, ldc, cin, ldcin);
      ctx->last_plan = exact_oneshot_plan(L, m, n, A, lda, B, ldb);
    }
    return e == cudaSuccess ? ok() : cuda_fail(e, "dgemm exact");
  }
  if (mode == MMWS_GPU_MODE_OZAKI) {
    // fp64 emulated on the int8 tensor cores (ozaki.cu); inputs read with
    // plain loads, so any layout works without packing
    if (cin) return fail(MMWS_GPU_ERR_DOMAIN, "matmul accumulate: not available in MODE_OZAKI");
    if (k > 131072)
      return fail(MMWS_GPU_ERR_DIMENSION, "dgemm ozaki: k must be <= 131072 (int32 accumulation)");
    void* wsp = nullptr;
    if ((e = workspace(ctx, ozaki_workspace_bytes(m, n, k), &wsp, L.stream)) != cudaSuccess)
      return cuda_fail(e, "dgemm ozaki workspace");
    if (int rc = ozaki_streams(ctx)) return rc;
    e = launch_dgemm_ozaki(L, m, n, k, A, lda, B, ldb, C, ldc, wsp, ctx->oz_stream, ctx->oz_ev);
    ctx->last_plan = "ozaki (int8 tcgen05 GEMMs + CRT)";
    return e == cudaSuccess ? ok() : cuda_fail(e, "dgemm ozaki");
  }
  if (mode != MMWS_GPU_MODE_AUTO && mode != MMWS_GPU_MODE_DMMA &&
      mode != MMWS_GPU_MODE_DMMA_SMALL)
    return fail(MMWS_GPU_ERR_DOMAIN, "dgemm: unknown mode " + std::to_string(mode));
  if (mode == MMWS_GPU_MODE_AUTO && n <= AUTO_SMALL_MAX && k <= AUTO_SMALL_MAX) {
    // latency path; chosen from (n, k) only, so every row slice of a problem
    // (row-block ranks, host-pipeline panels) takes the same kernel as the
    // whole problem and gets the same bits.  Above 96 the 32x32 DMMA tiles
    // are faster (GPU time per call: N=128 6.1 vs 8.2 us, 200 6.2 vs 12.3,
    // 256 8.2 vs 13.4; tools/dmma_plan_probe.py); up to 96 it stays, so the
    // latency server (server.cu, N <= 96, same DFMA chain) matches AUTO
    if (small16) {
      e = launch_dgemm_small16(L, false, m, n, k, A, lda, B, ldb, C, ldc, cin, ldcin);
      ctx->last_plan = "dgemm_small_kernel<DFMA, 16x16>";
    } else {
      e = launch_dgemm_small(L, false, m, n, k, A, lda, B, ldb, C, ldc, cin, ldcin);
      ctx->last_plan = "dgemm_small_kernel<DFMA, 32x32>";
    }
    return e == cudaSuccess ? ok() : cuda_fail(e, "dgemm small");
  }
  if (int rc = pack_operands()) return rc;
  // DMMA tile plan.  Every configuration computes each element as the same
  // DMMA chain in ascending k from +0.0, so the choice never changes the bits.
  // AUTO: 16x16 tiles below one 32x32 tile per SM (below), then
  // 32x32 tiles, 6 CTAs (24 math warps) per SM below three 128x128
  // tiles per SM; 64x64 tiles, 3 CTAs (12 math warps) per SM up to 64 tiles
  // per SM; 128x128 above.  GPU time per call, back to back
  // (tools/dmma_plan_probe.py, profiles/r01_dmma_plans.jsonl), against the
  // previous plan (64x64 with 2 CTAs/SM below 2 tiles per SM, then 128x128
  // stream-K / one-shot): N=500 14.4 vs 24.7 us, 1000 70.3 vs 74.6, 1500 205
  // vs 211, 2200 640 vs 667, 2700 1157 vs 1207, 3500 2461 vs 2508, 4099 4107
  // vs 4216, 8192 30.20 vs 30.34 ms, 10000 55.4 vs 57.3 ms.  More resident
  // math warps hide the DMMA and fragment-load latencies better than bigger
  // register tiles save operand traffic.  At N=16384 the 64x64 plan is only
  // 0.3-0.5 % faster (240.8 vs 241.9 ms) for 2.3x the DRAM reads (116 vs 50
  // GB), so the largest problems keep 128x128 tiles.  Stream-K over small
  // tiles lost to their one-shot launches at every size measured.
  // Below one 32x32 tile per SM (square N < ~390) AUTO takes 16x16 tiles
  // (2 math warps, 12-stage ring, 4 CTAs/SM): a lone tile's K loop is bound
  // by its dependent DMMA chains, so more, smaller tiles finish sooner --
  // GPU time per call (tools/dmma_plan_probe.py, profiles/r02_small_plans.jsonl)
  // 32x32 vs 16x16: N=100 5.8 vs 4.1 us, 128 6.1 vs 4.1, 160 6.2 vs 4.4,
  // 250 8.2 vs 6.2, 300 8.2 vs 7.2; from 400 on 32x32 wins (10.8 vs 12.3).
  const int64_t tiles32 = ((m + 31) / 32) * ((n + 31) / 32);
  int cfg = DMMA_128x128;
  if (mode == MMWS_GPU_MODE_AUTO && tiles32 < G)
    cfg = DMMA_16x16;
  else if (mode == MMWS_GPU_MODE_DMMA_SMALL || (mode == MMWS_GPU_MODE_AUTO && tiles128 < 3 * G))
    cfg = DMMA_32x32;
  else if (mode == MMWS_GPU_MODE_AUTO && tiles128 < 64 * G)
    cfg = DMMA_64x64;
  int sk_grid = sk ? static_cast<int>(G) : 0;
  if (!ctx->tune.dmma_plan.empty()) {
    const char* plan = ctx->tune.dmma_plan.c_str();
    // tuning override (tools/dmma_plan_probe.py): "<cfg>" one-shot, or
    // "<cfg>s<CTAs per SM>" stream-K
    char* end = nullptr;
    cfg = static_cast<int>(std::strtol(plan, &end, 10));
    sk_grid = end && *end == 's' ? static_cast<int>(G * std::strtol(end + 1, nullptr, 10)) : 0;
    const int64_t tiles = ((m + dmma_tile_rows(cfg) - 1) / dmma_tile_rows(cfg)) *
                          ((n + dmma_tile_cols(cfg) - 1) / dmma_tile_cols(cfg));
    // stream-K needs every CTA resident (a CTA may wait on its lower
    // neighbour), a whole tile per CTA, and workspace slots for the grid
    if (cfg < DMMA_128x128 || cfg > DMMA_16x16 || sk_grid < 0 ||
        (sk_grid > 0 && (sk_grid > 4 * G || sk_grid > G * dmma_ctas_per_sm(cfg) || tiles < sk_grid ||
                         static_cast<int64_t>(sk_grid) * dmma_tile_rows(cfg) * dmma_tile_cols(cfg) >
                             G * 128 * 128)))
      return fail(MMWS_GPU_ERR_DOMAIN, std::string("MMWS_GPU_DMMA_PLAN not usable here: ") + plan);
  }
  if (sk_grid > 0 && cin)
    return fail(MMWS_GPU_ERR_DOMAIN, "matmul accumulate: stream-K plans do not take Cin");
  if (sk_grid > 0) {
    if (int rc = sk_workspace(ctx, L.stream, &sk_partial, &sk_flags)) return rc;
    e = launch_dgemm_dmma_sk(L, cfg, m, n, k, A, lda, B, ldb, C, ldc, sk_partial, sk_flags,
                             sk_grid);
    ctx->last_plan = dmma_plan_name(cfg, 1);
    return e == cudaSuccess ? ok() : cuda_fail(e, "dgemm stream-K");
  }
  // accumulating launches run on the 4-math-warp plans (dgemm_dmma.cu)
  if (cin && (cfg == DMMA_128x128 || cfg == DMMA_128x64 || cfg == DMMA_64x64_W8)) cfg = DMMA_64x64;
  e = launch_dgemm_dmma(L, cfg, m, n, k, A, lda, B, ldb, C, ldc, cin, ldcin);
  ctx->last_plan = dmma_plan_name(cfg, 0);
  return e == cudaSuccess ? ok() : cuda_fail(e, "dgemm dmma");
}

int sgemm_dispatch(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const float* A,
                   int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int mode,
                   cudaStream_t stream, const float* cin, int64_t ldcin) {
  if (int rc = check_dims(m, n, k, lda, ldb, ldc, A, B, C)) return rc;
  if (cin && ldcin < n)
    return fail(MMWS_GPU_ERR_DIMENSION, "matmul accumulate: leading dimension of Cin smaller than n");
  if (mode != MMWS_GPU_MODE_AUTO && mode != MMWS_GPU_MODE_FFMA && mode != MMWS_GPU_MODE_OZAKI)
    return fail(MMWS_GPU_ERR_DOMAIN, "sgemm: unknown mode " + std::to_string(mode));
  const Launch L = ctx->launch(stream);
  if (mode == MMWS_GPU_MODE_OZAKI && cin)
    return fail(MMWS_GPU_ERR_DOMAIN, "matmul accumulate: not available in MODE_OZAKI");
  if (mode == MMWS_GPU_MODE_OZAKI) {  // fp32 through the int8 tensor-core scheme (ozaki.cu)
    if (k > 131072)
      return fail(MMWS_GPU_ERR_DIMENSION, "sgemm ozaki: k must be <= 131072 (int32 accumulation)");
    cudaError_t e;
    void* wsp = nullptr;
    if ((e = workspace(ctx, ozaki_workspace_bytes_f32(m, n, k), &wsp, L.stream)) != cudaSuccess)
      return cuda_fail(e, "sgemm ozaki workspace");
    if (int rc = ozaki_streams(ctx)) return rc;
    e = launch_sgemm_ozaki(L, m, n, k, A, lda, B, ldb, C, ldc, wsp, ctx->oz_stream, ctx->oz_ev);
    ctx->last_plan = "ozaki f32 (int8 tcgen05 GEMMs + CRT)";
    return e == cudaSuccess ? ok() : cuda_fail(e, "sgemm ozaki");
  }
  // TMA needs 16-byte aligned bases and row pitches that are multiples of 4
  // floats: other layouts are packed once into the workspace (one HBM-bound
  // pass, zero padding never read), so every layout runs the same kernel --
  // and gets the same bits.
  //
  // Wide problems take A transposed: one more HBM-bound pass writes A^T into
  // the workspace (any layout of A), and the kernel stages A k-major, which
  // keeps every row's A scalar in one register bank (sgemm_tma.cu; +6 % FFMA2
  // rate).  The pass costs 8mk bytes against 2mnk flops, ~40/n of the
  // multiply: taken from n = 2048.  Same FFMA chain per element either way,
  // so the same bits.
  cudaError_t e;
  const bool a_t = ctx->tune.sgemm_at < 0 ? n >= 2048 && m >= 128 : ctx->tune.sgemm_at == 1;
  const bool a_aligned = a_t || (lda % 4 == 0 && reinterpret_cast<uintptr_t>(A) % 16 == 0);
  const bool b_aligned = ldb % 4 == 0 && reinterpret_cast<uintptr_t>(B) % 16 == 0;
  if (a_t || !a_aligned || !b_aligned) {
    const int64_t lda_p = round_up(k, 4), ldb_p = round_up(n, 4), ldat = round_up(m, 4);
    const size_t bytes = sizeof(float) * ((a_t ? k * ldat : a_aligned ? 0 : m * lda_p) +
                                          (b_aligned ? 0 : k * ldb_p));
    void* wsp = nullptr;
    if ((e = workspace(ctx, bytes, &wsp, L.stream)) != cudaSuccess) return cuda_fail(e, "sgemm pack workspace");
    float* w = static_cast<float*>(wsp);
    if (a_t) {
      if ((e = launch_transpose_f32(L, A, m, k, lda, w, ldat)) != cudaSuccess)
        return cuda_fail(e, "sgemm transpose A");
      A = w;
      lda = ldat;
      w += k * ldat;
    } else if (!a_aligned) {
      if ((e = launch_pack_f32(L, A, m, k, lda, w, m, lda_p, lda_p)) != cudaSuccess)
        return cuda_fail(e, "sgemm pack A");
      A = w;
      lda = lda_p;
      w += m * lda_p;
    }
    if (!b_aligned) {
      if ((e = launch_pack_f32(L, B, k, n, ldb, w, k, ldb_p, ldb_p)) != cudaSuccess)
        return cuda_fail(e, "sgemm pack B");
      B = w;
      ldb = ldb_p;
    }
  }
  e = launch_sgemm_tma(L, m, n, k, A, lda, B, ldb, C, ldc, cin, ldcin, a_t);
  ctx->last_plan = a_t ? "sgemm_tma_kernel<128x256, FFMA2, A k-major>" : "sgemm_tma_kernel<128x256, FFMA2>";
  return e == cudaSuccess ? ok() : cuda_fail(e, "sgemm ffma");
}

int ipc_export(mmws_gpu_ctx* ctx, const void* ptr, uint8_t out[72]) {
  if (!ptr || !out) return fail(MMWS_GPU_ERR_DOMAIN, "ipc_export: null argument");
  if (!ctx->mem_range) return fail(MMWS_GPU_ERR_STATE, "ipc_export: cuMemGetAddressRange unavailable");
  CUdeviceptr base = 0;
  size_t size = 0;
  if (ctx->mem_range(&base, &size, static_cast<CUdeviceptr>(reinterpret_cast<uintptr_t>(ptr))) !=
      CUDA_SUCCESS)
    return fail(MMWS_GPU_ERR_CUDA, "ipc_export: pointer is not a device allocation");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(static_cast<uintptr_t>(base)));
  if (e != cudaSuccess) return cuda_fail(e, "ipc_export: cudaIpcGetMemHandle");
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
  const uint64_t offset = reinterpret_cast<uintptr_t>(ptr) - static_cast<uintptr_t>(base);
  std::memcpy(out, &h, 64);
  std::memcpy(out + 64, &offset, 8);
  return ok();
}

void ipc_close_scoped(mmws_gpu_ctx* ctx) {
  for (auto it = ctx->ipc_cache.begin(); it != ctx->ipc_cache.end();) {
    if (it->scope != IPC_CALLER) {
      cudaIpcCloseMemHandle(it->base);
      it = ctx->ipc_cache.erase(it);
    } else {
      ++it;
    }
  }
}

int ipc_open(mmws_gpu_ctx* ctx, const uint8_t in[72], void** ptr, int scope) {
  if (!in || !ptr) return fail(MMWS_GPU_ERR_DOMAIN, "ipc_open: null argument");
  uint64_t offset = 0;
  std::memcpy(&offset, in + 64, 8);
  ++ctx->ipc_clock;
  for (auto& mp : ctx->ipc_cache)
    if (std::memcmp(mp.handle, in, 64) == 0) {
      mp.last_use = ctx->ipc_clock;
      if (scope == IPC_CALLER) mp.scope = IPC_CALLER;  // the caller's own mapping stays
      *ptr = static_cast<char*>(mp.base) + offset;
      return ok();
    }
  if (scope == IPC_ROUND) {  // evict the least recently used round mappings
    for (;;) {
      int n = 0;
      auto lru = ctx->ipc_cache.end();
      for (auto it = ctx->ipc_cache.begin(); it != ctx->ipc_cache.end(); ++it)
        if (it->scope == IPC_ROUND) {
          ++n;
          if (lru == ctx->ipc_cache.end() || it->last_use < lru->last_use) lru = it;
        }
      if (n < IPC_ROUND_MAPPINGS) break;
      cudaIpcCloseMemHandle(lru->base);
      ctx->ipc_cache.erase(lru);
    }
  }
  cudaIpcMemHandle_t h;
  std::memcpy(&h, in, 64);
  void* base = nullptr;
  cudaError_t e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  if (e == cudaErrorAlreadyMapped && scope != IPC_CALLER) {
    // The exporter freed an allocation we still map and reallocated at its
    // address (a fresh C per round): the stale round mappings are idle
    // (rounds are synchronous) -- close them and map the new one.
    cudaGetLastError();
    for (auto it = ctx->ipc_cache.begin(); it != ctx->ipc_cache.end();) {
      if (it->scope == IPC_ROUND) {
        cudaIpcCloseMemHandle(it->base);
        it = ctx->ipc_cache.erase(it);
      } else {
        ++it;
      }
    }
    e = cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess);
  }
  if (e != cudaSuccess) return cuda_fail(e, "ipc_open: cudaIpcOpenMemHandle");
  mmws_gpu_ctx::IpcMap mp;
  std::memcpy(mp.handle, in, 64);
  mp.base = base;
  mp.scope = scope;
  mp.last_use = ctx->ipc_clock;
  ctx->ipc_cache.push_back(mp);
  *ptr = static_cast<char*>(base) + offset;
  return ok();
}

}  // namespace mmws_impl

using namespace mmws_impl;

struct mmws_gpu_graph {
  mmws_gpu_ctx* ctx = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  uint64_t kernels = 0;
  void* ws = nullptr;  // this graph's own packing / MODE_OZAKI workspace
  size_t ws_bytes = 0;
};

namespace {
// Device resources of a graph (its context's lock held).
void graph_release(mmws_gpu_ctx* ctx, mmws_gpu_graph* g) {
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  g->exec = nullptr;
  g->graph = nullptr;
  if (g->ws) {
    // a replay may still be running: free after the context's work, or at
    // server stop while the latency server holds the device
    if (ctx->server) ctx->deferred_free.push_back(g->ws);
    else cudaDeviceSynchronize(), cudaFree(g->ws);
    g->ws = nullptr;
  }
}

// The NCCL stream gets the highest priority so its CTAs are scheduled ahead of
// pending GEMM CTAs whenever an SM frees up -- otherwise the C gather of a
// finished sub-block would wait for the whole next multiply.
cudaError_t create_comm_stream(cudaStream_t* s) {
  int least = 0, greatest = 0;
  cudaError_t e = cudaDeviceGetStreamPriorityRange(&least, &greatest);
  if (e != cudaSuccess) return e;
  return cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, greatest);
}
}  // namespace

extern "C" {

int mmws_gpu_abi_version(void) { return MMWS_GPU_ABI_VERSION; }

const char* mmws_gpu_last_error(void) { return g_last_error.c_str(); }

int mmws_gpu_init(int device, mmws_gpu_ctx** out) {
  if (!out) return fail(MMWS_GPU_ERR_DOMAIN, "mmws_gpu_init: null out pointer");
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess) return cuda_fail(e, "mmws_gpu_init: no CUDA device");
  if (device < 0 || device >= count)
    return fail(MMWS_GPU_ERR_DOMAIN, "mmws_gpu_init: device " + std::to_string(device) +
                                         " out of range (" + std::to_string(count) + ")");
  if ((e = cudaSetDevice(device)) != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
  cudaDeviceProp prop;
  if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess)
    return cuda_fail(e, "cudaGetDeviceProperties");
  if (prop.major != 10)
    return fail(MMWS_GPU_ERR_STATE, std::string("mmws_gpu_init: built for sm_100a, device is ") +
                                        prop.name + " (sm_" + std::to_string(prop.major) +
                                        std::to_string(prop.minor) + ")");
  // Load every kernel of the library now: under CUDA_MODULE_LOADING=LAZY (the
  // default) a kernel's first launch would otherwise pay its module load
  // inside the caller's timed region (~70 ms on the first streamed host
  // multiply at N=16384), and the latency server relies on it (server.cu).
  if ((e = preload_dgemm_dmma()) || (e = preload_dgemm_exact()) || (e = preload_dgemm_small()) ||
      (e = preload_sgemm_tma()) || (e = preload_misc()) ||
      (e = preload_ozaki()))
    return cuda_fail(e, "mmws_gpu_init: load kernels");
  auto* ctx = new (std::nothrow) mmws_gpu_ctx();
  if (!ctx) return fail(MMWS_GPU_ERR_ALLOC, "mmws_gpu_init: out of host memory");
  ctx->device = device;
  ctx->tune = Tuning::from_env();
  ctx->num_sms = prop.multiProcessorCount;
  ctx->cc_major = prop.major;
  ctx->cc_minor = prop.minor;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
  ctx->clock_khz = clk;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn) {
    delete ctx;
    return fail(MMWS_GPU_ERR_CUDA, "mmws_gpu_init: cuTensorMapEncodeTiled unavailable");
  }
  ctx->encode = reinterpret_cast<EncodeTiledFn>(fn);
  void* mr = nullptr;
  if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &mr, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    ctx->mem_range = reinterpret_cast<decltype(ctx->mem_range)>(mr);
  void* wr = nullptr;
  void* wt = nullptr;
  if (cudaGetDriverEntryPoint("cuStreamWriteValue32", &wr, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess &&
      cudaGetDriverEntryPoint("cuStreamWaitValue32", &wt, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess && wr && wt) {
    ctx->write_value = reinterpret_cast<decltype(ctx->write_value)>(wr);
    ctx->wait_value = reinterpret_cast<decltype(ctx->wait_value)>(wt);
  }
  if ((e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = create_comm_stream(&ctx->comm_stream)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&ctx->copy_in, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&ctx->copy_out, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaEventCreate(&ctx->ev0)) != cudaSuccess ||
      (e = cudaEventCreate(&ctx->ev1)) != cudaSuccess ||
      (e = cudaEventCreate(&ctx->evk0)) != cudaSuccess ||
      (e = cudaEventCreate(&ctx->evk1)) != cudaSuccess ||
      (e = cudaMalloc(&ctx->sink, 4096 * sizeof(double))) != cudaSuccess ||
      (e = cudaMalloc(&ctx->ipc_stage, 256)) != cudaSuccess ||
      (e = cudaHostAlloc(reinterpret_cast<void**>(&ctx->host_stage), 512,
                         cudaHostAllocDefault)) != cudaSuccess) {
    mmws_gpu_destroy(ctx);
    return cuda_fail(e, "mmws_gpu_init");
  }
  *out = ctx;
  return ok();
}

int mmws_gpu_destroy(mmws_gpu_ctx* ctx) {
  if (!ctx) return ok();
  cudaSetDevice(ctx->device);
  server_destroy(ctx);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  for (mmws_gpu_graph* g : ctx->graphs) {  // detach: the caller still owns the handles
    graph_release(ctx, g);
    g->ctx = nullptr;
  }
  ctx->graphs.clear();
  if (ctx->comm && nccl().ok) nccl().CommDestroy(ctx->comm);
  for (auto& mp : ctx->ipc_cache) cudaIpcCloseMemHandle(mp.base);
  for (const auto& w : ctx->ws_spaces)
    if (w.mem) cudaFree(w.mem);
  for (void* p : {ctx->dA, ctx->dB, ctx->dC, ctx->rbA, ctx->rbB, ctx->rbC, ctx->rbAcc, ctx->sched,
                  ctx->ipc_stage, static_cast<void*>(ctx->board),
                  static_cast<void*>(ctx->sink)})
    if (p) cudaFree(p);
  for (void* p : ctx->deferred_free) cudaFree(p);
  if (ctx->host_stage) cudaFreeHost(ctx->host_stage);
  if (ctx->tiny_host) cudaFreeHost(ctx->tiny_host);
  for (const auto& sp : ctx->sk_spaces) cudaFree(sp.mem);
  staging_destroy(ctx);
  if (ctx->ev0) cudaEventDestroy(ctx->ev0);
  if (ctx->ev1) cudaEventDestroy(ctx->ev1);
  if (ctx->evk0) cudaEventDestroy(ctx->evk0);
  if (ctx->evk1) cudaEventDestroy(ctx->evk1);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  if (ctx->copy_in) cudaStreamDestroy(ctx->copy_in);
  if (ctx->copy_out) cudaStreamDestroy(ctx->copy_out);
  if (ctx->oz_stream) cudaStreamDestroy(ctx->oz_stream);
  for (cudaEvent_t ev : ctx->oz_ev)
    if (ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : ctx->pool) cudaEventDestroy(ev);
  delete ctx;
  return ok();
}

int mmws_gpu_device_info(mmws_gpu_ctx* ctx, int* num_sms, int* cc_major, int* cc_minor,
                         int* max_clock_khz) {
  if (!ctx) return fail(MMWS_GPU_ERR_STATE, "null mmws_gpu_ctx");
  if (num_sms) *num_sms = ctx->num_sms;
  if (cc_major) *cc_major = ctx->cc_major;
  if (cc_minor) *cc_minor = ctx->cc_minor;
  if (max_clock_khz) *max_clock_khz = ctx->clock_khz;
  return ok();
}

uint64_t mmws_gpu_launch_count(const mmws_gpu_ctx* ctx) { return ctx ? ctx->launches : 0; }

void* mmws_gpu_stream(mmws_gpu_ctx* ctx) { return ctx ? static_cast<void*>(ctx->stream) : nullptr; }

int mmws_gpu_tune(mmws_gpu_ctx* ctx, const char* knob, const char* value) {
  MMWS_CTX_GUARD(ctx);
  if (!knob) return fail(MMWS_GPU_ERR_DOMAIN, "tune: null knob name");
  if (!ctx->tune.set(knob, value))
    return fail(MMWS_GPU_ERR_DOMAIN, std::string("tune: unknown knob ") + knob);
  return ok();
}

// ------------------------------------------------------------------ host-only helpers
int mmws_gpu_split_rows(int64_t n_rows, int n_workers, int64_t* offset, int64_t* rows) {
  // protocol.hpp:33-46
  if (n_workers < 1) return fail(MMWS_GPU_ERR_DOMAIN, "split_rows: need at least one worker");
  if (n_rows < 0) return fail(MMWS_GPU_ERR_DOMAIN, "split_rows: negative row count");
  if (!offset || !rows) return fail(MMWS_GPU_ERR_DOMAIN, "split_rows: null output");
  const int64_t averow = n_rows / n_workers, extra = n_rows % n_workers;
  int64_t off = 0;
  for (int w = 0; w < n_workers; ++w) {
    offset[w] = off;
    rows[w] = averow + (w < extra ? 1 : 0);
    off += rows[w];
  }
  return ok();
}

int mmws_gpu_static_partition(uint64_t iterations, uint32_t workers, uint64_t* start,
                              uint64_t* len) {
  // workshare.hpp:33-46
  if (workers == 0)
    return fail(MMWS_GPU_ERR_DOMAIN, "static_partition: worker count must be >= 1");
  if (!start || !len) return fail(MMWS_GPU_ERR_DOMAIN, "static_partition: null output");
  const uint64_t base = iterations / workers, extra = iterations % workers;
  uint64_t s = 0;
  for (uint32_t w = 0; w < workers; ++w) {
    start[w] = s;
    len[w] = base + (w < extra ? 1 : 0);
    s += len[w];
  }
  return ok();
}

int mmws_gpu_op_count(int64_t n, uint64_t* out) {
  // matrix.hpp:130-134
  if (n < 1) return fail(MMWS_GPU_ERR_DOMAIN, "op_count: N must be >= 1, got " + std::to_string(n));
  if (!out) return fail(MMWS_GPU_ERR_DOMAIN, "op_count: null output");
  const uint64_t un = static_cast<uint64_t>(n);
  *out = un * un * (2 * un - 1);
  return ok();
}

// ------------------------------------------------------------------ multiply
int mmws_gpu_dgemm(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                   int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc, int mode,
                   void* stream) {
  MMWS_CTX_GUARD(ctx);
  return dgemm_dispatch(ctx, m, n, k, A, lda, B, ldb, C, ldc, mode,
                        static_cast<cudaStream_t>(stream));
}

int mmws_gpu_sgemm(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const float* A,
                   int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int mode,
                   void* stream) {
  MMWS_CTX_GUARD(ctx);
  return sgemm_dispatch(ctx, m, n, k, A, lda, B, ldb, C, ldc, mode,
                        static_cast<cudaStream_t>(stream));
}

int mmws_gpu_dgemm_acc(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                       int64_t lda, const double* B, int64_t ldb, const double* Cin,
                       int64_t ldcin, double* C, int64_t ldc, int mode, void* stream) {
  MMWS_CTX_GUARD(ctx);
  if (!Cin) return fail(MMWS_GPU_ERR_DOMAIN, "dgemm_acc: null Cin");
  return dgemm_dispatch(ctx, m, n, k, A, lda, B, ldb, C, ldc, mode,
                        static_cast<cudaStream_t>(stream), Cin, ldcin);
}

int mmws_gpu_sgemm_acc(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const float* A,
                       int64_t lda, const float* B, int64_t ldb, const float* Cin, int64_t ldcin,
                       float* C, int64_t ldc, int mode, void* stream) {
  MMWS_CTX_GUARD(ctx);
  if (!Cin) return fail(MMWS_GPU_ERR_DOMAIN, "sgemm_acc: null Cin");
  return sgemm_dispatch(ctx, m, n, k, A, lda, B, ldb, C, ldc, mode,
                        static_cast<cudaStream_t>(stream), Cin, ldcin);
}

int mmws_gpu_ozaki_plan(int64_t k, int* moduli, int* bits) {
  if (k < 1 || k > 131072 || !moduli || !bits)
    return fail(MMWS_GPU_ERR_DOMAIN, "ozaki_plan: k must be in [1, 131072], outputs non-null");
  ozaki_plan(k, moduli, bits);
  return ok();
}

int mmws_gpu_matmul_host(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                         const double* B, double* C, int mode, double* elapsed_s) {
  MMWS_CTX_GUARD(ctx);
  if (A && B && C && server_serves(ctx, m, n, k, mode))  // resident server (server.cu)
    return server_multiply(ctx, m, n, k, A, k, B, n, C, n, mode, elapsed_s);
  return host_multiply(ctx, m, n, k, A, B, C, mode, elapsed_s);
}

int mmws_gpu_matmul_host_f32(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k,
                             const float* A, const float* B, float* C, int mode,
                             double* elapsed_s) {
  MMWS_CTX_GUARD(ctx);
  return host_multiply(ctx, m, n, k, A, B, C, mode, elapsed_s);
}

// ------------------------------------------------------------------ generators
int mmws_gpu_fill(mmws_gpu_ctx* ctx, int dist, uint64_t seed, void* dst, int64_t rows,
                  int64_t cols, int64_t ld, int is_f32, uint64_t first, void* stream) {
  MMWS_CTX_GUARD(ctx);
  if (rows <= 0 || cols <= 0 || ld < cols)
    return fail(MMWS_GPU_ERR_DIMENSION, "fill: bad shape");
  if (dist < 0 || dist > 3 || (dist == MMWS_GPU_DIST_NORMAL && !is_f32) || !dst)
    return fail(MMWS_GPU_ERR_DOMAIN, "fill: bad distribution / dtype / pointer");
  cudaError_t e = launch_fill(ctx->launch(static_cast<cudaStream_t>(stream)), dist, seed, dst,
                              rows, cols, ld, is_f32, first);
  return e == cudaSuccess ? ok() : cuda_fail(e, "fill");
}

// ------------------------------------------------------------------ graphs
int mmws_gpu_graph_dgemm(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                         int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                         int mode, mmws_gpu_graph** out) {
  MMWS_CTX_GUARD(ctx);
  if (!out) return fail(MMWS_GPU_ERR_DOMAIN, "graph_dgemm: null out");
  *out = nullptr;
  auto* g = new (std::nothrow) mmws_gpu_graph();
  if (!g) return fail(MMWS_GPU_ERR_ALLOC, "graph_dgemm: out of host memory");
  g->ctx = ctx;
  // The graph gets its own workspace (a captured pointer into the
  // context's workspace would dangle once an eager call regrows it, and a
  // replay would race eager calls on other streams).
  struct WsRedirect {
    mmws_gpu_ctx* c;
    ~WsRedirect() { c->ws_cur = nullptr, c->ws_cur_bytes = nullptr; }
  } redirect{ctx};
  ctx->ws_cur = &g->ws;
  ctx->ws_cur_bytes = &g->ws_bytes;
  // One eager call first: sets kernel attributes and sizes the graph's
  // workspace, so nothing inside the capture allocates.
  cudaError_t e;
  if (int rc = dgemm_dispatch(ctx, m, n, k, A, lda, B, ldb, C, ldc, mode, ctx->stream)) {
    if (g->ws) cudaFree(g->ws);
    delete g;
    return rc;
  }
  if ((e = cudaStreamSynchronize(ctx->stream)) != cudaSuccess) {
    if (g->ws) cudaFree(g->ws);
    delete g;
    return cuda_fail(e, "graph warmup");
  }
  const uint64_t before = ctx->launches;
  if ((e = cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal)) != cudaSuccess) {
    delete g;
    return cuda_fail(e, "graph capture begin");
  }
  const int rc = dgemm_dispatch(ctx, m, n, k, A, lda, B, ldb, C, ldc, mode, ctx->stream);
  e = cudaStreamEndCapture(ctx->stream, &g->graph);
  g->kernels = ctx->launches - before;
  ctx->launches = before;  // counted on replay
  if (rc || e != cudaSuccess || (e = cudaGraphInstantiate(&g->exec, g->graph, 0)) != cudaSuccess) {
    if (g->graph) cudaGraphDestroy(g->graph);
    if (g->ws) cudaFree(g->ws);
    delete g;
    return rc ? rc : cuda_fail(e, "graph capture / instantiate");
  }
  ctx->graphs.push_back(g);
  *out = g;
  return ok();
}

int mmws_gpu_graph_launch(mmws_gpu_graph* g, void* stream) {
  if (!g) return fail(MMWS_GPU_ERR_STATE, "null graph");
  mmws_gpu_ctx* ctx = g->ctx;
  if (!ctx) return fail(MMWS_GPU_ERR_STATE, "graph_launch: the graph's context was destroyed");
  MMWS_CTX_GUARD(ctx);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  cudaError_t e = cudaGraphLaunch(g->exec, s);
  if (e != cudaSuccess) return cuda_fail(e, "graph launch");
  ctx->launches += g->kernels;
  return ok();
}


int mmws_gpu_graph_destroy(mmws_gpu_graph* g) {
  if (!g) return ok();
  mmws_gpu_ctx* ctx = g->ctx;
  if (!ctx) {  // its context was destroyed first: device resources already gone
    delete g;
    return ok();
  }
  MMWS_CTX_GUARD(ctx);
  graph_release(ctx, g);
  auto& gs = ctx->graphs;
  gs.erase(std::remove(gs.begin(), gs.end(), g), gs.end());
  delete g;
  return ok();
}

// ------------------------------------------------------------------ IPC
int mmws_gpu_synchronize(mmws_gpu_ctx* ctx) {
  MMWS_CTX_GUARD(ctx);
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  return e == cudaSuccess ? ok() : cuda_fail(e, "synchronize");
}

int mmws_gpu_ipc_export(mmws_gpu_ctx* ctx, const void* ptr, uint8_t out[72]) {
  MMWS_CTX_GUARD(ctx);
  return ipc_export(ctx, ptr, out);
}

int mmws_gpu_ipc_open(mmws_gpu_ctx* ctx, const uint8_t in[72], void** ptr) {
  MMWS_CTX_GUARD(ctx);
  return ipc_open(ctx, in, ptr);
}

// ------------------------------------------------------------------ measurement
int mmws_gpu_peak_probe(mmws_gpu_ctx* ctx, int which, int iters, double* tflops) {
  MMWS_CTX_GUARD(ctx);
  if (which < 0 || which > 5 || iters < 1 || !tflops)
    return fail(MMWS_GPU_ERR_DOMAIN, "peak_probe: bad arguments");
  const Launch L = ctx->launch(nullptr);
  double flops = 0;
  cudaError_t e = launch_peak_probe(L, which, iters, ctx->sink, &flops);  // warm-up
  if (e != cudaSuccess) return cuda_fail(e, "peak_probe");
  cudaEventRecord(ctx->ev0, ctx->stream);
  e = launch_peak_probe(L, which, iters, ctx->sink, &flops);
  cudaEventRecord(ctx->ev1, ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "peak_probe");
  if ((e = cudaStreamSynchronize(ctx->stream)) != cudaSuccess) return cuda_fail(e, "peak_probe");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  *tflops = flops / (ms * 1e-3) / 1e12;
  return ok();
}

int mmws_gpu_gemm_probe(mmws_gpu_ctx* ctx, int64_t n, int mode, int iters, double* flops_per_s) {
  MMWS_CTX_GUARD(ctx);
  if (n < 1 || n > 65536 || iters < 1 || !flops_per_s)
    return fail(MMWS_GPU_ERR_DOMAIN, "gemm_probe: bad arguments");
  const size_t bytes = sizeof(double) * n * n;
  void* buf = nullptr;
  cudaError_t e = cudaMalloc(&buf, 3 * bytes);
  if (e != cudaSuccess) return cuda_fail(e, "gemm_probe: buffers");
  double* A = static_cast<double*>(buf);
  double* B = A + n * n;
  double* C = B + n * n;
  const Launch L = ctx->launch(nullptr);
  int rc = MMWS_GPU_OK;
  if ((e = launch_fill(L, MMWS_GPU_DIST_UNIFORM, 0, A, n, n, n, 0, 0)) ||
      (e = launch_fill(L, MMWS_GPU_DIST_UNIFORM, 1, B, n, n, n, 0, 0))) {
    rc = cuda_fail(e, "gemm_probe: fill");
  } else if ((rc = dgemm_dispatch(ctx, n, n, n, A, n, B, n, C, n, mode, ctx->stream)) ==
             MMWS_GPU_OK) {  // warm-up
    cudaEventRecord(ctx->ev0, ctx->stream);
    for (int i = 0; i < iters && rc == MMWS_GPU_OK; ++i)
      rc = dgemm_dispatch(ctx, n, n, n, A, n, B, n, C, n, mode, ctx->stream);
    cudaEventRecord(ctx->ev1, ctx->stream);
    if (rc == MMWS_GPU_OK) {
      if ((e = cudaStreamSynchronize(ctx->stream)) != cudaSuccess) {
        rc = cuda_fail(e, "gemm_probe");
      } else {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        *flops_per_s = 2.0 * static_cast<double>(n) * n * n * iters / (ms * 1e-3);
      }
    }
  }
  cudaStreamSynchronize(ctx->stream);
  if (ctx->server) ctx->deferred_free.push_back(buf);  // cudaFree would wait for the server
  else cudaFree(buf);
  return rc == MMWS_GPU_OK ? ok() : rc;
}

}  // extern "C"

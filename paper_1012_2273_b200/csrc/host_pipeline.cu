// host_pipeline.cu -- host-buffer multiply with the PCIe copies overlapped
// with the GEMM (the matmul_seq / matmul_threads / single-GPU master_run entry
// for host data).
//
// Moving 3 x 8N^2 bytes over PCIe costs about half as long as the N=16384 fp64
// multiply itself, so copying everything in, multiplying, and copying out
// leaves the GPU idle a third of the time.  Instead the work is cut into row
// panels of C (R rows each) on three streams:
//   copy-in : A panel 0, then B in R-wide column blocks (2-D strided copies),
//             then A panels 1.. ;
//   compute : panel 0 as one GEMM per B column block (starts as soon as the
//             first block has landed), then one full-width GEMM per A panel;
//   copy-out: each finished C panel goes back while the next one computes.
// Every launch computes each element with the same kernel arithmetic and
// k-order as one big launch, so the result is bitwise that of the unsplit call.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../../include/mmws_gpu.h"
#include "ctx.h"
#include "kernels.h"

namespace mmws_impl {

namespace {

// Streamed variant (fp64 DMMA, big problems): one persistent GEMM over the
// whole C that starts on tiles whose A rows and B columns have already
// crossed PCIe.  Copy-in interleaves 256-row bands of A and 512-column bands
// of B, each followed by a cuStreamWriteValue32 flag; the kernel walks its
// tiles in arrival order; a per-tile-row completion counter, awaited with
// cuStreamWaitValue32, releases each finished 256-row band of C to the
// copy-out stream.  No launch-size wave quantisation, no panel-0 stall.
// Band sizes: the first tile can start once one A band and one B band have
// landed (48 MB at N=16384, ~1 ms of PCIe), and the last C band to ship after
// the multiply is 32 MB (~0.6 ms); B bands stay 4 KB wide per row so the 2-D
// copies run at full PCIe speed.
int host_multiply_streamed(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                           const double* B, double* C, double* elapsed_s) {
  constexpr int TILE = 128, BAND_A = 2, BAND_B = 4, BAND_C = 2;
  const int64_t tiles_m = (m + TILE - 1) / TILE, tiles_n = (n + TILE - 1) / TILE;
  const int64_t nba = (tiles_m + BAND_A - 1) / BAND_A, nbb = (tiles_n + BAND_B - 1) / BAND_B;
  const int64_t T = tiles_m * tiles_n;
  const size_t flag_ints = nba + nbb + tiles_m;
  cudaError_t e;
  if ((e = ensure(ctx, &ctx->sched, &ctx->sched_bytes, sizeof(int) * (T + flag_ints))) != cudaSuccess)
    return cuda_fail(e, "matmul_host: schedule buffer");
  int* order = static_cast<int*>(ctx->sched);
  int* ready_a = order + T;
  int* ready_b = ready_a + nba;
  int* done = ready_b + nbb;

  // Copy order: whichever operand has crossed fewer bytes goes next, so the
  // landed A rows and B columns grow as a square -- the unlocked tile count
  // (rows x columns) is then largest for the bytes moved.  The first ~15 ms
  // at N=16384 are data-starved whatever the order (tiles need all of K);
  // the square order loses ~4 ms less than a B-first one (simulated and
  // measured).
  std::vector<int64_t> seq_a(nba), seq_b(nbb);
  std::vector<std::pair<char, int64_t>> copies;
  auto push = [&](char w, int64_t i) {
    (w == 'A' ? seq_a : seq_b)[i] = static_cast<int64_t>(copies.size());
    copies.push_back({w, i});
  };
  {
    int64_t ia = 0, ib = 0;
    double bytes_a = 0, bytes_b = 0;
    const double band_a_bytes = static_cast<double>(BAND_A) * TILE * k;
    const double band_b_bytes = static_cast<double>(BAND_B) * TILE * k;
    while (ia < nba || ib < nbb) {
      if (ib >= nbb || (ia < nba && bytes_a <= bytes_b)) {
        push('A', ia++);
        bytes_a += band_a_bytes;
      } else {
        push('B', ib++);
        bytes_b += band_b_bytes;
      }
    }
  }
  if (ctx->sched_m != m || ctx->sched_n != n || ctx->sched_k != k) {
    // Tile order.  CTA c takes positions c, c + grid, ... so position p starts
    // around wave p / grid.  Positions whose wave starts before all inputs can
    // have crossed PCIe take tiles in arrival order (data-starved phase); the
    // rest take row-major order, so C rows complete -- and ship -- one band
    // after another instead of all at the end (arrival order finishes no row
    // before the last B band lands; measured D2H tail 28 ms -> 0.6 ms).
    std::vector<int64_t> key(T);
    std::vector<int> ord(T);
    for (int64_t t = 0; t < T; ++t) {
      const int64_t tm = t / tiles_n, tn = t % tiles_n;
      key[t] = std::max(seq_a[tm / BAND_A], seq_b[tn / BAND_B]) * T + t;
      ord[t] = static_cast<int>(t);
    }
    std::sort(ord.begin(), ord.end(), [&](int x, int y) { return key[x] < key[y]; });
    const double pcie_bytes_per_s = 50e9;  // PCIe 5.0 x16 H2D, conservative
    const double sm_flops_per_s =  // DMMA: 128 flop/clk/SM
        128.0 * (ctx->clock_khz > 0 ? ctx->clock_khz : 1900000) * 1e3;
    const double t_inputs = 8.0 * (static_cast<double>(m) * k + static_cast<double>(k) * n) /
                            pcie_bytes_per_s;
    const double t_tile = 2.0 * TILE * TILE * k / sm_flops_per_s;
    const int64_t grid = std::min<int64_t>(T, ctx->num_sms);
    const int64_t p_all =
        std::min<int64_t>(T, static_cast<int64_t>(t_inputs / t_tile) * grid);
    std::sort(ord.begin() + p_all, ord.end());
    if ((e = cudaMemcpy(order, ord.data(), sizeof(int) * T, cudaMemcpyHostToDevice)))
      return cuda_fail(e, "matmul_host: tile order");
    ctx->sched_m = m;
    ctx->sched_n = n;
    ctx->sched_k = k;
  }

  cudaStream_t in = ctx->copy_in, comp = ctx->stream, out = ctx->copy_out;
  if ((e = event_pool(ctx, 1)) != cudaSuccess) return cuda_fail(e, "matmul_host: events");
  cudaEvent_t ev_reset = ctx->pool[0];
  double* dA = static_cast<double*>(ctx->dA);
  double* dB = static_cast<double*>(ctx->dB);
  double* dC = static_cast<double*>(ctx->dC);
  auto dptr = [](const void* p) { return static_cast<CUdeviceptr>(reinterpret_cast<uintptr_t>(p)); };

  cudaEventRecord(ctx->ev0, comp);
  if ((e = cudaMemsetAsync(ready_a, 0, sizeof(int) * flag_ints, comp)))
    return cuda_fail(e, "matmul_host: reset flags");
  cudaEventRecord(ev_reset, comp);
  cudaStreamWaitEvent(in, ev_reset, 0);
  cudaStreamWaitEvent(out, ev_reset, 0);
  // optional timeline (MMWS_GPU_PIPELINE_TRACE=1): H2D end, kernel start/end
  cudaEvent_t tr[3] = {nullptr, nullptr, nullptr};
  const bool trace = ctx->tune.pipeline_trace;
  if (trace) {
    for (auto& ev : tr) cudaEventCreate(&ev);
    cudaEventRecord(tr[1], comp);
  }
  // ---- one persistent multiply, launched first: it waits on the arrival
  // flags, so the copy-in below may take as long as it needs (pageable host
  // buffers are pumped through pinned chunks by the CPU, staging.cu)
  DmmaStream st;
  st.order = order;
  st.count = static_cast<int>(T);
  st.ready_a = ready_a;
  st.ready_b = ready_b;
  st.band_a = BAND_A;
  st.band_b = BAND_B;
  st.done = done;
  const int grid = static_cast<int>(std::min<int64_t>(T, ctx->num_sms));
  ctx->last_plan = "dgemm_dmma_kernel<128x128, 8 math warps, streamed from host>";
  if ((e = launch_dgemm_dmma_stream(ctx->launch(comp), m, n, k, dA, k, dB, n, dC, n, st, grid)))
    return cuda_fail(e, "matmul_host: streamed dgemm");
  if (trace) cudaEventRecord(tr[2], comp);
  // The persistent kernel spins on the arrival flags: if anything below
  // fails, every flag is raised (on a stream the failed copy did not touch)
  // and the kernel drained before returning, so no later call queues behind
  // a kernel that never ends.  Its C is garbage; the call fails.
  auto abandon = [&](int rc) {
    cudaMemsetAsync(ready_a, 0x01, sizeof(int) * (nba + nbb), out);
    cudaStreamSynchronize(out);
    cudaStreamSynchronize(comp);
    return rc;
  };
  // ---- copy-in, each band followed by its arrival flag
  for (const auto& [which, i] : copies) {
    if (which == 'A') {
      const int64_t r0 = i * BAND_A * TILE, rows = std::min<int64_t>(BAND_A * TILE, m - r0);
      if ((e = copy_h2d(ctx, dA + r0 * k, sizeof(double) * k, A + r0 * k, sizeof(double) * k,
                        sizeof(double) * k, rows, in)))
        return abandon(cuda_fail(e, "matmul_host: H2D A"));
      if (ctx->write_value(in, dptr(ready_a + i), 1, 0) != CUDA_SUCCESS)
        return abandon(fail(MMWS_GPU_ERR_CUDA, "matmul_host: cuStreamWriteValue32 failed"));
    } else {
      const int64_t c0 = i * BAND_B * TILE, w = std::min<int64_t>(BAND_B * TILE, n - c0);
      if ((e = copy_h2d(ctx, dB + c0, sizeof(double) * n, B + c0, sizeof(double) * n,
                        sizeof(double) * w, k, in)))
        return abandon(cuda_fail(e, "matmul_host: H2D B"));
      if (ctx->write_value(in, dptr(ready_b + i), 1, 0) != CUDA_SUCCESS)
        return abandon(fail(MMWS_GPU_ERR_CUDA, "matmul_host: cuStreamWriteValue32 failed"));
    }
  }
  if (trace) cudaEventRecord(tr[0], in);
  // ---- copy-out: each 256-row band once all its tiles are counted
  D2hPump pump(ctx, out);
  for (int64_t t0 = 0; t0 < tiles_m; t0 += BAND_C) {
    const int64_t t1 = std::min<int64_t>(tiles_m, t0 + BAND_C);
    for (int64_t tm = t0; tm < t1; ++tm)
      if (ctx->wait_value(out, dptr(done + tm), static_cast<cuuint32_t>(tiles_n),
                          CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
        return fail(MMWS_GPU_ERR_CUDA, "matmul_host: cuStreamWaitValue32 failed");
    const int64_t r0 = t0 * TILE, rows = std::min<int64_t>(m, t1 * TILE) - r0;
    if ((e = pump.add(C + r0 * n, sizeof(double) * n, dC + r0 * n, sizeof(double) * n,
                      sizeof(double) * n, rows)))
      return cuda_fail(e, "matmul_host: D2H");
  }
  if ((e = pump.finish())) return cuda_fail(e, "matmul_host: D2H");
  cudaEventRecord(ctx->ev1, out);
  if ((e = cudaStreamSynchronize(out)) != cudaSuccess ||
      (e = cudaStreamSynchronize(comp)) != cudaSuccess ||
      (e = cudaStreamSynchronize(in)) != cudaSuccess)
    return cuda_fail(e, "matmul_host: sync");
  if (elapsed_s) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    *elapsed_s = ms * 1e-3;
  }
  if (trace) {
    float t[4] = {0.f, 0.f, 0.f, 0.f};
    for (int i = 0; i < 3; ++i) cudaEventElapsedTime(&t[i], ctx->ev0, tr[i]);
    cudaEventElapsedTime(&t[3], ctx->ev0, ctx->ev1);
    std::fprintf(stderr,
                 "[mmws_gpu pipeline] h2d_end_ms=%.3f kernel_start_ms=%.3f kernel_end_ms=%.3f "
                 "d2h_end_ms=%.3f\n", t[0], t[1], t[2], t[3]);
    for (auto& ev : tr) cudaEventDestroy(ev);
  }
  return ok();
}

// MODE_OZAKI with host buffers: B crosses PCIe first and is scaled and cut
// into residues once; A then follows in row panels, each emulated against the
// prepared B while the next panel is in flight, and each C panel goes back as
// soon as its reconstruction is done.  Nothing can start before all of B has
// landed (every output needs a whole column of B), so the floor is B's copy +
// the emulation + one panel's copy-out rather than copy-in + emulation +
// copy-out.  Bitwise the one-shot MODE_OZAKI result (each output row depends
// only on its own row of A).
template <class T>
int host_multiply_ozaki(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const T* A,
                        const T* B, T* C, double* elapsed_s) {
  if (k > 131072)
    return fail(MMWS_GPU_ERR_DIMENSION, "matmul ozaki: k must be <= 131072 (int32 accumulation)");
  const int64_t R = std::max<int64_t>(512, ((m + 7) / 8 + 255) / 256 * 256);
  const int64_t panels = (m + R - 1) / R;
  const size_t ws = sizeof(T) == 8 ? ozaki_workspace_bytes(R, n, k) : ozaki_workspace_bytes_f32(R, n, k);
  cudaError_t e;
  void* wsp = nullptr;
  if ((e = workspace(ctx, ws, &wsp, ctx->stream)) != cudaSuccess)
    return cuda_fail(e, "matmul ozaki: workspace");
  if ((e = event_pool(ctx, panels * 2 + 1)) != cudaSuccess)
    return cuda_fail(e, "matmul ozaki: events");
  cudaEvent_t* evA = ctx->pool.data();
  cudaEvent_t* evC = evA + panels;
  cudaEvent_t evB = evC[panels];
  T* dA = static_cast<T*>(ctx->dA);
  T* dB = static_cast<T*>(ctx->dB);
  T* dC = static_cast<T*>(ctx->dC);
  cudaStream_t in = ctx->copy_in, comp = ctx->stream, out = ctx->copy_out;
  const Launch L = ctx->launch(comp);
  auto rows_of = [&](int64_t i) { return std::min(R, m - i * R); };

  cudaEventRecord(ctx->ev0, in);
  if ((e = copy_h2d(ctx, dB, sizeof(T) * n, B, sizeof(T) * n, sizeof(T) * n, k, in)))
    return cuda_fail(e, "matmul ozaki: H2D B");
  cudaEventRecord(evB, in);
  cudaStreamWaitEvent(comp, evB, 0);
  ctx->last_plan = "ozaki (int8 tcgen05 GEMMs + CRT), B prepared once, A in row panels";
  if ((e = launch_ozaki_prepare_b(L, n, k, dB, n, wsp)) != cudaSuccess)
    return cuda_fail(e, "matmul ozaki: prepare B");
  for (int64_t i = 0; i < panels; ++i) {
    if ((e = copy_h2d(ctx, dA + i * R * k, sizeof(T) * k, A + i * R * k, sizeof(T) * k,
                      sizeof(T) * k, rows_of(i), in)))
      return cuda_fail(e, "matmul ozaki: H2D A");
    cudaEventRecord(evA[i], in);
    cudaStreamWaitEvent(comp, evA[i], 0);
    if ((e = launch_ozaki_panel(L, rows_of(i), n, k, dA + i * R * k, k, dC + i * R * n, n,
                                wsp)) != cudaSuccess)
      return cuda_fail(e, "matmul ozaki: panel");
    cudaEventRecord(evC[i], comp);
  }
  D2hPump pump(ctx, out);
  for (int64_t i = 0; i < panels; ++i) {
    cudaStreamWaitEvent(out, evC[i], 0);
    if ((e = pump.add(C + i * R * n, sizeof(T) * n, dC + i * R * n, sizeof(T) * n, sizeof(T) * n,
                      rows_of(i))))
      return cuda_fail(e, "matmul ozaki: D2H");
  }
  if ((e = pump.finish())) return cuda_fail(e, "matmul ozaki: D2H");
  cudaEventRecord(ctx->ev1, out);
  if ((e = cudaStreamSynchronize(out)) != cudaSuccess ||
      (e = cudaStreamSynchronize(comp)) != cudaSuccess ||
      (e = cudaStreamSynchronize(in)) != cudaSuccess)
    return cuda_fail(e, "matmul ozaki: sync");
  if (elapsed_s) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    *elapsed_s = ms * 1e-3;
  }
  return ok();
}

// Tiny problems (the paper's N = 10 .. ~70): A, B and C fit one small pinned,
// device-mapped bounce buffer.  A and B are packed into it with host memcpy.
// When the multiply takes the latency kernel (plain loads: n, k <= 96 in
// AUTO / EXACT) it reads A and B and writes C through the mapping -- no copy
// engine at all; otherwise A|B cross PCIe in ONE transfer and C in one D2H,
// on the same stream as the multiply, with one synchronisation (no
// driver-staged pageable copies, no cross-stream events: each costs
// microseconds at this size).  Same kernel, same bits as the other paths.
constexpr size_t TINY_BYTES = size_t(128) << 10;

template <class T>
int host_multiply_tiny(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const T* A,
                       const T* B, T* C, int mode, double* elapsed_s) {
  const size_t a_b = sizeof(T) * m * k, b_b = sizeof(T) * k * n, c_b = sizeof(T) * m * n;
  const size_t b_off = (a_b + 255) / 256 * 256;
  cudaError_t e;
  if (!ctx->tiny_host &&
      (e = cudaHostAlloc(&ctx->tiny_host, 2 * TINY_BYTES + 512, cudaHostAllocMapped)) != cudaSuccess) {
    ctx->tiny_host = nullptr;
    return cuda_fail(e, "matmul_host: pinned bounce buffer");
  }
  char* hin = static_cast<char*>(ctx->tiny_host);
  char* hout = hin + TINY_BYTES + 256;
  std::memcpy(hin, A, a_b);
  std::memcpy(hin + b_off, B, b_b);
  cudaStream_t s = ctx->stream;
  const bool zero_copy = sizeof(T) == 8 && n <= AUTO_SMALL_MAX && k <= AUTO_SMALL_MAX &&
                         (mode == MMWS_GPU_MODE_AUTO || mode == MMWS_GPU_MODE_EXACT);
  if (zero_copy) {  // the latency kernel reads and writes host memory (UVA mapping)
    cudaEventRecord(ctx->ev0, s);
    if (int rc = gemm<T>(ctx, m, n, k, reinterpret_cast<const T*>(hin), k,
                         reinterpret_cast<const T*>(hin + b_off), n, reinterpret_cast<T*>(hout),
                         n, mode, s))
      return rc;
  } else {
    if ((e = ensure(ctx, &ctx->dA, &ctx->dA_bytes, b_off + b_b)) != cudaSuccess ||
        (e = ensure(ctx, &ctx->dC, &ctx->dC_bytes, c_b)) != cudaSuccess)
      return cuda_fail(e, "matmul_host: device buffers");
    char* dAB = static_cast<char*>(ctx->dA);
    cudaEventRecord(ctx->ev0, s);
    if ((e = cudaMemcpyAsync(dAB, hin, b_off + b_b, cudaMemcpyHostToDevice, s)) != cudaSuccess)
      return cuda_fail(e, "matmul_host: H2D");
    if (int rc = gemm<T>(ctx, m, n, k, reinterpret_cast<const T*>(dAB), k,
                         reinterpret_cast<const T*>(dAB + b_off), n, static_cast<T*>(ctx->dC), n,
                         mode, s))
      return rc;
    if ((e = cudaMemcpyAsync(hout, ctx->dC, c_b, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
      return cuda_fail(e, "matmul_host: D2H");
  }
  cudaEventRecord(ctx->ev1, s);
  if ((e = cudaEventSynchronize(ctx->ev1)) != cudaSuccess) return cuda_fail(e, "matmul_host: sync");
  std::memcpy(C, hout, c_b);
  if (elapsed_s) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    *elapsed_s = ms * 1e-3;
  }
  return ok();
}

}  // namespace

template <class T>
int host_multiply(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const T* A, const T* B,
                  T* C, int mode, double* elapsed_s) {
  if (m <= 0 || n <= 0 || k <= 0)
    return fail(MMWS_GPU_ERR_DIMENSION, "matmul: dimensions must be positive");
  if (!A || !B || !C) return fail(MMWS_GPU_ERR_DOMAIN, "matmul: null host pointer");
  const size_t a_b = sizeof(T) * m * k, b_b = sizeof(T) * k * n, c_b = sizeof(T) * m * n;
  if (a_b + 256 + b_b <= TINY_BYTES && c_b <= TINY_BYTES)
    return host_multiply_tiny(ctx, m, n, k, A, B, C, mode, elapsed_s);
  cudaError_t e;
  if ((e = ensure(ctx, &ctx->dA, &ctx->dA_bytes, a_b)) != cudaSuccess ||
      (e = ensure(ctx, &ctx->dB, &ctx->dB_bytes, b_b)) != cudaSuccess ||
      (e = ensure(ctx, &ctx->dC, &ctx->dC_bytes, c_b)) != cudaSuccess)
    return cuda_fail(e, "matmul_host: device buffers");
  if constexpr (sizeof(T) == 8) {
    // big fp64 tensor-path problems whose dense device copies TMA can read
    const int64_t tiles128 = ((m + 127) / 128) * ((n + 127) / 128);
    if ((mode == MMWS_GPU_MODE_AUTO || mode == MMWS_GPU_MODE_DMMA) && ctx->write_value &&
        ctx->wait_value && tiles128 >= 2 * static_cast<int64_t>(ctx->num_sms) && k % 2 == 0 &&
        n % 2 == 0 && (n > AUTO_SMALL_MAX || k > AUTO_SMALL_MAX))
      return host_multiply_streamed(ctx, m, n, k, A, B, C, elapsed_s);
  }
  // big emulated problems: B prepared once, A streamed in row panels
  if (mode == MMWS_GPU_MODE_OZAKI && m >= 1024 && static_cast<double>(m) * n * k >= 1.0e10)
    return host_multiply_ozaki(ctx, m, n, k, A, B, C, elapsed_s);
  T* dA = static_cast<T*>(ctx->dA);
  T* dB = static_cast<T*>(ctx->dB);
  T* dC = static_cast<T*>(ctx->dC);
  cudaStream_t in = ctx->copy_in, comp = ctx->stream, out = ctx->copy_out;

  // Row panels (multiples of 128 rows) once the problem is big enough for the
  // overlap to matter (m*n*k >= 1e8); one panel otherwise.  Pinned buffers:
  // 1/8 of the rows, 1/16 from m*n*k = 1e13 (host-buffer multiply, min of 25 interleaved calls: N=750
  // 260.5 vs 292.4 us in one panel, 1000 415.2 vs 514.7, 1250 648.5 vs
  // 818.8).  Pageable buffers: every panel's copy is pumped through the
  // pinned staging ring by the host copy pool in chunks of its own, so fewer,
  // bigger panels -- 4 below 1.5e9, 2 below 4.5e9, 3 below 1.5e10, 8 above
  // (min of 20 interleaved calls, tools/host_panels_probe.py, 1 / 2 / 3 / 4 /
  // 8 panels: N=500 236 / 208 / 207 / 194 / 187 us, 1000 836 / 727 / 719 /
  // 726 / 715, 1500 2177 / 1356 / 1576 / 1613 / 1622, 1750 2692 / 2281 /
  // 2087 / 2239 / 2271, 2100 4892 / 3078 / 2668 / 2847 / 3196; the steps
  // follow how the panels' copies fall into staging chunks).
  // MMWS_GPU_HOST_PANELS overrides the count; the bits never change.
  const double work = static_cast<double>(m) * n * k;
  const bool pinned = !is_pageable(A) && !is_pageable(C);
  int want = work < 1.0e8 ? 1 : work < 1.0e13 ? 8 : 16;  // fp32 N=32768: 1085 vs 1106 ms (tools/f32_host_panels_probe.py)
  if (!pinned && want > 1) want = work < 1.5e9 ? 4 : work < 4.5e9 ? 2 : work < 1.5e10 ? 3 : 8;
  if (ctx->tune.host_panels > 0 && work >= 1.0e7) want = ctx->tune.host_panels;
  // small MODE_OZAKI problems would recompute B's residues per launch: one panel
  const int64_t R = (want <= 1 || mode == MMWS_GPU_MODE_OZAKI)
                        ? m
                        : std::max<int64_t>(128, ((m + want - 1) / want + 127) / 128 * 128);
  const int64_t panels = (m + R - 1) / R;
  // column blocks never narrower than 512 unless n itself is: a block then
  // takes the same kernel as the whole problem (see dgemm_dispatch).  A
  // remainder narrower than W is folded into the last block (width in
  // [W, 2W)), so no block can drop onto the latency kernel.
  const int64_t W = panels > 1 ? std::min<int64_t>(n, std::max<int64_t>(R, 512)) : n;
  const int64_t blocks = std::max<int64_t>(1, n / W);
  auto width_of = [&](int64_t j) { return j + 1 < blocks ? W : n - j * W; };
  if ((e = event_pool(ctx, panels * 2 + blocks)) != cudaSuccess)
    return cuda_fail(e, "matmul_host: events");
  cudaEvent_t* evA = ctx->pool.data();
  cudaEvent_t* evC = evA + panels;
  cudaEvent_t* evB = evC + panels;

  cudaEventRecord(ctx->ev0, in);
  // Copy-in and compute are queued in lockstep -- a multiply right after the
  // copy it needs -- so a pageable copy that the CPU pumps through pinned
  // chunks (staging.cu) already overlaps the multiplies queued before it.
  auto rows_of = [&](int64_t i) { return std::min(R, m - i * R); };
  // panel 0 of A, then B block by block, each block's panel-0 multiply next
  if ((e = copy_h2d(ctx, dA, sizeof(T) * k, A, sizeof(T) * k, sizeof(T) * k, rows_of(0), in)))
    return cuda_fail(e, "matmul_host: H2D A");
  cudaEventRecord(evA[0], in);
  cudaStreamWaitEvent(comp, evA[0], 0);
  for (int64_t j = 0; j < blocks; ++j) {
    const int64_t w = width_of(j);
    if ((e = copy_h2d(ctx, dB + j * W, sizeof(T) * n, B + j * W, sizeof(T) * n, sizeof(T) * w, k,
                      in)))
      return cuda_fail(e, "matmul_host: H2D B");
    cudaEventRecord(evB[j], in);
    cudaStreamWaitEvent(comp, evB[j], 0);
    if (int rc = gemm<T>(ctx, rows_of(0), w, k, dA, k, dB + j * W, n, dC + j * W, n, mode, comp))
      return rc;
  }
  cudaEventRecord(evC[0], comp);
  // the other A panels, each followed by its full-width multiply
  for (int64_t i = 1; i < panels; ++i) {
    if ((e = copy_h2d(ctx, dA + i * R * k, sizeof(T) * k, A + i * R * k, sizeof(T) * k,
                      sizeof(T) * k, rows_of(i), in)))
      return cuda_fail(e, "matmul_host: H2D A");
    cudaEventRecord(evA[i], in);
    cudaStreamWaitEvent(comp, evA[i], 0);
    if (int rc = gemm<T>(ctx, rows_of(i), n, k, dA + i * R * k, k, dB, n, dC + i * R * n, n, mode,
                         comp))
      return rc;
    cudaEventRecord(evC[i], comp);
  }
  // ---- copy-out, panel by panel as the multiplies finish
  D2hPump pump(ctx, out);
  for (int64_t i = 0; i < panels; ++i) {
    cudaStreamWaitEvent(out, evC[i], 0);
    if ((e = pump.add(C + i * R * n, sizeof(T) * n, dC + i * R * n, sizeof(T) * n, sizeof(T) * n,
                      rows_of(i))))
      return cuda_fail(e, "matmul_host: D2H");
  }
  if ((e = pump.finish())) return cuda_fail(e, "matmul_host: D2H");
  cudaEventRecord(ctx->ev1, out);
  if ((e = cudaStreamSynchronize(out)) != cudaSuccess ||
      (e = cudaStreamSynchronize(comp)) != cudaSuccess ||
      (e = cudaStreamSynchronize(in)) != cudaSuccess)
    return cuda_fail(e, "matmul_host: sync");
  if (elapsed_s) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    *elapsed_s = ms * 1e-3;
  }
  return ok();
}

template int host_multiply<double>(mmws_gpu_ctx*, int64_t, int64_t, int64_t, const double*,
                                   const double*, double*, int, double*);
template int host_multiply<float>(mmws_gpu_ctx*, int64_t, int64_t, int64_t, const float*,
                                  const float*, float*, int, double*);

}  // namespace mmws_impl

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
#include <vector>

#include "../../include/mmws_gpu.h"
#include "ctx.h"

namespace mmws_impl {

namespace {

cudaError_t event_pool(mmws_gpu_ctx* ctx, size_t need) {
  while (ctx->pool.size() < need) {
    cudaEvent_t ev;
    cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    ctx->pool.push_back(ev);
  }
  return cudaSuccess;
}

template <class T>
int gemm(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const T* A, int64_t lda, const T* B,
         int64_t ldb, T* C, int64_t ldc, int mode, cudaStream_t s) {
  if constexpr (sizeof(T) == 8)
    return dgemm_dispatch(ctx, m, n, k, A, lda, B, ldb, C, ldc, mode, s);
  else
    return sgemm_dispatch(ctx, m, n, k, A, lda, B, ldb, C, ldc, mode, s);
}

}  // namespace

template <class T>
int host_multiply(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const T* A, const T* B,
                  T* C, int mode, double* elapsed_s) {
  if (m <= 0 || n <= 0 || k <= 0)
    return fail(MMWS_GPU_ERR_DIMENSION, "matmul: dimensions must be positive");
  if (!A || !B || !C) return fail(MMWS_GPU_ERR_DOMAIN, "matmul: null host pointer");
  const size_t a_b = sizeof(T) * m * k, b_b = sizeof(T) * k * n, c_b = sizeof(T) * m * n;
  cudaError_t e;
  if ((e = ensure(&ctx->dA, &ctx->dA_bytes, a_b)) != cudaSuccess ||
      (e = ensure(&ctx->dB, &ctx->dB_bytes, b_b)) != cudaSuccess ||
      (e = ensure(&ctx->dC, &ctx->dC_bytes, c_b)) != cudaSuccess)
    return cuda_fail(e, "matmul_host: device buffers");
  T* dA = static_cast<T*>(ctx->dA);
  T* dB = static_cast<T*>(ctx->dB);
  T* dC = static_cast<T*>(ctx->dC);
  cudaStream_t in = ctx->copy_in, comp = ctx->stream, out = ctx->copy_out;

  // Panels of 1/8 of the rows (multiples of 128) once the problem is big
  // enough for the overlap to matter; one panel otherwise.
  const double work = static_cast<double>(m) * n * k;
  const int64_t R = work < 2.0e9 ? m : std::max<int64_t>(128, ((m + 7) / 8 + 127) / 128 * 128);
  const int64_t panels = (m + R - 1) / R;
  // column blocks never narrower than 512 unless n itself is: a block then
  // takes the same kernel as the whole problem (see dgemm_dispatch)
  const int64_t W = panels > 1 ? std::min<int64_t>(n, std::max<int64_t>(R, 512)) : n;
  const int64_t blocks = (n + W - 1) / W;
  if ((e = event_pool(ctx, panels * 2 + blocks)) != cudaSuccess)
    return cuda_fail(e, "matmul_host: events");
  cudaEvent_t* evA = ctx->pool.data();
  cudaEvent_t* evC = evA + panels;
  cudaEvent_t* evB = evC + panels;

  cudaEventRecord(ctx->ev0, in);
  // ---- copy-in
  auto rows_of = [&](int64_t i) { return std::min(R, m - i * R); };
  if ((e = cudaMemcpyAsync(dA, A, sizeof(T) * rows_of(0) * k, cudaMemcpyHostToDevice, in)))
    return cuda_fail(e, "matmul_host: H2D A");
  cudaEventRecord(evA[0], in);
  for (int64_t j = 0; j < blocks; ++j) {
    const int64_t w = std::min(W, n - j * W);
    if ((e = cudaMemcpy2DAsync(dB + j * W, sizeof(T) * n, B + j * W, sizeof(T) * n, sizeof(T) * w,
                               k, cudaMemcpyHostToDevice, in)))
      return cuda_fail(e, "matmul_host: H2D B");
    cudaEventRecord(evB[j], in);
  }
  for (int64_t i = 1; i < panels; ++i) {
    if ((e = cudaMemcpyAsync(dA + i * R * k, A + i * R * k, sizeof(T) * rows_of(i) * k,
                             cudaMemcpyHostToDevice, in)))
      return cuda_fail(e, "matmul_host: H2D A");
    cudaEventRecord(evA[i], in);
  }
  // ---- compute
  cudaStreamWaitEvent(comp, evA[0], 0);
  for (int64_t j = 0; j < blocks; ++j) {
    cudaStreamWaitEvent(comp, evB[j], 0);
    const int64_t w = std::min(W, n - j * W);
    if (int rc = gemm<T>(ctx, rows_of(0), w, k, dA, k, dB + j * W, n, dC + j * W, n, mode, comp))
      return rc;
  }
  cudaEventRecord(evC[0], comp);
  for (int64_t i = 1; i < panels; ++i) {
    cudaStreamWaitEvent(comp, evA[i], 0);
    if (int rc = gemm<T>(ctx, rows_of(i), n, k, dA + i * R * k, k, dB, n, dC + i * R * n, n, mode,
                         comp))
      return rc;
    cudaEventRecord(evC[i], comp);
  }
  // ---- copy-out
  for (int64_t i = 0; i < panels; ++i) {
    cudaStreamWaitEvent(out, evC[i], 0);
    if ((e = cudaMemcpyAsync(C + i * R * n, dC + i * R * n, sizeof(T) * rows_of(i) * n,
                             cudaMemcpyDeviceToHost, out)))
      return cuda_fail(e, "matmul_host: D2H");
  }
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

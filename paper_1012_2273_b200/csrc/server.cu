// server.cu -- persistent latency server for tiny fp64 multiplies (N <= 96).
//
// For the smallest sizes of the paper's sweep the multiply is ~1 us of work and
// everything else is overhead: launching a kernel (or replaying a graph), two
// PCIe copies, and synchronising cost 25-50 us of wall time per call.  Here a
// small resident grid waits for requests in pinned, mapped host memory:
//   host:   memcpy A, B into the pinned staging area, publish the request with
//           one 64-bit store (sequence number + shape + mode);
//   device: CTA 0 polls that word (and forwards it); each CTA pulls a slice of A|B over PCIe
//           (wide cache-volatile loads, all issued before any is consumed --
//           one SM alone cannot keep enough PCIe reads in flight) into an HBM
//           scratch copy; grid barrier; each CTA computes a block of C rows --
//           with exactly the arithmetic of dgemm_small_kernel (EXACT:
//           acc = RN(acc + RN(a*b)), otherwise one DFMA per step, k ascending
//           from +0.0) -- stores them straight into the staging area, fences;
//           the last CTA to finish publishes "done";
//   host:   spins on "done", copies C out.
// Only CTA 0 polls the host; it forwards grid-wide requests to the others
// through device memory.  Requests of at most SOLO_PAIRS double pairs are
// served by CTA 0 alone (one load wave, no barrier).  No launch, no stream synchronisation, no copy
// engine on the critical path.  The grid (MMWS_GPU_SERVER_CTAS, default 8)
// occupies that many SMs until mmws_gpu_server_stop.
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/mmws_gpu.h"
#include "ctx.h"

namespace mmws_impl {
namespace {

constexpr int SRV_MAX = 96;        // largest m, n, k served
constexpr int SRV_THREADS = 256;
constexpr int SRV_UNROLL = 8;      // 16-byte loads in flight per thread
constexpr int SOLO_PAIRS = 3072;  // measured break-even: N = 50 solo 21.5 us vs grid 26 us; N = 64 30.4 vs 26.9
constexpr int SRV_DEFAULT_CTAS = 8;  // N = 96: 1 CTA 70 us, 4: 44, 8: 36, 16: 36
constexpr long long SRV_STOP = -1;

// One 64-bit control word, written by the host with a single store so the
// device never sees a sequence number without its descriptor:
//   bits 0..31 sequence number (-1 = stop), 32..39 m, 40..47 n, 48..55 k,
//   56 exact.
struct Mailbox {                   // pinned, mapped host memory
  volatile long long ctl;
  volatile int done;               // device writes the served sequence number
  int pad[13];
  double ab[2 * SRV_MAX * SRV_MAX];  // A (m x k) then B (k x n), both dense
  double c[SRV_MAX * SRV_MAX];
};

struct GridSync {                  // device memory, zeroed at start
  volatile long long ctl;          // CTA 0's copy of a multi-CTA request (or stop)
  unsigned int arrive;             // CTAs that finished pulling, monotonic
  unsigned int finish;             // CTAs that finished storing C, monotonic
};

// Served by the whole grid (or a stop, which every CTA must see)?
__device__ __forceinline__ bool is_multi(long long v, int G) {
  if (static_cast<int>(v & 0xffffffffll) == static_cast<int>(SRV_STOP)) return true;
  const int m = static_cast<int>((v >> 32) & 0xff), n = static_cast<int>((v >> 40) & 0xff);
  const int k = static_cast<int>((v >> 48) & 0xff);
  return G > 1 && (m * k + k * n + 1) / 2 > SOLO_PAIRS;
}

constexpr int SRV_SMEM = 2 * SRV_MAX * SRV_MAX * sizeof(double);

__device__ __forceinline__ double2 ld_cv2(const double2* p) {
  double2 v;
  asm volatile("ld.global.cv.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

// Copy pairs [lo, hi) of src to dst, SRV_UNROLL loads in flight per thread.
template <bool kFromHost>
__device__ __forceinline__ void pull(double2* dst, const double2* src, int lo, int hi) {
  for (int base = lo; base < hi; base += SRV_THREADS * SRV_UNROLL) {
    double2 r[SRV_UNROLL];
#pragma unroll
    for (int u = 0; u < SRV_UNROLL; ++u) {
      const int i = base + u * SRV_THREADS + threadIdx.x;
      if (i < hi) r[u] = kFromHost ? ld_cv2(src + i) : __ldcg(src + i);
    }
#pragma unroll
    for (int u = 0; u < SRV_UNROLL; ++u) {
      const int i = base + u * SRV_THREADS + threadIdx.x;
      if (i < hi) dst[i - lo] = r[u];
    }
  }
}

// C rows [r0, r1) from A rows (As, row stride k, first row r0) and B (k x n);
// two independent output elements per step (latency of the dependent chain).
__device__ __forceinline__ void multiply_rows(const double* As, const double* Bs, double* C,
                                              int r0, int r1, int n, int k, bool exact) {
  const int cnt = (r1 - r0) * n;
  for (int e0 = threadIdx.x; e0 < cnt; e0 += 2 * SRV_THREADS) {
    const int e1 = e0 + SRV_THREADS;
    const bool two = e1 < cnt;
    const int i0 = e0 / n, c0 = e0 % n;
    const int i1 = two ? e1 / n : i0, c1 = two ? e1 % n : c0;
    double acc0 = 0.0, acc1 = 0.0;
    if (exact) {
      for (int j = 0; j < k; ++j) {
        acc0 = __dadd_rn(acc0, __dmul_rn(As[i0 * k + j], Bs[j * n + c0]));
        acc1 = __dadd_rn(acc1, __dmul_rn(As[i1 * k + j], Bs[j * n + c1]));
      }
    } else {
      for (int j = 0; j < k; ++j) {
        acc0 = fma(As[i0 * k + j], Bs[j * n + c0], acc0);
        acc1 = fma(As[i1 * k + j], Bs[j * n + c1], acc1);
      }
    }
    C[r0 * n + e0] = acc0;
    if (two) C[r0 * n + e1] = acc1;
  }
}

__global__ void __launch_bounds__(SRV_THREADS, 1)
    server_kernel(Mailbox* box, double* scratch, GridSync* sync) {
  extern __shared__ double2 srv_smem2[];
  double* S = reinterpret_cast<double*>(srv_smem2);
  __shared__ long long s_ctl;
  const int G = gridDim.x;
  int last = box->done;            // CTA 0: last request seen; others: last broadcast seen
  unsigned int epoch = 0;          // multi-CTA requests served so far
  for (;;) {
    if (threadIdx.x == 0) {
      long long v;
      if (blockIdx.x == 0) {
        // only CTA 0 polls host memory: every extra PCIe poller of the
        // control line delays the host's store to it by microseconds
        for (;;) {
          v = box->ctl;
          if (static_cast<int>(v & 0xffffffffll) != last) break;
          __nanosleep(32);
        }
        if (is_multi(v, G)) {      // hand the request to the other CTAs through L2
          __threadfence_system();
          sync->ctl = v;
          __threadfence();
        }
      } else {
        for (;;) {
          v = sync->ctl;
          if (static_cast<int>(v & 0xffffffffll) != last) break;
          __nanosleep(20);
        }
        __threadfence_system();
      }
      s_ctl = v;
    }
    __syncthreads();
    const long long v = s_ctl;
    __syncthreads();               // s_ctl is rewritten by the next poll
    const int seq = static_cast<int>(v & 0xffffffffll);
    if (seq == static_cast<int>(SRV_STOP)) return;
    last = seq;
    const int m = static_cast<int>((v >> 32) & 0xff), n = static_cast<int>((v >> 40) & 0xff);
    const int k = static_cast<int>((v >> 48) & 0xff);
    const bool exact = (v >> 56) & 1;
    // A|B as one dense run of m*k + k*n doubles, read as pairs (host pads).
    const int pairs = (m * k + k * n + 1) / 2;
    const double2* src = reinterpret_cast<const double2*>(box->ab);

    if (!is_multi(v, G)) {         // only CTA 0 gets here
      pull<true>(srv_smem2, src, 0, pairs);
      __syncthreads();
      multiply_rows(S, S + m * k, box->c, 0, m, n, k, exact);
      __threadfence_system();
      __syncthreads();
      if (threadIdx.x == 0) {
        box->done = seq;
        __threadfence_system();
      }
      continue;
    }

    ++epoch;
    // 1. this CTA's slice of A|B: PCIe -> registers -> HBM scratch
    const int per = (pairs + G - 1) / G;
    const int lo = min(pairs, blockIdx.x * per), hi = min(pairs, lo + per);
    pull<true>(reinterpret_cast<double2*>(scratch) + lo, src, lo, hi);
    __syncthreads();
    // 2. grid barrier (monotonic counter: target epoch * G)
    if (threadIdx.x == 0) {
      __threadfence();
      atomicAdd(&sync->arrive, 1u);
      const unsigned int target = epoch * static_cast<unsigned int>(G);
      while (static_cast<int>(*reinterpret_cast<volatile unsigned int*>(&sync->arrive) - target) < 0)
        __nanosleep(20);
      __threadfence();
    }
    __syncthreads();
    // 3. this CTA's C rows: its A rows and all of B from L2 into shared memory
    const int rows = (m + G - 1) / G;
    const int r0 = min(m, blockIdx.x * rows), r1 = min(m, r0 + rows);
    if (r1 > r0) {
      // A rows [r0, r1) start at double r0*k; copy whole pairs covering them
      const int a_lo = (r0 * k) / 2, a_hi = (r1 * k + 1) / 2;
      pull<false>(srv_smem2, reinterpret_cast<const double2*>(scratch), a_lo, a_hi);
      const double* As = S + (r0 * k - 2 * a_lo);
      // B starts at double m*k; stage it after the A pairs, pair-aligned
      const int b_lo = (m * k) / 2, b_hi = pairs;
      double2* Bdst = srv_smem2 + (a_hi - a_lo);
      pull<false>(Bdst, reinterpret_cast<const double2*>(scratch), b_lo, b_hi);
      const double* Bs = reinterpret_cast<const double*>(Bdst) + (m * k - 2 * b_lo);
      __syncthreads();
      multiply_rows(As, Bs, box->c, r0, r1, n, k, exact);
    }
    // 4. completion: the last CTA to finish publishes "done"
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned int prev = atomicAdd(&sync->finish, 1u);
      if (prev == epoch * static_cast<unsigned int>(G) - 1) {
        __threadfence_system();
        box->done = seq;
        __threadfence_system();
      }
    }
  }
}

}  // namespace

struct ServerState {
  Mailbox* host = nullptr;  // cudaHostAlloc'd, mapped
  Mailbox* dev = nullptr;   // device alias of host
  double* scratch = nullptr;  // device copy of A|B for the multi-CTA path
  GridSync* sync = nullptr;
  cudaStream_t stream = nullptr;
  int seq = 0;
  int ctas = 0;
};

static void server_free(ServerState* s) {
  if (s->stream) cudaStreamDestroy(s->stream);
  if (s->scratch) cudaFree(s->scratch);
  if (s->sync) cudaFree(s->sync);
  if (s->host) cudaFreeHost(s->host);
  delete s;
}

void server_destroy(mmws_gpu_ctx* ctx) {
  ServerState* s = static_cast<ServerState*>(ctx->server);
  if (!s) return;
  if (s->host) {
    s->host->ctl = static_cast<long long>(static_cast<unsigned int>(SRV_STOP));
    std::atomic_thread_fence(std::memory_order_seq_cst);
  }
  if (s->stream) cudaStreamSynchronize(s->stream);
  server_free(s);
  ctx->server = nullptr;
  for (void* p : ctx->deferred_free) cudaFree(p);
  ctx->deferred_free.clear();
}

}  // namespace mmws_impl

using namespace mmws_impl;

extern "C" {

int mmws_gpu_server_start(mmws_gpu_ctx* ctx) {
  MMWS_CTX_GUARD(ctx);
  if (ctx->server) return ok();
  auto* s = new ServerState();
  s->ctas = SRV_DEFAULT_CTAS;
  if (ctx->tune.server_ctas != 0) s->ctas = ctx->tune.server_ctas;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
  if (s->ctas < 1 || s->ctas > sms) {
    delete s;
    return fail(MMWS_GPU_ERR_DOMAIN, "server_start: MMWS_GPU_SERVER_CTAS must be in [1, SMs]");
  }
  cudaError_t e;
  if ((e = cudaHostAlloc(reinterpret_cast<void**>(&s->host), sizeof(Mailbox),
                         cudaHostAllocMapped)) != cudaSuccess) {
    delete s;
    return cuda_fail(e, "server_start: pinned mailbox");
  }
  std::memset(static_cast<void*>(s->host), 0, sizeof(Mailbox));
  if ((e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&s->dev), s->host, 0)) ||
      (e = cudaMalloc(&s->scratch, sizeof(double) * 2 * SRV_MAX * SRV_MAX)) ||
      (e = cudaMalloc(&s->sync, sizeof(GridSync))) ||
      (e = cudaMemset(s->sync, 0, sizeof(GridSync))) ||
      (e = cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking)) ||
      (e = cudaFuncSetAttribute(server_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                SRV_SMEM))) {
    server_free(s);
    return cuda_fail(e, "server_start");
  }
  // (every other kernel of the library was loaded by mmws_gpu_init)
  // cooperative launch: all CTAs must be co-resident for the grid barrier
  void* args[] = {&s->dev, &s->scratch, &s->sync};
  if ((e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(server_kernel), dim3(s->ctas),
                                       dim3(SRV_THREADS), args, SRV_SMEM, s->stream))) {
    server_free(s);
    return cuda_fail(e, "server_start: launch");
  }
  ctx->launches += 1;
  ctx->server = s;
  return ok();
}

}  // extern "C"

namespace mmws_impl {

bool server_serves(const mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, int mode) {
  return ctx->server && m >= 1 && n >= 1 && k >= 1 && m <= SRV_MAX && n <= SRV_MAX &&
         k <= SRV_MAX && (mode == MMWS_GPU_MODE_AUTO || mode == MMWS_GPU_MODE_EXACT);
}

// Caller holds ctx->mu.
int server_multiply(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                    int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc, int mode,
                    double* elapsed_s) {
  ServerState* s = static_cast<ServerState*>(ctx->server);
  if (!s) return fail(MMWS_GPU_ERR_STATE, "server_dgemm: server not started");
  if (m <= 0 || n <= 0 || k <= 0)
    return fail(MMWS_GPU_ERR_DIMENSION, "server_dgemm: dimensions must be positive");
  if (m > SRV_MAX || n > SRV_MAX || k > SRV_MAX)
    return fail(MMWS_GPU_ERR_DIMENSION, "server_dgemm: the server takes m, n, k <= 96");
  if (lda < k || ldb < n || ldc < n)
    return fail(MMWS_GPU_ERR_DIMENSION, "server_dgemm: leading dimension smaller than row");
  if (!A || !B || !C) return fail(MMWS_GPU_ERR_DOMAIN, "server_dgemm: null host pointer");
  if (mode != MMWS_GPU_MODE_AUTO && mode != MMWS_GPU_MODE_EXACT)
    return fail(MMWS_GPU_ERR_DOMAIN, "server_dgemm: mode must be AUTO or EXACT");
  const auto t0 = std::chrono::steady_clock::now();
  Mailbox* box = s->host;
  double* a = box->ab;
  double* b = box->ab + m * k;
  if (lda == k) std::memcpy(a, A, sizeof(double) * m * k);
  else for (int64_t i = 0; i < m; ++i) std::memcpy(a + i * k, A + i * lda, sizeof(double) * k);
  if (ldb == n) std::memcpy(b, B, sizeof(double) * k * n);
  else for (int64_t j = 0; j < k; ++j) std::memcpy(b + j * n, B + j * ldb, sizeof(double) * n);
  const int want = s->seq = s->seq % 0x3fffffff + 1;   // 1..2^30-1: never -1 (stop) or 0
  const long long ctl = static_cast<long long>(static_cast<unsigned int>(want)) | (m << 32) |
                        (n << 40) | (k << 48) |
                        (static_cast<long long>(mode == MMWS_GPU_MODE_EXACT) << 56);
  std::atomic_thread_fence(std::memory_order_seq_cst);
  box->ctl = ctl;
  std::atomic_thread_fence(std::memory_order_seq_cst);
  const auto deadline = t0 + std::chrono::seconds(10);
  while (box->done != want) {
    if (std::chrono::steady_clock::now() > deadline) {
      const cudaError_t e = cudaStreamQuery(s->stream);
      return fail(MMWS_GPU_ERR_CUDA, std::string("server_dgemm: no answer within 10 s (") +
                                         cudaGetErrorString(e) + ")");
    }
  }
  std::atomic_thread_fence(std::memory_order_seq_cst);
  for (int64_t i = 0; i < m; ++i) std::memcpy(C + i * ldc, box->c + i * n, sizeof(double) * n);
  if (elapsed_s)
    *elapsed_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return ok();
}

}  // namespace mmws_impl

extern "C" {

int mmws_gpu_server_dgemm(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                          int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                          int mode, double* elapsed_s) {
  if (!ctx) return fail(MMWS_GPU_ERR_STATE, "null mmws_gpu_ctx");
  std::lock_guard<std::mutex> guard(ctx->mu);
  return server_multiply(ctx, m, n, k, A, lda, B, ldb, C, ldc, mode, elapsed_s);
}

int mmws_gpu_server_stop(mmws_gpu_ctx* ctx) {
  if (!ctx) return fail(MMWS_GPU_ERR_STATE, "null mmws_gpu_ctx");
  std::lock_guard<std::mutex> guard(ctx->mu);
  cudaSetDevice(ctx->device);
  server_destroy(ctx);
  return ok();
}

}  // extern "C"

// ctx.h -- the context object behind mmws_gpu_ctx (internal).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <mutex>
#include <string>
#include <vector>

#include "kernels.h"

namespace mmws_impl {
// MMWS_GPU_* tuning / test knobs, read once from the environment by
// mmws_gpu_init (never on a per-call path).
struct Tuning {
  bool no_streamk = false;      // MMWS_GPU_NO_STREAMK: never use stream-K launches
  std::string dmma_plan;        // MMWS_GPU_DMMA_PLAN: "<cfg>" or "<cfg>s<CTAs/SM>" override
  int raster_group = 0;         // MMWS_GPU_RASTER_GROUP: DMMA tile raster group (0 = built-in)
  bool pipeline_trace = false;  // MMWS_GPU_PIPELINE_TRACE: host-pipeline timeline on stderr
  int rowblock_ranks = 0;       // MMWS_GPU_ROWBLOCK_RANKS: 0 cost model, -1 "all", 1 rank 0 alone
  int server_ctas = 0;          // MMWS_GPU_SERVER_CTAS (0 = default)
  int copy_threads = 0;         // MMWS_GPU_COPY_THREADS (0 = 3/4 of the host cores, <= 12)
  int host_panels = 0;          // MMWS_GPU_HOST_PANELS: row panels of a host-buffer multiply (0 = built-in)
  double timeout_s = 30.0;      // MMWS_GPU_TIMEOUT_S: deadline of one distributed step
  bool nccl_gather = false;     // MMWS_GPU_NCCL_GATHER: C-slices as NCCL messages, no fused IPC
  int sgemm_at = -1;            // MMWS_GPU_SGEMM_AT: fp32 A staged k-major; -1 by size, 0 never, 1 always
  static Tuning from_env();
  // Set one knob by its environment name (value NULL: back to the default);
  // false for an unknown name.
  bool set(const char* name, const char* value);
};
}  // namespace mmws_impl

struct mmws_gpu_graph;

struct mmws_gpu_ctx {
  int device = 0;
  int num_sms = 0;
  int cc_major = 0, cc_minor = 0, clock_khz = 0;
  cudaStream_t stream = nullptr;                       // compute
  cudaStream_t copy_in = nullptr, copy_out = nullptr;  // host-entry PCIe copies
  std::vector<cudaEvent_t> pool;                       // host-pipeline ordering events
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  cudaEvent_t evk0 = nullptr, evk1 = nullptr;  // around the row-block multiply
  double last_kernel_ms = 0.0;
  const char* last_plan = "";  // kernel configuration of the latest multiply (static string)
  mmws_impl::EncodeTiledFn encode = nullptr;
  // stream memory operations (cuStreamWriteValue32 / cuStreamWaitValue32) for
  // the streamed host path; null if the driver does not offer them
  CUresult (*write_value)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  CUresult (*wait_value)(CUstream, CUdeviceptr, cuuint32_t, unsigned int) = nullptr;
  void* server = nullptr;  // latency server state (server.cu), null when not running
  void* stager = nullptr;  // pinned chunk ring + host copy threads (staging.cu), lazy
  void* tiny_host = nullptr;  // pinned bounce buffer of tiny host-buffer multiplies, lazy
  uint64_t stage_next = 0;  // next pinned chunk (round robin)
  std::vector<void*> deferred_free;  // buffers outgrown while the server ran
  // CUDA IPC (fused C gather of the row-block path)
  CUresult (*mem_range)(CUdeviceptr*, size_t*, CUdeviceptr) = nullptr;
  struct IpcMap {
    unsigned char handle[64];
    void* base;
    int scope;           // IPC_CALLER / IPC_ROUND / IPC_COMM (ipc_open)
    uint64_t last_use;
  };
  std::vector<IpcMap> ipc_cache;
  uint64_t ipc_clock = 0;
  // live graphs: mmws_gpu_destroy releases their device resources and
  // detaches them, so a graph destroyed (or launched) after its context is
  // an error, not a use after free
  std::vector<mmws_gpu_graph*> graphs;
  void* ipc_stage = nullptr;  // 256-byte device staging for the handle broadcast / barrier
  unsigned char* host_stage = nullptr;  // 512 bytes of pinned host memory: its host end
  unsigned char last_handle[80] = {0};  // row-block: handle bytes of the last call
  int last_fused = -1;                  // row-block: agreed fused-gather decision for it
  // streamed host path: [tile order | ready_a | ready_b | done] on the device
  void* sched = nullptr;
  size_t sched_bytes = 0;
  int64_t sched_m = -1, sched_n = -1, sched_k = -1;  // shape the uploaded tile order belongs to
  uint64_t launches = 0;
  std::mutex mu;
  mmws_impl::Tuning tune;

  // packing / MODE_OZAKI workspaces (device), one per launch stream, grown on
  // demand: stream order keeps each one safe, and a call on one stream never
  // overwrites the workspace a call still running on another stream reads.
  // While a CUDA graph is built, ws_cur points at that graph's own workspace
  // instead, so a replay never shares (or outlives) the eager calls' buffers.
  struct WsSpace {
    cudaStream_t stream;
    void* mem;
    size_t bytes;
    uint64_t last_use;
  };
  std::vector<WsSpace> ws_spaces;
  uint64_t space_clock = 0;  // LRU clock of the per-stream workspaces
  void** ws_cur = nullptr;
  size_t* ws_cur_bytes = nullptr;
  // stream-K workspaces, one per launch stream (fixed size, never moved):
  // (num_sms + 1) accumulator slots of 128 x 128 doubles + their flags
  struct SkSpace {
    cudaStream_t stream;
    void* mem;
    uint64_t last_use;
  };
  std::vector<SkSpace> sk_spaces;
  bool allow_streamk = true;  // false while a row-block round overlaps NCCL with multiplies
  // MODE_OZAKI: second stream for its tensor-core GEMMs + ordering events (lazy)
  cudaStream_t oz_stream = nullptr;
  cudaEvent_t oz_ev[8] = {};
  // host-entry staging buffers (device)
  void* dA = nullptr;
  void* dB = nullptr;
  void* dC = nullptr;
  size_t dA_bytes = 0, dB_bytes = 0, dC_bytes = 0;
  // probe sink
  double* sink = nullptr;

  // row-block distribution
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  cudaStream_t comm_stream = nullptr;
  void* rbA = nullptr;  // worker-side A slice / B copy / C slice
  void* rbB = nullptr;
  void* rbC = nullptr;
  void* rbAcc = nullptr;  // worker: running accumulators of its first sub-block (B in panels)
  size_t rbA_bytes = 0, rbB_bytes = 0, rbC_bytes = 0, rbAcc_bytes = 0;
  // failure detection (rowblock.cu): every rank stores its progress through
  // each round into rank 0's board, one word per rank (round * 8 + stage)
  unsigned* board = nullptr;       // rank 0: the board (device memory, IPC-exported)
  unsigned* board_peer = nullptr;  // where this rank's stores go / rank 0's board as seen here
  uint32_t round = 0;              // rounds started on this communicator
  double round_work_s = 0.0;       // deadline allowance for the current step's own work
  bool comm_failed = false;        // a round timed out / a peer failed: communicator aborted
  int last_gather = 0;             // last round: 0 one GPU, 1 fused IPC stores, 2 NCCL C-slices
  int last_active = 1;             // last round: ranks that multiplied
  int last_panels = 1;             // last round: B broadcast in this many k-panels

  mmws_impl::Launch launch(cudaStream_t s) {
    mmws_impl::Launch L;
    L.stream = s ? s : stream;
    L.num_sms = num_sms;
    L.encode = encode;
    L.launches = &launches;
    L.raster_group = tune.raster_group;
    return L;
  }
};

namespace mmws_impl {
// error plumbing shared by the C-ABI translation units
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);
int ok();
// Grow a device buffer to at least `bytes`.  While the latency server runs,
// cudaFree (a device-wide synchronisation) would wait for it forever, so the
// old buffer is parked in deferred_free instead (growth at least doubles).
cudaError_t ensure(mmws_gpu_ctx* ctx, void** buf, size_t* have, size_t bytes);
// At most MAX_STREAM_SPACES per-stream workspaces of each kind are kept: a
// caller cycling through many streams would otherwise keep one per stream
// alive.  Over the cap the least recently used one is freed after a device
// synchronisation (not while the latency server holds the device -- its
// kernel never ends -- then the list just grows).
constexpr size_t MAX_STREAM_SPACES = 16;
template <class V>
void trim_stream_spaces(mmws_gpu_ctx* ctx, V& spaces) {
  while (spaces.size() >= MAX_STREAM_SPACES && !ctx->server) {
    auto lru = spaces.begin();
    for (auto it = spaces.begin(); it != spaces.end(); ++it)
      if (it->last_use < lru->last_use) lru = it;
    cudaDeviceSynchronize();
    if (lru->mem) cudaFree(lru->mem);
    spaces.erase(lru);
  }
}

// The multiply workspace for work queued on `stream` (NULL: the context
// stream) -- that stream's own, or the graph's being built -- at least
// `bytes` long.
inline cudaError_t workspace(mmws_gpu_ctx* ctx, size_t bytes, void** out, cudaStream_t stream) {
  void** buf = ctx->ws_cur;
  size_t* have = ctx->ws_cur_bytes;
  if (!buf) {
    const cudaStream_t s = stream ? stream : ctx->stream;
    mmws_gpu_ctx::WsSpace* sp = nullptr;
    for (auto& w : ctx->ws_spaces)
      if (w.stream == s) sp = &w;
    if (!sp) {
      trim_stream_spaces(ctx, ctx->ws_spaces);
      ctx->ws_spaces.push_back({s, nullptr, 0, 0});
      sp = &ctx->ws_spaces.back();
    }
    sp->last_use = ++ctx->space_clock;
    buf = &sp->mem;
    have = &sp->bytes;
  }
  const cudaError_t e = ensure(ctx, buf, have, bytes);
  *out = *buf;
  return e;
}
// the fp64 multiply dispatch used by dgemm / host / graph / row-block paths
// cin (optional): accumulate, C = Cin + A.B continuing Cin's chains (no
// stream-K; not in MODE_OZAKI).
int dgemm_dispatch(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                   int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc, int mode,
                   cudaStream_t stream, const double* cin = nullptr, int64_t ldcin = 0);
// Host -> device copy of `rows` rows of `width` bytes (row pitches in bytes),
// queued on s.  Pageable host memory goes through pinned chunks filled by
// host threads (staging.cu); pinned memory is copied directly.  Returns once
// everything is queued (the host buffer is no longer needed).
cudaError_t copy_h2d(mmws_gpu_ctx* ctx, void* dst, size_t dpitch, const void* src, size_t spitch,
                     size_t width, size_t rows, cudaStream_t s);
// Device -> host copies queued on one stream, pageable destinations through
// the pinned chunk ring with up to 3 chunks in flight across add() calls
// (a chunk is copied out while the next ones transfer).  Pinned destinations
// are plain cudaMemcpy2DAsync.  finish() (or the destructor) returns once
// every staged destination is filled.
class D2hPump {
 public:
  D2hPump(mmws_gpu_ctx* ctx, cudaStream_t s);
  ~D2hPump();
  cudaError_t add(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                  size_t rows);
  cudaError_t finish();

 private:
  struct Pending {
    char* dst;
    size_t dpitch, width, rows;
    int slot;
  };
  cudaError_t drain_one();
  mmws_gpu_ctx* ctx_;
  cudaStream_t s_;
  std::vector<Pending> pending_;
};
bool is_pageable(const void* p);
void staging_destroy(mmws_gpu_ctx* ctx);
// Stop the latency server (if running) and free its resources.
void server_destroy(mmws_gpu_ctx* ctx);
// Would the running latency server take this host-buffer multiply?
bool server_serves(const mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, int mode);
// Serve it (caller holds ctx->mu).
int server_multiply(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                    int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc, int mode,
                    double* elapsed_s);
// CUDA IPC: 64-byte handle of the allocation holding ptr + 8-byte offset.
int ipc_export(mmws_gpu_ctx* ctx, const void* ptr, uint8_t out[72]);
// Mapping scopes: IPC_CALLER -- mmws_gpu_ipc_open's, open until the context
// goes away; IPC_ROUND -- rank 0's C as a row-block round maps it: at most
// IPC_ROUND_MAPPINGS stay open, least recently used closed first (a caller
// that gives every round a fresh C allocation would otherwise keep every old
// one mapped, and its memory alive on rank 0; rounds are synchronous, so no
// work uses an evicted mapping); IPC_COMM -- the progress board.  Round and
// communicator mappings are closed by mmws_gpu_comm_destroy.
enum { IPC_CALLER = 0, IPC_ROUND = 1, IPC_COMM = 2 };
int ipc_open(mmws_gpu_ctx* ctx, const uint8_t in[72], void** ptr, int scope = IPC_CALLER);
void ipc_close_scoped(mmws_gpu_ctx* ctx);
constexpr int IPC_ROUND_MAPPINGS = 4;
// Host-buffer multiply with PCIe copies overlapped (host_pipeline.cu).
template <class T>
int host_multiply(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const T* A, const T* B,
                  T* C, int mode, double* elapsed_s);
int sgemm_dispatch(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const float* A,
                   int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int mode,
                   cudaStream_t stream, const float* cin = nullptr, int64_t ldcin = 0);

// fp64 / fp32 multiply through the matching dispatch
template <class T>
int gemm(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const T* A, int64_t lda, const T* B,
         int64_t ldb, T* C, int64_t ldc, int mode, cudaStream_t s, const T* cin = nullptr,
         int64_t ldcin = 0) {
  if constexpr (sizeof(T) == 8)
    return dgemm_dispatch(ctx, m, n, k, A, lda, B, ldb, C, ldc, mode, s, cin, ldcin);
  else
    return sgemm_dispatch(ctx, m, n, k, A, lda, B, ldb, C, ldc, mode, s, cin, ldcin);
}

// at least `need` ordering events (timing disabled) in ctx->pool
inline cudaError_t event_pool(mmws_gpu_ctx* ctx, size_t need) {
  while (ctx->pool.size() < need) {
    cudaEvent_t ev;
    cudaError_t e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
    ctx->pool.push_back(ev);
  }
  return cudaSuccess;
}
}  // namespace mmws_impl

// Entry guard of every C-ABI function taking a context: null check, the
// context's mutex for the rest of the call, its device made current.
#define MMWS_CTX_GUARD(ctx)                                                  \
  if (!(ctx)) return mmws_impl::fail(MMWS_GPU_ERR_STATE, "null mmws_gpu_ctx"); \
  std::lock_guard<std::mutex> guard_((ctx)->mu);                             \
  if (cudaError_t e_ = cudaSetDevice((ctx)->device); e_ != cudaSuccess)      \
    return mmws_impl::cuda_fail(e_, "cudaSetDevice");

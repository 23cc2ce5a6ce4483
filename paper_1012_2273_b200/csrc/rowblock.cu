// rowblock.cu -- master/worker row-block distribution over NCCL (one rank per
// GPU), the device-side re-expression of master_run / worker_run
// (reference include/mmws/protocol.hpp:50-147).
//
// Reference protocol (TCP): the master sends every worker offset, rows,
// A-slice and all of B on tag 1 (protocol.hpp:68-73), then receives offset,
// rows and C-slice on tag 2 in rank order (protocol.hpp:85-103); workers with
// rows == 0 still handshake (protocol.hpp:122-123); elapsed = first send ->
// last receive (protocol.hpp:63,105).
//
// Here: every rank derives (offset, rows) from split_rows itself (no
// metadata messages), the A-slices go out as one grouped ncclSend/ncclRecv
// batch, B is one ncclBroadcast (NVLink/NVSwitch, not P-1 re-sends), each rank
// multiplies its slice with the same kernel configuration as a 1-GPU call --
// per-element arithmetic does not depend on the row offset or the slice
// height, so P-GPU results are bitwise the 1-GPU results -- and the C-slices
// come back as one grouped receive batch into C's row blocks on rank 0.  Rank
// 0 is master AND worker 0 (its GPU would otherwise idle).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <string>
#include <vector>

#include "../../include/mmws_gpu.h"
#include "ctx.h"
#include "nccl_dl.h"

using namespace mmws_impl;

namespace {

int nccl_fail(ncclResult_t r, const char* what) {
  return fail(MMWS_GPU_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
}

#define NCCL_REQUIRE()                                                          \
  if (!nccl().ok) return fail(MMWS_GPU_ERR_NCCL, "libnccl.so.2 could not be loaded");



#define NCCL_TRY(call, what)                                   \
  do {                                                         \
    ncclResult_t r_ = (call);                                  \
    if (r_ != ncclSuccess) return nccl_fail(r_, what);         \
  } while (0)

template <class T>
T* as_mut(const T* p) {
  return const_cast<T*>(p);
}

// Enqueue one master/worker round on ctx->stream (no synchronisation).  Rank
// 0 passes device A, B, C; other ranks pass nulls and use library buffers.
template <class T>
int rowblock_enqueue(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const T* A, const T* B,
                     T* C, int mode) {
  if (m <= 0 || n <= 0 || k <= 0)
    return fail(MMWS_GPU_ERR_DIMENSION, "rowblock: dimensions must be positive");
  const int P = ctx->comm ? ctx->nranks : 1;
  const int me = ctx->comm ? ctx->rank : 0;
  if (me == 0 && (!A || !B || !C))
    return fail(MMWS_GPU_ERR_DOMAIN, "rowblock: rank 0 needs A, B and C");
  if (P > 1) NCCL_REQUIRE();
  std::vector<int64_t> off(P), rows(P);
  if (int rc = mmws_gpu_split_rows(m, P, off.data(), rows.data())) return rc;

  const ncclDataType_t dt = sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
  cudaStream_t s = ctx->stream;
  cudaError_t e;

  const T* a_loc = A;
  const T* b_loc = B;
  T* c_loc = C;
  if (me != 0) {
    if ((e = ensure(&ctx->rbA, &ctx->rbA_bytes, sizeof(T) * (rows[me] * k + 1))) != cudaSuccess ||
        (e = ensure(&ctx->rbB, &ctx->rbB_bytes, sizeof(T) * k * n)) != cudaSuccess ||
        (e = ensure(&ctx->rbC, &ctx->rbC_bytes, sizeof(T) * (rows[me] * n + 1))) != cudaSuccess)
      return cuda_fail(e, "rowblock: worker buffers");
    a_loc = static_cast<const T*>(ctx->rbA);
    b_loc = static_cast<const T*>(ctx->rbB);
    c_loc = static_cast<T*>(ctx->rbC);
  }

  if (P > 1) {
    // tag 1: A-slices (protocol.hpp:70-72) ...
    NCCL_TRY(nccl().GroupStart(), "ncclGroupStart");
    if (me == 0) {
      for (int r = 1; r < P; ++r)
        if (rows[r] > 0)
          NCCL_TRY(nccl().Send(A + off[r] * k, rows[r] * k, dt, r, ctx->comm, s), "send A-slice");
    } else if (rows[me] > 0) {
      NCCL_TRY(nccl().Recv(as_mut(a_loc), rows[me] * k, dt, 0, ctx->comm, s), "recv A-slice");
    }
    NCCL_TRY(nccl().GroupEnd(), "ncclGroupEnd");
    // ... and all of B (protocol.hpp:73), once, as a broadcast.
    void* bbuf = me == 0 ? as_mut(B) : as_mut(b_loc);
    NCCL_TRY(nccl().Broadcast(bbuf, bbuf, k * n, dt, 0, ctx->comm, s), "broadcast B");
  }

  // worker body (protocol.hpp:132-141) on this rank's rows, timed on its stream
  cudaEventRecord(ctx->evk0, s);
  if (rows[me] > 0) {
    int rc;
    if constexpr (sizeof(T) == 8)
      rc = dgemm_dispatch(ctx, rows[me], n, k, a_loc, k, b_loc, n, c_loc, n, mode, s);
    else
      rc = sgemm_dispatch(ctx, rows[me], n, k, a_loc, k, b_loc, n, c_loc, n, mode, s);
    if (rc) return rc;
  }
  cudaEventRecord(ctx->evk1, s);

  if (P > 1) {
    // tag 2: C-slices back into C's row blocks, rank order (protocol.hpp:85-103)
    NCCL_TRY(nccl().GroupStart(), "ncclGroupStart");
    if (me == 0) {
      for (int r = 1; r < P; ++r)
        if (rows[r] > 0)
          NCCL_TRY(nccl().Recv(C + off[r] * n, rows[r] * n, dt, r, ctx->comm, s), "recv C-slice");
    } else if (rows[me] > 0) {
      NCCL_TRY(nccl().Send(c_loc, rows[me] * n, dt, 0, ctx->comm, s), "send C-slice");
    }
    NCCL_TRY(nccl().GroupEnd(), "ncclGroupEnd");
  }
  return MMWS_GPU_OK;
}

int finish(mmws_gpu_ctx* ctx, bool timed, double* elapsed_s) {
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess) return cuda_fail(e, "rowblock: sync");
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, ctx->evk0, ctx->evk1) == cudaSuccess) ctx->last_kernel_ms = ms;
  if (timed && elapsed_s) {
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    *elapsed_s = ms * 1e-3;
  }
  return ok();
}

template <class T>
int rowblock(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const T* A, const T* B, T* C,
             int mode, double* elapsed_s) {
  const bool root = !ctx->comm || ctx->rank == 0;
  if (root) cudaEventRecord(ctx->ev0, ctx->stream);  // first send
  if (int rc = rowblock_enqueue(ctx, m, n, k, A, B, C, mode)) return rc;
  if (root) cudaEventRecord(ctx->ev1, ctx->stream);  // last receive
  return finish(ctx, root, elapsed_s);
}

// master_run with host matrices on rank 0: H2D of A and B, the round, D2H of
// C, all inside the elapsed bracket (the reference's master holds host data).
template <class T>
int master_run_host(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const T* A, const T* B,
                    T* C, int mode, double* elapsed_s) {
  const bool root = !ctx->comm || ctx->rank == 0;
  if (!root) return rowblock(ctx, m, n, k, static_cast<const T*>(nullptr),
                             static_cast<const T*>(nullptr), static_cast<T*>(nullptr), mode,
                             elapsed_s);
  if (!ctx->comm || ctx->nranks == 1)  // one GPU: copies overlapped with the multiply
    return host_multiply(ctx, m, n, k, A, B, C, mode, elapsed_s);
  if (m <= 0 || n <= 0 || k <= 0)
    return fail(MMWS_GPU_ERR_DIMENSION, "master_run: dimensions must be positive");
  if (!A || !B || !C) return fail(MMWS_GPU_ERR_DOMAIN, "master_run: null host matrix");
  const size_t a_b = sizeof(T) * m * k, b_b = sizeof(T) * k * n, c_b = sizeof(T) * m * n;
  cudaError_t e;
  if ((e = ensure(&ctx->dA, &ctx->dA_bytes, a_b)) != cudaSuccess ||
      (e = ensure(&ctx->dB, &ctx->dB_bytes, b_b)) != cudaSuccess ||
      (e = ensure(&ctx->dC, &ctx->dC_bytes, c_b)) != cudaSuccess)
    return cuda_fail(e, "master_run: device buffers");
  cudaStream_t s = ctx->stream;
  cudaEventRecord(ctx->ev0, s);
  if ((e = cudaMemcpyAsync(ctx->dA, A, a_b, cudaMemcpyHostToDevice, s)) != cudaSuccess ||
      (e = cudaMemcpyAsync(ctx->dB, B, b_b, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "master_run: H2D");
  if (int rc = rowblock_enqueue(ctx, m, n, k, static_cast<const T*>(ctx->dA),
                                static_cast<const T*>(ctx->dB), static_cast<T*>(ctx->dC), mode))
    return rc;
  if ((e = cudaMemcpyAsync(C, ctx->dC, c_b, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return cuda_fail(e, "master_run: D2H");
  cudaEventRecord(ctx->ev1, s);
  return finish(ctx, true, elapsed_s);
}

}  // namespace

#define MMWS_CTX_GUARD(ctx)                                              \
  if (!(ctx)) return fail(MMWS_GPU_ERR_STATE, "null mmws_gpu_ctx");      \
  std::lock_guard<std::mutex> guard_((ctx)->mu);                         \
  if (cudaError_t e_ = cudaSetDevice((ctx)->device); e_ != cudaSuccess)  \
    return cuda_fail(e_, "cudaSetDevice");

extern "C" {

int mmws_gpu_nccl_unique_id(uint8_t out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  if (!out) return fail(MMWS_GPU_ERR_DOMAIN, "nccl_unique_id: null out");
  NCCL_REQUIRE();
  ncclUniqueId id;
  NCCL_TRY(nccl().GetUniqueId(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
  return ok();
}

int mmws_gpu_comm_init(mmws_gpu_ctx* ctx, int nranks, int rank, const uint8_t id[128]) {
  MMWS_CTX_GUARD(ctx);
  if (nranks < 1) return fail(MMWS_GPU_ERR_DOMAIN, "comm_init: nranks must be >= 1");
  if (rank < 0 || rank >= nranks)
    return fail(MMWS_GPU_ERR_RANK, "comm_init: rank " + std::to_string(rank) +
                                       " outside world of " + std::to_string(nranks));
  if (!id) return fail(MMWS_GPU_ERR_DOMAIN, "comm_init: null unique id");
  if (ctx->comm) return fail(MMWS_GPU_ERR_STATE, "comm_init: communicator already initialised");
  NCCL_REQUIRE();
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, 128);
  NCCL_TRY(nccl().CommInitRank(&ctx->comm, nranks, uid, rank), "ncclCommInitRank");
  ctx->nranks = nranks;
  ctx->rank = rank;
  return ok();
}

int mmws_gpu_comm_destroy(mmws_gpu_ctx* ctx) {
  MMWS_CTX_GUARD(ctx);
  if (ctx->comm) {
    NCCL_TRY(nccl().CommDestroy(ctx->comm), "ncclCommDestroy");
    ctx->comm = nullptr;
  }
  ctx->nranks = 1;
  ctx->rank = 0;
  return ok();
}

int mmws_gpu_rowblock_dgemm(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k,
                            const double* A, const double* B, double* C, int mode,
                            double* elapsed_s) {
  MMWS_CTX_GUARD(ctx);
  return rowblock<double>(ctx, m, n, k, A, B, C, mode, elapsed_s);
}

int mmws_gpu_rowblock_sgemm(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const float* A,
                            const float* B, float* C, int mode, double* elapsed_s) {
  MMWS_CTX_GUARD(ctx);
  return rowblock<float>(ctx, m, n, k, A, B, C, mode, elapsed_s);
}

int mmws_gpu_master_run_host(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k,
                             const double* A, const double* B, double* C, int mode,
                             double* elapsed_s) {
  MMWS_CTX_GUARD(ctx);
  return master_run_host<double>(ctx, m, n, k, A, B, C, mode, elapsed_s);
}

int mmws_gpu_master_run_host_f32(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k,
                                 const float* A, const float* B, float* C, int mode,
                                 double* elapsed_s) {
  MMWS_CTX_GUARD(ctx);
  return master_run_host<float>(ctx, m, n, k, A, B, C, mode, elapsed_s);
}

int mmws_gpu_last_kernel_ms(mmws_gpu_ctx* ctx, double* ms) {
  if (!ctx || !ms) return fail(MMWS_GPU_ERR_DOMAIN, "last_kernel_ms: null argument");
  *ms = ctx->last_kernel_ms;
  return ok();
}

int mmws_gpu_rowblock_plan(int64_t m, int64_t n, int64_t k, int nranks, int32_t* peer,
                           int32_t* tag, int32_t* kind, int64_t* count, int32_t* dir,
                           int32_t* n_entries) {
  if (!n_entries) return fail(MMWS_GPU_ERR_DOMAIN, "rowblock_plan: null n_entries");
  if (m <= 0 || n <= 0 || k <= 0)
    return fail(MMWS_GPU_ERR_DIMENSION, "rowblock_plan: dimensions must be positive");
  if (nranks < 1) return fail(MMWS_GPU_ERR_DOMAIN, "rowblock_plan: nranks must be >= 1");
  std::vector<int64_t> off(nranks), rows(nranks);
  mmws_gpu_split_rows(m, nranks, off.data(), rows.data());
  struct E { int32_t peer, tag, kind; int64_t count; int32_t dir; };
  std::vector<E> plan;
  if (nranks > 1) {
    for (int r = 1; r < nranks; ++r)
      if (rows[r] > 0) plan.push_back({r, 1, 1, rows[r] * k, 0});
    plan.push_back({-1, 1, 1, k * n, 2});
    for (int r = 1; r < nranks; ++r)
      if (rows[r] > 0) plan.push_back({r, 2, 1, rows[r] * n, 1});
  }
  const int32_t cap = *n_entries;
  *n_entries = static_cast<int32_t>(plan.size());
  if (cap < *n_entries) return ok();
  for (size_t i = 0; i < plan.size(); ++i) {
    if (peer) peer[i] = plan[i].peer;
    if (tag) tag[i] = plan[i].tag;
    if (kind) kind[i] = plan[i].kind;
    if (count) count[i] = plan[i].count;
    if (dir) dir[i] = plan[i].dir;
  }
  return ok();
}

}  // extern "C"

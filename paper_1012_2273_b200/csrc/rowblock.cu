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
// metadata messages), the A-slices go out as grouped ncclSend/ncclRecv
// batches, B as ncclBroadcasts (NVLink/NVSwitch, not P-1 re-sends; in
// k-panels for big rounds, multiplied as they land), each rank multiplies its
// slice with kernels whose per-element arithmetic does not depend on the row
// offset, the slice height or a K split -- so P-GPU results are bitwise the
// 1-GPU results -- and the workers' C rows are stored by their GEMM epilogues
// straight into rank 0's C (CUDA IPC over NVLink; grouped C-slice messages
// when the allocation cannot be exported).  Rank 0 is master AND worker 0 (its
// GPU would otherwise idle).
//
// Failure detection (the reference's receive deadline, comm.hpp:144 /
// net.hpp:116-132, and its dead-worker ProtocolError naming the rank,
// protocol.hpp:74-77,88-101): communicators are created non-blocking
// (ncclConfig_t.blocking = 0), so no NCCL call parks the host thread; the
// host waits for a round with a deadline (MMWS_GPU_TIMEOUT_S, default 30 s)
// while polling ncclCommGetAsyncError.  Every rank stores its progress
// through a round (joined / inputs landed / multiplied / done) into a board
// on rank 0 -- one word per rank, mapped into the workers by CUDA IPC -- so
// when a round fails rank 0 can name the ranks that fell behind.  A failed
// round aborts the communicator (ncclCommAbort); mmws_gpu_comm_destroy +
// mmws_gpu_comm_init rebuild it.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/mmws_gpu.h"
#include "ctx.h"
#include "nccl_dl.h"

using namespace mmws_impl;

namespace {

#define NCCL_REQUIRE()                                                          \
  if (!nccl().ok) return fail(MMWS_GPU_ERR_NCCL, "libnccl.so.2 could not be loaded");

template <class T>
T* as_mut(const T* p) {
  return const_cast<T*>(p);
}

// ---------------------------------------------------------------- failure detection
using Clock = std::chrono::steady_clock;

struct Deadline {
  Clock::time_point end;
  explicit Deadline(double seconds)
      : end(Clock::now() + std::chrono::duration_cast<Clock::duration>(
                               std::chrono::duration<double>(seconds))) {}
  bool passed() const { return Clock::now() >= end; }
};

// Spin briefly (a round usually completes within microseconds of the event),
// then back off to 50 us sleeps.
inline void backoff(int& spins) {
  if (++spins < 4096) std::this_thread::yield();
  else std::this_thread::sleep_for(std::chrono::microseconds(50));
}

enum Stage : unsigned { JOINED = 1, INPUTS = 2, MULTIPLIED = 3, DONE = 4 };

const char* stage_name(unsigned s) {
  switch (s) {
    case JOINED: return "joined";
    case INPUTS: return "received its A rows and B";
    case MULTIPLIED: return "multiplied";
    case DONE: return "done";
    default: return "no round yet";
  }
}

// This rank's progress word in rank 0's board, in stream order on s.
void mark(mmws_gpu_ctx* ctx, cudaStream_t s, unsigned stage) {
  if (ctx->board_peer)
    launch_board_mark(ctx->launch(s), ctx->board_peer + ctx->rank, ctx->round * 8u + stage);
}

// Rank 0: the workers that had not finished round ctx->round, from the board
// (read on the idle copy stream), lowest progress first.
std::string laggards(mmws_gpu_ctx* ctx) {
  if (ctx->rank != 0 || !ctx->board || ctx->nranks < 2) return "";
  std::vector<unsigned> b(ctx->nranks, 0);
  if (cudaMemcpyAsync(b.data(), ctx->board, sizeof(unsigned) * ctx->nranks,
                      cudaMemcpyDeviceToHost, ctx->copy_in) != cudaSuccess ||
      cudaStreamSynchronize(ctx->copy_in) != cudaSuccess)
    return "";
  const unsigned want = ctx->round * 8u + DONE;
  unsigned low = want;
  for (int r = 1; r < ctx->nranks; ++r) low = std::min(low, b[r]);
  if (low >= want) return "";
  std::string out;
  for (int r = 1; r < ctx->nranks; ++r) {
    if (b[r] != low) continue;
    out += out.empty() ? "worker rank " : ", worker rank ";
    out += std::to_string(r);
  }
  const unsigned rd = low / 8u, st = low % 8u;
  out += low / 8u == ctx->round
             ? std::string(" stopped in round ") + std::to_string(rd) + " after it " + stage_name(st)
             : std::string(" never joined round ") + std::to_string(ctx->round) +
                   (low == 0 ? std::string(" (no round seen)")
                             : " (last seen: round " + std::to_string(rd) + ", " +
                                   stage_name(st) + ")");
  return out;
}

// A round (or the bootstrap) failed: name who fell behind, abort the
// communicator (its kernels exit, so every queued stream drains), report.
int round_failed(mmws_gpu_ctx* ctx, const char* what, ncclResult_t async, bool timed_out) {
  std::string who = laggards(ctx);
  if (ctx->comm) {
    nccl().CommAbort(ctx->comm);
    ctx->comm = nullptr;
  }
  ctx->comm_failed = true;
  cudaStreamSynchronize(ctx->comm_stream);
  cudaStreamSynchronize(ctx->stream);
  cudaGetLastError();
  std::string msg = std::string(what) + " (round " + std::to_string(ctx->round) + ", rank " +
                    std::to_string(ctx->rank) + " of " + std::to_string(ctx->nranks) + "): ";
  if (!timed_out)
    msg += std::string("NCCL reported ") + nccl().GetErrorString(async);
  else
    msg += "no progress within " + std::to_string(ctx->tune.timeout_s) + " s (deadlock-suspected)";
  if (!who.empty()) msg += "; " + who;
  else if (ctx->rank != 0) msg += "; waiting on the master (rank 0) or a peer";
  msg += "; communicator aborted (mmws_gpu_comm_destroy + mmws_gpu_comm_init to rebuild)";
  // a named rank that failed is the reference's ProtocolError
  // (protocol.hpp:74-77,88-101); an anonymous stall its TimeoutError (comm.hpp:144)
  return fail(!who.empty() || !timed_out ? MMWS_GPU_ERR_PROTOCOL : MMWS_GPU_ERR_TIMEOUT, msg);
}

// Wait for `ev` with the deadline while watching the communicator.  A round's
// deadline is the step timeout plus a generous allowance for its own
// arithmetic (ctx->round_work_s): like the reference's receive timeout, it
// must not fire on a worker that is merely still multiplying a big block.
int await(mmws_gpu_ctx* ctx, cudaEvent_t ev, const char* what) {
  const Deadline dl(ctx->tune.timeout_s + ctx->round_work_s);
  for (int spins = 0;; backoff(spins)) {
    const cudaError_t q = cudaEventQuery(ev);
    if (q == cudaSuccess) return MMWS_GPU_OK;
    if (q != cudaErrorNotReady) return cuda_fail(q, what);
    ncclResult_t a = ncclSuccess;
    if (ctx->comm && nccl().CommGetAsyncError(ctx->comm, &a) == ncclSuccess && a != ncclSuccess &&
        a != ncclInProgress)
      return round_failed(ctx, what, a, false);
    if (dl.passed()) return round_failed(ctx, what, ncclSuccess, true);
  }
}

// Result of an NCCL call on a non-blocking communicator: ncclInProgress
// means the call is still being set up (connections, ...) -- the next NCCL
// call may only follow once the communicator reports ncclSuccess.
int settle(mmws_gpu_ctx* ctx, ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return MMWS_GPU_OK;
  if (r != ncclInProgress) {
    ncclResult_t a = ncclSuccess;
    if (ctx->comm && nccl().CommGetAsyncError(ctx->comm, &a) == ncclSuccess && a != ncclSuccess &&
        a != ncclInProgress)
      return round_failed(ctx, what, a, false);
    return fail(MMWS_GPU_ERR_NCCL, std::string(what) + ": " + nccl().GetErrorString(r));
  }
  const Deadline dl(ctx->tune.timeout_s);
  for (int spins = 0;; backoff(spins)) {
    ncclResult_t a = ncclInProgress;
    nccl().CommGetAsyncError(ctx->comm, &a);
    if (a == ncclSuccess) return MMWS_GPU_OK;
    if (a != ncclInProgress) return round_failed(ctx, what, a, false);
    if (dl.passed()) return round_failed(ctx, what, ncclSuccess, true);
  }
}

#define NCCL_TRY(call, what)                                  \
  do {                                                        \
    if (int rc_ = settle(ctx, (call), what)) return rc_;       \
  } while (0)

// Who holds which rows, and the sub-block cut of every rank's rows -- derived
// by every rank from split_rows (protocol.hpp:33-46), so no metadata messages
// are needed.  S = 2 for the big configs: each sub-block is a whole number of
// 128-row bands, so a sub-block launch loses <2% to wave quantisation on 148
// SMs while half of the C gather hides behind the second multiply.
//
// B in k-panels (KP > 1, big rounds): B goes out as KP broadcasts of row
// panels of B (contiguous in row-major B), after the workers' first A
// sub-blocks, and a worker multiplies its first sub-block panel by panel as
// they land -- each launch continuing the previous one's accumulators
// (mmws_gpu_dgemm_acc semantics: bitwise the one-launch result, panel edges
// at multiples of 1024 k) -- instead of waiting for all of B (2 GiB at
// N=16384 fp64: ~3 ms of NVLink before any worker could start).
struct Schedule {
  int P = 1, S = 1, KP = 1;
  std::vector<int64_t> off, rows;
  std::vector<std::vector<int64_t>> soff, srows;  // [rank][sub-block], offsets within the rank
  std::vector<int64_t> kb;                        // B panel edges: KP + 1 entries, 0 .. k
};

constexpr int64_t PANEL_ELEMS = int64_t{32} << 20;  // 256 MiB of fp64 per B panel
constexpr int64_t PANEL_QUANTUM = 1024;              // fp32's partial-sum chunk (and 64 fp64 k-tiles)
constexpr int MAX_PANELS = 8;

// panels: the mode can continue accumulators across launches (all but OZAKI);
// host: a master_run round from host memory (B also streams over PCIe into
// rank 0, so rank 0 takes panels too -- even in a 1-rank world)
Schedule make_schedule(int64_t m, int64_t n, int64_t k, int P, bool panels, bool host = false) {
  Schedule sc;
  sc.P = P;
  sc.off.resize(P);
  sc.rows.resize(P);
  mmws_gpu_split_rows(m, P, sc.off.data(), sc.rows.data());
  sc.S = P > 1 && m / P >= 1024 ? 2 : 1;
  sc.soff.assign(P, std::vector<int64_t>(sc.S));
  sc.srows.assign(P, std::vector<int64_t>(sc.S));
  for (int r = 0; r < P; ++r)
    mmws_gpu_split_rows(sc.rows[r], sc.S, sc.soff[r].data(), sc.srows[r].data());
  sc.kb = {0};
  const double b_elems = static_cast<double>(k) * n;
  if ((P > 1 || host) && panels && b_elems >= 2.0 * PANEL_ELEMS) {
    const int want = static_cast<int>(std::min<double>(MAX_PANELS, b_elems / PANEL_ELEMS));
    for (int j = 1; j < want; ++j) {
      const int64_t e = (k * j / want) / PANEL_QUANTUM * PANEL_QUANTUM;
      if (e > sc.kb.back() && e < k) sc.kb.push_back(e);
    }
  }
  sc.kb.push_back(k);
  sc.KP = static_cast<int>(sc.kb.size()) - 1;
  return sc;
}

// Planning rates of mmws_gpu_rowblock_ranks (fixed, so every rank reaches
// the same decision without exchanging anything): the measured B200 peer
// copy bandwidth per direction (B200_PROFILING.md: 770 GB/s) and the
// measured 1-GPU multiply rates of this library (DMMA 36.3
// TFLOP/s at N=16384, FFMA2 67 TFLOP/s at N=32768), 60 us of collective
// latency per round.
constexpr double PLAN_LINK_BPS = 770e9;
constexpr double PLAN_FP64_FLOPS = 36.3e12, PLAN_FP32_FLOPS = 67e12;
constexpr double PLAN_ROUND_LATENCY_S = 60e-6;

// force: 0 cost model, -1 every rank, 1 rank 0 alone (MMWS_GPU_ROWBLOCK_RANKS)
int rowblock_active(int64_t m, int64_t n, int64_t k, int P, int elem_bytes, int force) {
  if (P <= 1) return 1;
  if (force == -1) return P;
  if (force == 1) return 1;
  double t1 = 0, tp = 0;
  const double rate = elem_bytes == 8 ? PLAN_FP64_FLOPS : PLAN_FP32_FLOPS;
  mmws_gpu_rowblock_cost(m, n, k, 1, elem_bytes, PLAN_LINK_BPS, rate, &t1, nullptr, nullptr);
  mmws_gpu_rowblock_cost(m, n, k, P, elem_bytes, PLAN_LINK_BPS, rate, &tp, nullptr, nullptr);
  ok();
  return tp + PLAN_ROUND_LATENCY_S < t1 ? P : 1;
}

// Enqueue one master/worker round.  Rank 0 passes device A, B, C (dense); the
// other ranks pass nulls and use library buffers.  On return ctx->ev1 (rank 0)
// is recorded after the last C row has landed and *done (if given) after this
// rank's part of the round.
//
// Without a communicator: one multiply.  With one (one rank per GPU, NCCL on
// ctx->comm_stream, multiplies on ctx->stream -- a 1-rank world takes this
// path too):
//   * fused gather: rank 0's C is mapped into every worker (CUDA IPC over
//     NVLink) and each worker's GEMM epilogue stores its rows straight into
//     it; a 4-byte allreduce after the last multiply is the completion
//     barrier.  The 80-byte handle is broadcast every call; whether the
//     mapping works is voted on (allreduce-min) only when the handle changed,
//     so a steady-state call needs no host round trip on rank 0;
//   * comm order, identical on every rank: handle, [vote], then either B (one
//     broadcast) and every rank's A-slice in S sub-blocks (grouped send/recv),
//     or -- B in KP k-panels (Schedule) -- the first A sub-blocks, the B
//     panels, the other A sub-blocks; without the fused gather, per sub-block
//     s the C-slice messages (grouped send/recv into C's row block on rank 0);
//   * a worker multiplies sub-block s as soon as its A rows and B landed (its
//     first sub-block panel by panel, continuing the accumulators);
//   * rank 0 multiplies its own rows meanwhile (it holds A and B already).
// Every launch computes each element with the same kernel and k-order as a
// 1-GPU launch, so the assembled C is bitwise the 1-GPU result.
//
// Host rounds (master_run_host, host = true on every rank): rank 0's A, B
// are the device staging buffers and hA, hB the caller's host matrices; rank
// 0 copies each piece over PCIe (copy_in stream) right before the NCCL
// operation that sends it -- the workers' first A rows, its own rows, the B
// panels, the workers' other A rows -- so the exchange and the workers start
// while the rest of A and B is still crossing PCIe, and rank 0 multiplies its
// own rows panel by panel as B lands, like a worker.  *own_done (rank 0) is
// recorded once rank 0's own rows of C are final.
template <class T>
int rowblock_enqueue(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const T* A, const T* B,
                     T* C, int mode, bool bracket, cudaEvent_t* done, bool host = false,
                     const T* hA = nullptr, const T* hB = nullptr,
                     cudaEvent_t* own_done = nullptr) {
  if (m <= 0 || n <= 0 || k <= 0)
    return fail(MMWS_GPU_ERR_DIMENSION, "rowblock: dimensions must be positive");
  if (ctx->comm_failed)
    return fail(MMWS_GPU_ERR_STATE, "rowblock: the communicator was aborted after a failed "
                                    "round; mmws_gpu_comm_destroy + mmws_gpu_comm_init first");
  const int P = ctx->comm ? ctx->nranks : 1;
  const int me = ctx->comm ? ctx->rank : 0;
  if (me == 0 && (!A || !B || !C))
    return fail(MMWS_GPU_ERR_DOMAIN, "rowblock: rank 0 needs A, B and C");
  cudaStream_t comp = ctx->stream, comm = ctx->comm_stream;
  cudaError_t e;
  if ((e = event_pool(ctx, 1)) != cudaSuccess) return cuda_fail(e, "rowblock: events");
  cudaEvent_t evDone = ctx->pool[0];
  if (done) *done = evDone;
  ctx->last_gather = 0;
  ctx->last_active = 1;

  if (!ctx->comm) {  // no communicator: one multiply
    if (bracket) cudaEventRecord(ctx->ev0, comp);
    cudaEventRecord(ctx->evk0, comp);
    if (int rc = gemm<T>(ctx, m, n, k, A, k, B, n, C, n, mode, comp)) return rc;
    cudaEventRecord(ctx->evk1, comp);
    if (bracket) cudaEventRecord(ctx->ev1, comp);
    cudaEventRecord(evDone, comp);
    return MMWS_GPU_OK;
  }
  NCCL_REQUIRE();
  if (P > 1 && rowblock_active(m, n, k, P, sizeof(T), ctx->tune.rowblock_ranks) == 1) {
    // too small to amortise the exchange: rank 0 multiplies alone, the
    // workers have nothing to do (every rank takes this branch for the same
    // arguments, so no collective is left half-matched).  A 1-rank world
    // still runs the exchange engine below (it is how one GPU tests it).
    cudaEventRecord(ctx->evk0, comp);
    if (me != 0) {
      cudaEventRecord(ctx->evk1, comp);
      cudaEventRecord(evDone, comp);
      return MMWS_GPU_OK;
    }
    if (bracket) cudaEventRecord(ctx->ev0, comp);
    if (int rc = gemm<T>(ctx, m, n, k, A, k, B, n, C, n, mode, comp)) return rc;
    cudaEventRecord(ctx->evk1, comp);
    if (bracket) cudaEventRecord(ctx->ev1, comp);
    cudaEventRecord(evDone, comp);
    return MMWS_GPU_OK;
  }
  // the multiplies below overlap NCCL transfers: no persistent (stream-K)
  // launches, which would keep the communication kernels off the SMs
  struct NoStreamK {
    mmws_gpu_ctx* c;
    ~NoStreamK() { c->allow_streamk = true; }
  } no_sk{ctx};
  ctx->allow_streamk = false;
  const Schedule sc = make_schedule(m, n, k, P, mode != MMWS_GPU_MODE_OZAKI, host);
  const int S = sc.S, KP = sc.KP;
  const bool stream_in = me == 0 && hA && hB;  // rank 0 of a host round
  const auto& off = sc.off;
  const auto& rows = sc.rows;
  const auto& soff = sc.soff;
  const auto& srows = sc.srows;
  const auto& kb = sc.kb;
  const ncclDataType_t dt = sizeof(T) == 8 ? ncclFloat64 : ncclFloat32;
  ++ctx->round;
  ctx->last_active = P;
  ctx->last_panels = KP;
  {
    int64_t rows_max = 0;
    for (int r = 0; r < P; ++r) rows_max = std::max(rows_max, rows[r]);
    // twice the slowest rank's multiply at 5 TFLOP/s (well below every mode)
    ctx->round_work_s = 2.0 * 2.0 * static_cast<double>(rows_max) * n * k / 5e12;
  }

  if ((e = event_pool(ctx, 3 * S + 2 * KP + 5)) != cudaSuccess)
    return cuda_fail(e, "rowblock: events");
  cudaEvent_t* evA = ctx->pool.data() + 1;
  cudaEvent_t* evC = evA + S;
  cudaEvent_t* evBp = evC + S;  // B panel j has landed
  cudaEvent_t evStart = evBp[KP], evJoin = evBp[KP + 1], evHost = evBp[KP + 2];
  cudaEvent_t* evHA = evBp + KP + 3;  // host round, rank 0: workers' A rows of sub-block s copied in
  cudaEvent_t* evHB = evHA + S;       // ... B panel j copied in
  cudaEvent_t evHself = evHB[KP];     // ... rank 0's own rows copied in
  if (own_done) *own_done = evC[S - 1];

  // the exchange starts after everything already queued on the compute stream
  // (e.g. the H2D copies of master_run_host)
  if (me == 0 && bracket) cudaEventRecord(ctx->ev0, comp);  // first send
  cudaEventRecord(evStart, comp);
  cudaStreamWaitEvent(comm, evStart, 0);
  mark(ctx, comm, JOINED);

  // ---- fused gather set-up (see above)
  // host ends of the small exchanges live in pinned memory: a copy to or from
  // pageable memory would block this thread on the comm stream (past the
  // deadline if a peer is gone)
  unsigned char* stage = static_cast<unsigned char*>(ctx->ipc_stage);
  unsigned char* hbuf = ctx->host_stage;
  int* vote_host = reinterpret_cast<int*>(ctx->host_stage + 128);
  std::memset(hbuf, 0, 80);
  if (me == 0) {
    hbuf[72] = !ctx->tune.nccl_gather && ipc_export(ctx, C, hbuf) == MMWS_GPU_OK ? 1 : 0;
    if ((e = cudaMemcpyAsync(stage, hbuf, 80, cudaMemcpyHostToDevice, comm)))
      return cuda_fail(e, "rowblock: stage IPC handle");
  }
  NCCL_TRY(nccl().Broadcast(stage, stage, 80, ncclUint8, 0, ctx->comm, comm), "broadcast C handle");
  if (me != 0) {
    if ((e = cudaMemcpyAsync(hbuf, stage, 80, cudaMemcpyDeviceToHost, comm)))
      return cuda_fail(e, "rowblock: fetch IPC handle");
    cudaEventRecord(evHost, comm);
    if (int rc = await(ctx, evHost, "rowblock: receive the master's C handle")) return rc;
  }
  T* c_peer = nullptr;
  int ok_here = hbuf[72] && !ctx->tune.nccl_gather;
  if (me != 0 && ok_here) {
    void* p = nullptr;
    ok_here = ipc_open(ctx, hbuf, &p, IPC_ROUND) == MMWS_GPU_OK ? 1 : 0;
    c_peer = static_cast<T*>(p);
  }
  int fused = ctx->last_fused;
  if (fused < 0 || std::memcmp(hbuf, ctx->last_handle, 80) != 0) {  // new handle: vote
    int* vote = reinterpret_cast<int*>(stage + 128);
    vote_host[0] = ok_here;
    if ((e = cudaMemcpyAsync(vote, vote_host, sizeof(int), cudaMemcpyHostToDevice, comm)))
      return cuda_fail(e, "rowblock: vote");
    NCCL_TRY(nccl().AllReduce(vote, vote, 1, ncclInt32, ncclMin, ctx->comm, comm),
             "agree on fused gather");
    if ((e = cudaMemcpyAsync(vote_host + 1, vote, sizeof(int), cudaMemcpyDeviceToHost, comm)))
      return cuda_fail(e, "rowblock: vote result");
    cudaEventRecord(evHost, comm);
    if (int rc = await(ctx, evHost, "rowblock: agree on the C gather")) return rc;
    fused = vote_host[1];
    std::memcpy(ctx->last_handle, hbuf, 80);
    ctx->last_fused = fused;
  }
  ok();  // a failed export/open only selects the NCCL gather
  ctx->last_gather = fused ? 1 : 2;

  const T* a_loc = A;
  const T* b_loc = B;
  T* c_loc = C;
  if (me != 0) {
    if ((e = ensure(ctx, &ctx->rbA, &ctx->rbA_bytes, sizeof(T) * (rows[me] * k + 1))) != cudaSuccess ||
        (e = ensure(ctx, &ctx->rbB, &ctx->rbB_bytes, sizeof(T) * k * n)) != cudaSuccess ||
        (!fused &&
         (e = ensure(ctx, &ctx->rbC, &ctx->rbC_bytes, sizeof(T) * (rows[me] * n + 1))) != cudaSuccess))
      return cuda_fail(e, "rowblock: worker buffers");
    a_loc = static_cast<const T*>(ctx->rbA);
    b_loc = static_cast<const T*>(ctx->rbB);
    c_loc = fused ? c_peer + off[me] * n : static_cast<T*>(ctx->rbC);
  }
  T* c_dst = c_loc;  // rank 0: C; workers: rank 0's C (fused) or the local slice
  // worker's (or a host round's rank 0's) running accumulators of its first
  // sub-block while B's panels land
  const bool paneled = KP > 1 && (me != 0 || stream_in);
  T* acc0 = nullptr;
  if (paneled && srows[me][0] > 0) {
    if ((e = ensure(ctx, &ctx->rbAcc, &ctx->rbAcc_bytes, sizeof(T) * srows[me][0] * n)) !=
        cudaSuccess)
      return cuda_fail(e, "rowblock: worker accumulators");
    acc0 = static_cast<T*>(ctx->rbAcc);
  }

  // ---- comm stream, part 1: the A-slices (protocol.hpp:70-72) sub-block by
  // sub-block and all of B (protocol.hpp:73) as KP panel broadcasts.  One
  // panel: B first (nothing can finish without all of it), then the A
  // sub-blocks.  Several: the first A sub-blocks, the panels, the other A
  // sub-blocks -- a worker starts once its first rows and panel 0 are in.
  // host round, rank 0: one piece over PCIe, then an event the dependent
  // NCCL operation (comm stream) or multiply (compute stream) waits on
  cudaStream_t in = ctx->copy_in;
  auto h2d_rows = [&](T* dst, const T* src, int64_t r0, int64_t nr, int64_t w) -> cudaError_t {
    if (nr <= 0) return cudaSuccess;
    return copy_h2d(ctx, dst + r0 * w, sizeof(T) * w, src + r0 * w, sizeof(T) * w,
                    sizeof(T) * w, static_cast<size_t>(nr), in);
  };
  auto h2d_a = [&](int s) -> int {  // every worker's A rows of sub-block s
    for (int r = 1; r < P; ++r)
      if ((e = h2d_rows(as_mut(A), hA, off[r] + soff[r][s], srows[r][s], k)) != cudaSuccess)
        return cuda_fail(e, "master_run: H2D A");
    cudaEventRecord(evHA[s], in);
    cudaStreamWaitEvent(comm, evHA[s], 0);
    return MMWS_GPU_OK;
  };
  auto h2d_self = [&]() -> int {  // rank 0's own rows
    if ((e = h2d_rows(as_mut(A), hA, 0, rows[0], k)) != cudaSuccess)
      return cuda_fail(e, "master_run: H2D A");
    cudaEventRecord(evHself, in);
    return MMWS_GPU_OK;
  };
  auto send_a = [&](int s) -> int {
    if (stream_in)
      if (int rc = h2d_a(s)) return rc;
    NCCL_TRY(nccl().GroupStart(), "ncclGroupStart");
    if (me == 0) {
      for (int r = 1; r < P; ++r)
        if (srows[r][s] > 0)
          NCCL_TRY(nccl().Send(A + (off[r] + soff[r][s]) * k, srows[r][s] * k, dt, r, ctx->comm,
                               comm), "send A-slice");
    } else if (srows[me][s] > 0) {
      NCCL_TRY(nccl().Recv(as_mut(a_loc) + soff[me][s] * k, srows[me][s] * k, dt, 0, ctx->comm,
                           comm), "recv A-slice");
    }
    NCCL_TRY(nccl().GroupEnd(), "ncclGroupEnd");
    cudaEventRecord(evA[s], comm);
    return MMWS_GPU_OK;
  };
  if (stream_in && bracket) cudaEventRecord(ctx->ev0, in);
  if (stream_in && KP == 1)
    if (int rc = h2d_self()) return rc;
  if (KP > 1)
    if (int rc = send_a(0)) return rc;
  if (stream_in && KP > 1)
    if (int rc = h2d_self()) return rc;
  for (int j = 0; j < KP; ++j) {
    T* bp = as_mut(b_loc) + kb[j] * n;
    if (stream_in) {
      if ((e = h2d_rows(bp - kb[j] * n, hB, kb[j], kb[j + 1] - kb[j], n)) != cudaSuccess)
        return cuda_fail(e, "master_run: H2D B");
      cudaEventRecord(evHB[j], in);
      cudaStreamWaitEvent(comm, evHB[j], 0);
    }
    NCCL_TRY(nccl().Broadcast(bp, bp, (kb[j + 1] - kb[j]) * n, dt, 0, ctx->comm, comm),
             "broadcast B");
    cudaEventRecord(evBp[j], comm);
  }
  for (int s = KP > 1 ? 1 : 0; s < S; ++s)
    if (int rc = send_a(s)) return rc;
  mark(ctx, comm, INPUTS);

  // ---- compute stream: this rank's rows (worker_run's body, protocol.hpp:132-141)
  cudaEventRecord(ctx->evk0, comp);
  // where this rank's inputs land: workers by NCCL; rank 0 of a host round by
  // its own H2D copies; rank 0 otherwise already holds them
  auto wait_b = [&](int j) {
    if (me != 0) cudaStreamWaitEvent(comp, evBp[j], 0);
    else if (stream_in) cudaStreamWaitEvent(comp, evHB[j], 0);
  };
  if (stream_in) cudaStreamWaitEvent(comp, evHself, 0);
  for (int s = 0; s < S; ++s) {
    const int64_t r0 = soff[me][s], rs = srows[me][s];
    if (me != 0) cudaStreamWaitEvent(comp, evA[s], 0);
    if (paneled && s == 0) {
      // panel by panel as B lands: launch j continues launch j-1's
      // accumulators (acc0), the last one stores into the destination
      for (int j = 0; j < KP; ++j) {
        wait_b(j);
        if (rs == 0) continue;
        T* out = j + 1 < KP ? acc0 : c_dst + r0 * n;
        if (int rc = gemm<T>(ctx, rs, n, kb[j + 1] - kb[j], a_loc + r0 * k + kb[j], k,
                             b_loc + kb[j] * n, n, out, n, mode, comp, j ? acc0 : nullptr, n))
          return rc;
      }
    } else {
      wait_b(KP - 1);  // all of B
      if (rs > 0)
        if (int rc = gemm<T>(ctx, rs, n, k, a_loc + r0 * k, k, b_loc, n, c_dst + r0 * n, n, mode,
                             comp))
          return rc;
    }
    if (s == S - 1) {
      cudaEventRecord(ctx->evk1, comp);
      mark(ctx, comp, MULTIPLIED);  // before evC: the DONE mark below waits on it
    }
    cudaEventRecord(evC[s], comp);
  }

  // ---- comm stream, part 2 (fused): the C rows are already in rank 0's C; one
  // 4-byte allreduce after every rank's last multiply is the completion
  // barrier (kernel completion makes the peer stores visible).
  if (fused) {
    cudaStreamWaitEvent(comm, evC[S - 1], 0);
    int* token = reinterpret_cast<int*>(static_cast<unsigned char*>(ctx->ipc_stage) + 192);
    NCCL_TRY(nccl().AllReduce(token, token, 1, ncclInt32, ncclSum, ctx->comm, comm),
             "completion barrier");
  }
  // ---- comm stream, part 2 (fallback): C-slices back into C's row blocks, rank
  // order (protocol.hpp:85-103), one grouped exchange per sub-block
  for (int s = 0; !fused && s < S; ++s) {
    if (me != 0) cudaStreamWaitEvent(comm, evC[s], 0);
    NCCL_TRY(nccl().GroupStart(), "ncclGroupStart");
    if (me == 0) {
      for (int r = 1; r < P; ++r)
        if (srows[r][s] > 0)
          NCCL_TRY(nccl().Recv(C + (off[r] + soff[r][s]) * n, srows[r][s] * n, dt, r, ctx->comm,
                               comm), "recv C-slice");
    } else if (srows[me][s] > 0) {
      NCCL_TRY(nccl().Send(c_dst + soff[me][s] * n, srows[me][s] * n, dt, 0, ctx->comm, comm),
               "send C-slice");
    }
    NCCL_TRY(nccl().GroupEnd(), "ncclGroupEnd");
  }
  if (!fused) cudaStreamWaitEvent(comm, evC[S - 1], 0);
  mark(ctx, comm, DONE);
  // join: the compute stream waits for the exchange, so the caller only
  // needs to synchronise ctx->stream
  cudaEventRecord(evJoin, comm);
  cudaStreamWaitEvent(comp, evJoin, 0);
  if (me == 0 && bracket) cudaEventRecord(ctx->ev1, comp);  // last receive
  cudaEventRecord(evDone, comp);
  return MMWS_GPU_OK;
}

// Wait for this rank's part of the round (with the deadline when peers are
// involved), then read the kernel and bracket timers.
int finish(mmws_gpu_ctx* ctx, cudaEvent_t done, bool timed, double* elapsed_s) {
  if (ctx->comm) {
    if (int rc = await(ctx, done, "rowblock round")) return rc;
  }
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
  cudaEvent_t done = nullptr;
  if (int rc = rowblock_enqueue(ctx, m, n, k, A, B, C, mode, true, &done)) return rc;
  return finish(ctx, done, root, elapsed_s);
}

// master_run with host matrices on rank 0: H2D of A and B, the round, D2H of
// C, all inside the elapsed bracket (the reference's master holds host data).
template <class T>
int master_run_host(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const T* A, const T* B,
                    T* C, int mode, double* elapsed_s) {
  const bool root = !ctx->comm || ctx->rank == 0;
  if (!root) {  // worker_run: the host round's schedule (B in panels where rank 0 uses them)
    cudaEvent_t done = nullptr;
    if (int rc = rowblock_enqueue(ctx, m, n, k, static_cast<const T*>(nullptr),
                                  static_cast<const T*>(nullptr), static_cast<T*>(nullptr), mode,
                                  true, &done, true))
      return rc;
    return finish(ctx, done, false, elapsed_s);
  }
  if (ctx->comm_failed)
    return fail(MMWS_GPU_ERR_STATE, "master_run: the communicator was aborted after a failed "
                                    "round; mmws_gpu_comm_destroy + mmws_gpu_comm_init first");
  // one GPU, or a round too small to distribute (rank 0 alone; the workers
  // return at once from the rowblock call above): copies overlapped with
  // the multiply
  if (!ctx->comm || (ctx->nranks > 1 && m > 0 && n > 0 && k > 0 &&
                     rowblock_active(m, n, k, ctx->nranks, sizeof(T),
                                     ctx->tune.rowblock_ranks) == 1)) {
    ctx->last_gather = 0;
    ctx->last_active = 1;
    return host_multiply(ctx, m, n, k, A, B, C, mode, elapsed_s);
  }
  if (m <= 0 || n <= 0 || k <= 0)
    return fail(MMWS_GPU_ERR_DIMENSION, "master_run: dimensions must be positive");
  if (!A || !B || !C) return fail(MMWS_GPU_ERR_DOMAIN, "master_run: null host matrix");
  const size_t a_b = sizeof(T) * m * k, b_b = sizeof(T) * k * n, c_b = sizeof(T) * m * n;
  cudaError_t e;
  if ((e = ensure(ctx, &ctx->dA, &ctx->dA_bytes, a_b)) != cudaSuccess ||
      (e = ensure(ctx, &ctx->dB, &ctx->dB_bytes, b_b)) != cudaSuccess ||
      (e = ensure(ctx, &ctx->dC, &ctx->dC_bytes, c_b)) != cudaSuccess)
    return cuda_fail(e, "master_run: device buffers");
  // the engine copies A and B in piece by piece, each right before the
  // exchange (or rank 0's multiply) that needs it; ev0 precedes the first copy
  cudaEvent_t done = nullptr, own = nullptr;
  if (int rc = rowblock_enqueue(ctx, m, n, k, static_cast<const T*>(ctx->dA),
                                static_cast<const T*>(ctx->dB), static_cast<T*>(ctx->dC), mode,
                                true, &done, true, A, B, &own))
    return rc;
  // copy-out: rank 0's own rows as soon as they are final, the workers' rows
  // once the round completed (within the deadline: a pageable C is pumped by
  // this thread, which would otherwise block on an unfinished round)
  const int64_t rows0 = make_schedule(m, n, k, ctx->nranks, false).rows[0];
  cudaStream_t out = ctx->copy_out;
  cudaStreamWaitEvent(out, own, 0);
  D2hPump pump(ctx, out);
  if ((e = pump.add(C, sizeof(T) * n, ctx->dC, sizeof(T) * n, sizeof(T) * n, rows0)) !=
      cudaSuccess)
    return cuda_fail(e, "master_run: D2H");
  if (int rc = await(ctx, done, "master_run round")) return rc;
  cudaStreamWaitEvent(out, done, 0);
  if ((e = pump.add(C + rows0 * n, sizeof(T) * n, static_cast<T*>(ctx->dC) + rows0 * n,
                    sizeof(T) * n, sizeof(T) * n, m - rows0)) != cudaSuccess ||
      (e = pump.finish()) != cudaSuccess)
    return cuda_fail(e, "master_run: D2H");
  cudaEventRecord(ctx->ev1, out);
  cudaEventRecord(done, out);
  if ((e = cudaStreamSynchronize(out)) != cudaSuccess) return cuda_fail(e, "master_run: sync");
  return finish(ctx, done, true, elapsed_s);
}

// Non-blocking communicator (see the header): returns once every rank has
// joined, or fails with MMWS_GPU_ERR_TIMEOUT after the deadline.
int comm_create(mmws_gpu_ctx* ctx, int nranks, int rank, const ncclUniqueId& uid) {
  ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
  cfg.blocking = 0;
  ncclComm_t comm = nullptr;
  ncclResult_t r = nccl().CommInitRankConfig(&comm, nranks, uid, rank, &cfg);
  if (r != ncclSuccess && r != ncclInProgress) {
    if (comm) nccl().CommAbort(comm);
    return fail(MMWS_GPU_ERR_NCCL, std::string("ncclCommInitRankConfig: ") + nccl().GetErrorString(r));
  }
  const Deadline dl(ctx->tune.timeout_s);
  for (int spins = 0;; backoff(spins)) {
    ncclResult_t a = ncclInProgress;
    nccl().CommGetAsyncError(comm, &a);
    if (a == ncclSuccess) break;
    if (a != ncclInProgress || dl.passed()) {
      nccl().CommAbort(comm);
      if (a != ncclInProgress)
        return fail(MMWS_GPU_ERR_NCCL, std::string("comm_init: ") + nccl().GetErrorString(a));
      return fail(MMWS_GPU_ERR_TIMEOUT,
                  "comm_init: rank " + std::to_string(rank) + " waited " +
                      std::to_string(ctx->tune.timeout_s) + " s for the other " +
                      std::to_string(nranks - 1) + " rank(s) of the world to join "
                      "(deadlock-suspected)");
    }
  }
  ctx->comm = comm;
  ctx->nranks = nranks;
  ctx->rank = rank;
  ctx->round = 0;
  ctx->round_work_s = 0.0;
  ctx->comm_failed = false;
  ctx->last_fused = -1;
  return MMWS_GPU_OK;
}

// The progress board: rank 0 allocates it and broadcasts its IPC handle;
// every rank maps it.  Without IPC the deadline still holds, the error just
// cannot name the rank that fell behind.
int board_setup(mmws_gpu_ctx* ctx) {
  cudaError_t e;
  unsigned char* h = ctx->host_stage + 256;  // pinned (see rowblock_enqueue)
  std::memset(h, 0, 80);
  if (ctx->rank == 0) {
    if ((e = cudaMalloc(&ctx->board, 256 + sizeof(unsigned) * ctx->nranks)) != cudaSuccess ||
        (e = cudaMemset(ctx->board, 0, 256 + sizeof(unsigned) * ctx->nranks)) != cudaSuccess)
      return cuda_fail(e, "comm_init: progress board");
    ctx->board_peer = ctx->board;
    h[72] = ipc_export(ctx, ctx->board, h) == MMWS_GPU_OK ? 1 : 0;
    ok();
  }
  unsigned char* stage = static_cast<unsigned char*>(ctx->ipc_stage);
  cudaStream_t s = ctx->comm_stream;
  if ((e = cudaMemcpyAsync(stage, h, 80, cudaMemcpyHostToDevice, s)) != cudaSuccess)
    return cuda_fail(e, "comm_init: board handle");
  NCCL_TRY(nccl().Broadcast(stage, stage, 80, ncclUint8, 0, ctx->comm, s), "comm_init: board handle");
  if ((e = cudaMemcpyAsync(h, stage, 80, cudaMemcpyDeviceToHost, s)) != cudaSuccess)
    return cuda_fail(e, "comm_init: board handle");
  if ((e = event_pool(ctx, 1)) != cudaSuccess) return cuda_fail(e, "comm_init: events");
  cudaEventRecord(ctx->pool[0], s);
  if (int rc = await(ctx, ctx->pool[0], "comm_init: board handle")) return rc;
  if (ctx->rank != 0 && h[72]) {
    void* p = nullptr;
    if (ipc_open(ctx, h, &p, IPC_COMM) == MMWS_GPU_OK) ctx->board_peer = static_cast<unsigned*>(p);
    ok();
  }
  return MMWS_GPU_OK;
}

// The host-only planning query (no context, not on a per-multiply path)
// reads the knob at call time.
Tuning host_tuning() { return Tuning::from_env(); }

}  // namespace

extern "C" {

int mmws_gpu_nccl_unique_id(uint8_t out[128]) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  if (!out) return fail(MMWS_GPU_ERR_DOMAIN, "nccl_unique_id: null out");
  NCCL_REQUIRE();
  ncclUniqueId id;
  if (ncclResult_t r = nccl().GetUniqueId(&id); r != ncclSuccess)
    return fail(MMWS_GPU_ERR_NCCL, std::string("ncclGetUniqueId: ") + nccl().GetErrorString(r));
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
  if (ctx->comm_failed)
    return fail(MMWS_GPU_ERR_STATE, "comm_init: call mmws_gpu_comm_destroy after a failed round");
  NCCL_REQUIRE();
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, 128);
  if (int rc = comm_create(ctx, nranks, rank, uid)) return rc;
  if (int rc = board_setup(ctx)) return rc;
  return ok();
}

int mmws_gpu_comm_destroy(mmws_gpu_ctx* ctx) {
  MMWS_CTX_GUARD(ctx);
  if (ctx->comm) {
    cudaStreamSynchronize(ctx->comm_stream);
    cudaStreamSynchronize(ctx->stream);
    const ncclResult_t r = nccl().CommDestroy(ctx->comm);
    ctx->comm = nullptr;
    if (r != ncclSuccess && r != ncclInProgress)
      return fail(MMWS_GPU_ERR_NCCL, std::string("ncclCommDestroy: ") + nccl().GetErrorString(r));
  }
  if (ctx->board) {
    cudaFree(ctx->board);
    ctx->board = nullptr;
  }
  ctx->board_peer = nullptr;
  ipc_close_scoped(ctx);  // this communicator's C and board mappings
  std::memset(ctx->last_handle, 0, sizeof ctx->last_handle);
  ctx->comm_failed = false;
  ctx->round = 0;
  ctx->nranks = 1;
  ctx->rank = 0;
  ctx->last_fused = -1;
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

int mmws_gpu_last_plan(mmws_gpu_ctx* ctx, const char** name) {
  if (!ctx || !name) return fail(MMWS_GPU_ERR_DOMAIN, "last_plan: null argument");
  *name = ctx->last_plan;
  return ok();
}

int mmws_gpu_link_probe(mmws_gpu_ctx* ctx, int64_t bytes, int iters, double* bytes_per_s) {
  MMWS_CTX_GUARD(ctx);
  if (bytes < 1 || iters < 1 || !bytes_per_s)
    return fail(MMWS_GPU_ERR_DOMAIN, "link_probe: bad arguments");
  if (!ctx->comm) return fail(MMWS_GPU_ERR_STATE, "link_probe: no communicator (comm_init)");
  NCCL_REQUIRE();
  cudaError_t e;
  if ((e = ensure(ctx, &ctx->rbB, &ctx->rbB_bytes, static_cast<size_t>(bytes))) != cudaSuccess)
    return cuda_fail(e, "link_probe: buffer");
  if ((e = event_pool(ctx, 1)) != cudaSuccess) return cuda_fail(e, "link_probe: events");
  ctx->round_work_s = static_cast<double>(bytes) * iters / 1e9;  // >= 1 GB/s
  cudaStream_t s = ctx->comm_stream;
  NCCL_TRY(nccl().Broadcast(ctx->rbB, ctx->rbB, bytes, ncclUint8, 0, ctx->comm, s),
           "link_probe warm-up");
  cudaEventRecord(ctx->ev0, s);
  for (int i = 0; i < iters; ++i)
    NCCL_TRY(nccl().Broadcast(ctx->rbB, ctx->rbB, bytes, ncclUint8, 0, ctx->comm, s),
             "link_probe broadcast");
  cudaEventRecord(ctx->ev1, s);
  cudaEventRecord(ctx->pool[0], s);
  if (int rc = await(ctx, ctx->pool[0], "link_probe")) return rc;
  float ms = 0.f;
  cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
  *bytes_per_s = static_cast<double>(bytes) * iters / (ms * 1e-3);
  return ok();
}

int mmws_gpu_p2p_probe(mmws_gpu_ctx* ctx, int64_t bytes, int iters, double* bytes_per_s) {
  MMWS_CTX_GUARD(ctx);
  if (bytes < 1 || iters < 1 || !bytes_per_s)
    return fail(MMWS_GPU_ERR_DOMAIN, "p2p_probe: bad arguments");
  if (!ctx->comm) return fail(MMWS_GPU_ERR_STATE, "p2p_probe: no communicator (comm_init)");
  NCCL_REQUIRE();
  *bytes_per_s = 0.0;
  if (ctx->nranks < 2) return ok();
  cudaError_t e;
  if ((e = ensure(ctx, &ctx->rbB, &ctx->rbB_bytes, static_cast<size_t>(bytes))) != cudaSuccess)
    return cuda_fail(e, "p2p_probe: buffer");
  if ((e = event_pool(ctx, 1)) != cudaSuccess) return cuda_fail(e, "p2p_probe: events");
  ctx->round_work_s = static_cast<double>(bytes) * (iters + 1) * ctx->nranks / 1e9;
  cudaStream_t s = ctx->comm_stream;
  // rank 0 -> rank r, one peer at a time (the A-slice / C-slice link); the
  // slowest peer is reported (rank 0's view; workers report their own link)
  double worst = 0.0;
  for (int r = 1; r < ctx->nranks; ++r) {
    if (ctx->rank != 0 && ctx->rank != r) continue;
    for (int i = 0; i <= iters; ++i) {  // i == 0: warm-up (connection set-up)
      if (i == 1) cudaEventRecord(ctx->ev0, s);
      if (ctx->rank == 0)
        NCCL_TRY(nccl().Send(ctx->rbB, bytes, ncclUint8, r, ctx->comm, s), "p2p_probe send");
      else
        NCCL_TRY(nccl().Recv(ctx->rbB, bytes, ncclUint8, 0, ctx->comm, s), "p2p_probe recv");
    }
    cudaEventRecord(ctx->ev1, s);
    cudaEventRecord(ctx->pool[0], s);
    if (int rc = await(ctx, ctx->pool[0], "p2p_probe")) return rc;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    const double bw = static_cast<double>(bytes) * iters / (ms * 1e-3);
    worst = worst == 0.0 ? bw : std::min(worst, bw);
  }
  *bytes_per_s = worst;
  return ok();
}

int mmws_gpu_last_round(mmws_gpu_ctx* ctx, int* active_ranks, int* gather, int* b_panels) {
  if (!ctx) return fail(MMWS_GPU_ERR_STATE, "null mmws_gpu_ctx");
  if (active_ranks) *active_ranks = ctx->last_active;
  if (gather) *gather = ctx->last_gather;
  if (b_panels) *b_panels = ctx->last_gather ? ctx->last_panels : 1;
  return ok();
}

int mmws_gpu_set_timeout(mmws_gpu_ctx* ctx, double seconds) {
  MMWS_CTX_GUARD(ctx);
  if (!(seconds > 0)) return fail(MMWS_GPU_ERR_DOMAIN, "set_timeout: seconds must be > 0");
  ctx->tune.timeout_s = seconds;
  return ok();
}

int mmws_gpu_rowblock_cost(int64_t m, int64_t n, int64_t k, int nranks, int elem_bytes,
                           double link_bytes_per_s, double gemm_flops_per_s, double* seconds,
                           double* root_egress_bytes, double* root_ingress_bytes) {
  // The analogue of the reference's cost model (cost_model.hpp:36-70, paper
  // s3.1.1: ((P-1)N^2 + 2N)(tc + tf) datums through the master) for this
  // schedule.  Rank 0's NVLink egress carries B once (broadcast) plus the
  // workers' A rows; its ingress carries the workers' C rows (peer stores).
  // Time = the slowest rank, a worker's multiplies starting as their inputs
  // arrive through rank 0's link in issue order (B in panels where the round
  // uses them); the C rows land while tiles finish (fused gather), so there
  // is no gather tail.  Per-op latencies are ignored (microseconds vs ms).
  if (m <= 0 || n <= 0 || k <= 0)
    return fail(MMWS_GPU_ERR_DIMENSION, "rowblock_cost: dimensions must be positive");
  if (nranks < 1 || (elem_bytes != 4 && elem_bytes != 8) || !(link_bytes_per_s > 0) ||
      !(gemm_flops_per_s > 0))
    return fail(MMWS_GPU_ERR_DOMAIN, "rowblock_cost: bad nranks / element size / rates");
  const Schedule sc = make_schedule(m, n, k, nranks, true);
  const double eb = elem_bytes, link = link_bytes_per_s, rate = gemm_flops_per_s;
  int64_t a_rows = 0;
  for (int r = 1; r < nranks; ++r) a_rows += sc.rows[r];
  const double egress = nranks > 1 ? eb * (static_cast<double>(k) * n + static_cast<double>(a_rows) * k) : 0.0;
  const double ingress = nranks > 1 ? eb * static_cast<double>(a_rows) * n : 0.0;
  // rank 0 alone, then (P > 1) each worker on the arrival times of rank 0's
  // egress sequence: [A sub-block 0 | B panels | A sub-blocks 1..] or, with
  // one panel, [B | A sub-blocks] -- rank 0's link carries them one after
  // another; the C rows land as tiles finish (fused gather)
  double t = 2.0 * static_cast<double>(sc.rows[0]) * n * k / rate;
  if (nranks > 1) {
    auto a_bytes = [&](int s) {
      double b = 0;
      for (int r = 1; r < nranks; ++r) b += eb * static_cast<double>(sc.srows[r][s]) * k;
      return b;
    };
    std::vector<double> t_a(sc.S), t_b(sc.KP);
    double sent = 0;
    if (sc.KP > 1) t_a[0] = (sent += a_bytes(0)) / link;
    for (int j = 0; j < sc.KP; ++j)
      t_b[j] = (sent += eb * static_cast<double>(sc.kb[j + 1] - sc.kb[j]) * n) / link;
    for (int s = sc.KP > 1 ? 1 : 0; s < sc.S; ++s) t_a[s] = (sent += a_bytes(s)) / link;
    for (int r = 1; r < nranks; ++r) {
      double tw = 0;
      for (int s = 0; s < sc.S; ++s) {
        const double rs = static_cast<double>(sc.srows[r][s]);
        if (s == 0 && sc.KP > 1) {
          tw = std::max(tw, t_a[0]);
          for (int j = 0; j < sc.KP; ++j)
            tw = std::max(tw, t_b[j]) + 2.0 * rs * n * (sc.kb[j + 1] - sc.kb[j]) / rate;
        } else {
          tw = std::max(tw, std::max(t_a[s], t_b[sc.KP - 1])) + 2.0 * rs * n * k / rate;
        }
      }
      t = std::max(t, tw);
    }
  }
  if (seconds) *seconds = t;
  if (root_egress_bytes) *root_egress_bytes = egress;
  if (root_ingress_bytes) *root_ingress_bytes = ingress;
  return ok();
}

int mmws_gpu_rowblock_ranks(int64_t m, int64_t n, int64_t k, int nranks, int elem_bytes,
                            int* active) {
  if (!active) return fail(MMWS_GPU_ERR_DOMAIN, "rowblock_ranks: null active");
  if (m <= 0 || n <= 0 || k <= 0)
    return fail(MMWS_GPU_ERR_DIMENSION, "rowblock_ranks: dimensions must be positive");
  if (nranks < 1 || (elem_bytes != 4 && elem_bytes != 8))
    return fail(MMWS_GPU_ERR_DOMAIN, "rowblock_ranks: bad nranks / element size");
  *active = rowblock_active(m, n, k, nranks, elem_bytes, host_tuning().rowblock_ranks);
  return ok();
}

int mmws_gpu_rowblock_plan(int64_t m, int64_t n, int64_t k, int nranks, int32_t* peer,
                           int32_t* tag, int32_t* kind, int64_t* count, int64_t* row0,
                           int32_t* dir, int32_t* n_entries) {
  if (!n_entries) return fail(MMWS_GPU_ERR_DOMAIN, "rowblock_plan: null n_entries");
  if (m <= 0 || n <= 0 || k <= 0)
    return fail(MMWS_GPU_ERR_DIMENSION, "rowblock_plan: dimensions must be positive");
  if (nranks < 1) return fail(MMWS_GPU_ERR_DOMAIN, "rowblock_plan: nranks must be >= 1");
  const Schedule sc = make_schedule(m, n, k, nranks, true);
  struct E { int32_t peer, tag, kind; int64_t count, row0; int32_t dir; };
  std::vector<E> plan;  // the order rowblock_enqueue issues on rank 0
  if (nranks > 1) {
    auto sends = [&](int s) {
      for (int r = 1; r < nranks; ++r)
        if (sc.srows[r][s] > 0)
          plan.push_back({r, 1, 1, sc.srows[r][s] * k, sc.off[r] + sc.soff[r][s], 0});
    };
    if (sc.KP > 1) sends(0);
    for (int j = 0; j < sc.KP; ++j)  // B panel j: rows [kb_j, kb_j+1) of B
      plan.push_back({-1, 1, 1, (sc.kb[j + 1] - sc.kb[j]) * n, sc.KP > 1 ? sc.kb[j] : -1, 2});
    for (int s = sc.KP > 1 ? 1 : 0; s < sc.S; ++s) sends(s);
    for (int s = 0; s < sc.S; ++s)
      for (int r = 1; r < nranks; ++r)
        if (sc.srows[r][s] > 0)
          plan.push_back({r, 2, 1, sc.srows[r][s] * n, sc.off[r] + sc.soff[r][s], 1});
  }
  const int32_t cap = *n_entries;
  *n_entries = static_cast<int32_t>(plan.size());
  if (cap < *n_entries) return ok();
  for (size_t i = 0; i < plan.size(); ++i) {
    if (peer) peer[i] = plan[i].peer;
    if (tag) tag[i] = plan[i].tag;
    if (kind) kind[i] = plan[i].kind;
    if (count) count[i] = plan[i].count;
    if (row0) row0[i] = plan[i].row0;
    if (dir) dir[i] = plan[i].dir;
  }
  return ok();
}

}  // extern "C"

/*
 * mmws_gpu.h -- C ABI of libmmws_gpu, the B200 (sm_100a) implementation of the
 * reference's dense-matmul hot path (arxiv/paper_1012_2273, "mmws").
 *
 * The reference exposes its hot path as inline C++ in namespace mmws (no FFI):
 *   Matrix matmul_seq(const Matrix&, const Matrix&)            matrix.hpp:112-126
 *   Matrix matmul_threads(const Matrix&, const Matrix&, unsigned) workshare.hpp:98-113
 *   std::vector<WorkAssignment> split_rows(int64_t, int)       protocol.hpp:33-46
 *   std::pair<Matrix,double> master_run(Communicator&, A, B)   protocol.hpp:50-108
 *   void worker_run(Communicator&)                              protocol.hpp:112-147
 *   Partition static_partition(size_t, unsigned)               workshare.hpp:33-46
 *   uint64_t op_count(int64_t)                                  matrix.hpp:130-134
 * Each entry point below names the one it replaces.  All paths are relative
 * to the reference tree's proj/ directory.  The C++ drop-in adapter that
 * restores the reference's signatures and exception types on top of this ABI
 * is include/mmws_gpu.hpp.
 *
 * Conventions: plain pointers and sizes, row-major matrices with explicit
 * leading dimensions (elements), every function returns an int status
 * (MMWS_GPU_OK == 0), no exception crosses the ABI, and the message of the
 * last failure on the calling thread is mmws_gpu_last_error().  A context is
 * bound to one CUDA device and serialises its callers with a mutex.  There is
 * no CPU fallback: without a usable sm_100 device mmws_gpu_init fails.
 */
#ifndef MMWS_GPU_H_
#define MMWS_GPU_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MMWS_GPU_ABI_VERSION 1

/* Status codes.  DIMENSION / DOMAIN mirror the reference's DimensionError /
 * DomainError (error.hpp:9-17); RANK / PROTOCOL / TIMEOUT mirror RankError /
 * ProtocolError / TimeoutError (error.hpp:20-39); CUDA / NCCL / ALLOC / STATE
 * are device-side failures the reference cannot have. */
enum {
  MMWS_GPU_OK = 0,
  MMWS_GPU_ERR_DIMENSION = 1,
  MMWS_GPU_ERR_DOMAIN = 2,
  MMWS_GPU_ERR_CUDA = 3,
  MMWS_GPU_ERR_NCCL = 4,
  MMWS_GPU_ERR_RANK = 5,
  MMWS_GPU_ERR_PROTOCOL = 6,
  MMWS_GPU_ERR_STATE = 7,
  MMWS_GPU_ERR_ALLOC = 8,
  MMWS_GPU_ERR_TIMEOUT = 9
};

/* Multiply modes.
 *   EXACT      per element acc = +0.0, then acc += a*b for k ascending with
 *              separate roundings: bitwise identical to matmul_seq for every
 *              NaN-free input (matrix.hpp:118-124).  FP64 pipe, DMUL+DADD.
 *   DMMA       FP64 tensor path (mma.sync m8n8k4 -> DMMA.8x8x4), 128x128 tiles,
 *              TMA + mbarrier pipeline.  Bit-exact for integer-valued inputs
 *              whose partial sums stay below 2^53; normwise <= 1e-12 otherwise.
 *   DMMA_SMALL same math on 32x32 tiles, 6 CTAs per SM (more CTAs for
 *              N < ~2000); bitwise the DMMA result.
 *   AUTO       fp64: the latency path (32x32 tiles, one DFMA chain per
 *              element, no TMA) when n <= 96 and k <= 96, else DMMA or
 *              DMMA_SMALL by tile count -- the choice never depends on m, so
 *              row slices of a problem get the whole problem's bits; fp32: FFMA.
 *              EXACT also switches to 32x32 tiles for small problems.
 *   FFMA       fp32 register-blocked FFMA GEMM (sgemm only).
 *   OZAKI      fp64 emulated exactly on the int8 tensor cores (tcgen05
 *              .kind::i8): power-of-two row/column scaling to t-bit integers,
 *              residues mod 14 coprime moduli <= 256, exact int8 GEMMs, CRT
 *              reconstruction.  Normwise error ~1e-14 for random inputs,
 *              bit-exact for integer-valued inputs, row-slice invariant;
 *              finite inputs only (Inf/NaN rows or columns give NaN), k <=
 *              131072.  Opt-in: AUTO stays on the FP64 tensor path (dgemm).
 *              sgemm takes it too (30-bit scaling, ~10 moduli: normwise error
 *              ~3e-8 -- the fp32 output rounding -- at 3.7x the FFMA2 rate). */
enum {
  MMWS_GPU_MODE_AUTO = 0,
  MMWS_GPU_MODE_EXACT = 1,
  MMWS_GPU_MODE_DMMA = 2,
  MMWS_GPU_MODE_DMMA_SMALL = 3,
  MMWS_GPU_MODE_FFMA = 4,
  MMWS_GPU_MODE_OZAKI = 5
};

/* Generator distributions over the reference's splitmix64 stream
 * (matrix.hpp:23-33, random_matrix matrix.hpp:101-107): element i of a
 * matrix is derived from the (i+1)-th output for `seed`.
 *   UNIT     (bits>>11) * 2^-53 in [0,1)         == mmws::random_matrix
 *   UNIFORM  2u - 1 in [-1,1)                     (configs C1, C2, C4)
 *   INT8     ((bits>>11)*17 >> 53) - 8 in [-8,8]  (config C3, exact)
 *   NORMAL   Box-Muller from draws 2i, 2i+1       (config C5, fp32)  */
enum {
  MMWS_GPU_DIST_UNIT = 0,
  MMWS_GPU_DIST_UNIFORM = 1,
  MMWS_GPU_DIST_INT8 = 2,
  MMWS_GPU_DIST_NORMAL = 3
};

/* Peak probes (mmws_gpu_peak_probe).  FFMA2_OUTER is the fp32 GEMM's own
 * operand pattern (a fresh broadcast register operand per FFMA2) in registers
 * only -- one such loop, below the plain FFMA2 peak; not a ceiling (its rate
 * depends on the register assignment). */
enum {
  MMWS_GPU_PROBE_DMMA = 0,
  MMWS_GPU_PROBE_DFMA = 1,
  MMWS_GPU_PROBE_DMUL_DADD = 2,
  MMWS_GPU_PROBE_FFMA = 3,
  MMWS_GPU_PROBE_FFMA2 = 4,
  MMWS_GPU_PROBE_FFMA2_OUTER = 5
};

typedef struct mmws_gpu_ctx mmws_gpu_ctx;
typedef struct mmws_gpu_graph mmws_gpu_graph;

/* ---------------------------------------------------------------- library */
int mmws_gpu_abi_version(void);
/* Message of the last failing call on this thread ("" if none). */
const char* mmws_gpu_last_error(void);

/* ---------------------------------------------------------------- context */
int mmws_gpu_init(int device, mmws_gpu_ctx** out);
int mmws_gpu_destroy(mmws_gpu_ctx* ctx);
int mmws_gpu_device_info(mmws_gpu_ctx* ctx, int* num_sms, int* cc_major, int* cc_minor,
                         int* max_clock_khz);
/* Number of kernels this context has launched so far (launch accounting). */
uint64_t mmws_gpu_launch_count(const mmws_gpu_ctx* ctx);
/* The context's own stream (cudaStream_t), used when a call passes NULL. */
void* mmws_gpu_stream(mmws_gpu_ctx* ctx);
/* Tuning / test knobs.  mmws_gpu_init reads them once from the environment
 * (never per call); this sets one on a live context by the same name (value
 * NULL or "": the default).  Knobs: MMWS_GPU_NO_STREAMK, MMWS_GPU_DMMA_PLAN,
 * MMWS_GPU_RASTER_GROUP, MMWS_GPU_PIPELINE_TRACE, MMWS_GPU_ROWBLOCK_RANKS
 * (all | 1), MMWS_GPU_SERVER_CTAS, MMWS_GPU_COPY_THREADS, MMWS_GPU_TIMEOUT_S,
 * MMWS_GPU_NCCL_GATHER (C-slices as NCCL messages instead of fused stores),
 * MMWS_GPU_SGEMM_AT (0 | 1: fp32 A staged as it lies | transposed, k-major). */
int mmws_gpu_tune(mmws_gpu_ctx* ctx, const char* knob, const char* value);

/* ---------------------------------------------------------------- host-only helpers */
/* split_rows (protocol.hpp:33-46): offset/rows arrays of n_workers entries. */
int mmws_gpu_split_rows(int64_t n_rows, int n_workers, int64_t* offset, int64_t* rows);
/* static_partition (workshare.hpp:33-46): start/len arrays of `workers` entries. */
int mmws_gpu_static_partition(uint64_t iterations, uint32_t workers, uint64_t* start,
                              uint64_t* len);
/* op_count (matrix.hpp:130-134): N^2 (2N - 1). */
int mmws_gpu_op_count(int64_t n, uint64_t* out);

/* ---------------------------------------------------------------- multiply, device pointers */
/* C[m,n] = A[m,k] . B[k,n] on device memory; replaces the inner loops of
 * matmul_seq (matrix.hpp:118-124), matmul_threads' body (workshare.hpp:105-111)
 * and worker_run's body (protocol.hpp:132-141).  Asynchronous on `stream`
 * (NULL = the context stream).  Zero dimensions are MMWS_GPU_ERR_DIMENSION as
 * in Matrix's constructor (matrix.hpp:72-78). */
int mmws_gpu_dgemm(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                   int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc, int mode,
                   void* stream);
int mmws_gpu_sgemm(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const float* A,
                   int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc, int mode,
                   void* stream);

/* Accumulating multiply, C = Cin + A.B (Cin m x n, leading dimension ldcin;
 * Cin may be C itself): every element's chain starts from its Cin value
 * instead of +0.0 and continues exactly as in mmws_gpu_dgemm.  Splitting K
 * into panels at multiples of 16 (fp64) / 1024 (fp32, the partial-sum chunk)
 * and chaining the calls (the first from +0.0 via mmws_gpu_dgemm / _sgemm)
 * therefore gives bitwise the one-call result -- what the row-block workers
 * use to multiply while B is still arriving -- as long as every call takes
 * the same kernel family as the one call: always in MODE_DMMA, MODE_DMMA_SMALL
 * and MODE_EXACT; in MODE_AUTO unless a piece falls under the DFMA latency
 * kernel's limit (n <= 96 and k <= 96) while the whole does not (or the
 * reverse).  All modes but OZAKI. */
int mmws_gpu_dgemm_acc(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                       int64_t lda, const double* B, int64_t ldb, const double* Cin,
                       int64_t ldcin, double* C, int64_t ldc, int mode, void* stream);
int mmws_gpu_sgemm_acc(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const float* A,
                       int64_t lda, const float* B, int64_t ldb, const float* Cin, int64_t ldcin,
                       float* C, int64_t ldc, int mode, void* stream);

/* MMWS_GPU_MODE_OZAKI plan for inner dimension k: number of int8 tensor-core
 * GEMMs (moduli) and the integer bits each row of A / column of B is scaled to
 * (normwise error ~1.4 * 2^-bits for random inputs).  Host-only. */
int mmws_gpu_ozaki_plan(int64_t k, int* moduli, int* bits);

/* ---------------------------------------------------------------- multiply, host buffers */
/* The matmul_seq / matmul_threads replacement for host data: dense row-major
 * A (m x k), B (k x n) in, C (m x n) out.  Copies in, multiplies, copies out
 * and synchronises.  *elapsed_s (optional) is the device-measured time of the
 * whole call (H2D + multiply + D2H) -- the host wall time when the latency
 * server below takes the call.  Pinned host buffers give full PCIe
 * bandwidth; pageable ones work too. */
int mmws_gpu_matmul_host(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                         const double* B, double* C, int mode, double* elapsed_s);
int mmws_gpu_matmul_host_f32(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k,
                             const float* A, const float* B, float* C, int mode,
                             double* elapsed_s);

/* ---------------------------------------------------------------- generators */
/* Fill dst[rows, cols] (leading dimension ld, fp64 or fp32) with elements
 * first .. first + rows*cols - 1 of the seeded stream.  dist NORMAL requires
 * is_f32 == 1. */
int mmws_gpu_fill(mmws_gpu_ctx* ctx, int dist, uint64_t seed, void* dst, int64_t rows,
                  int64_t cols, int64_t ld, int is_f32, uint64_t first, void* stream);

/* ---------------------------------------------------------------- CUDA graphs (small-N path) */
/* Capture one fp64 multiply on fixed device buffers into a CUDA graph; replay
 * with mmws_gpu_graph_launch to pay one graph launch instead of the per-call
 * host work (tensor-map encoding, packing decisions, kernel launches). */
int mmws_gpu_graph_dgemm(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                         int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                         int mode, mmws_gpu_graph** out);
int mmws_gpu_graph_launch(mmws_gpu_graph* graph, void* stream);
/* A graph may outlive its context: mmws_gpu_destroy releases the device
 * resources of the context's live graphs, after which mmws_gpu_graph_launch
 * returns MMWS_GPU_ERR_STATE and mmws_gpu_graph_destroy only frees the handle
 * (which the caller still owns). */
int mmws_gpu_graph_destroy(mmws_gpu_graph* graph);

/* ---------------------------------------------------------------- latency server (N <= 96) */
/* A small resident grid serving tiny fp64 multiplies through pinned, mapped
 * host memory: no launch, copy or stream synchronisation per call.  While it
 * runs, mmws_gpu_matmul_host routes the shapes and modes it takes to it.
 * Results are bitwise those of mmws_gpu_dgemm in the same mode (AUTO or
 * EXACT).  The kernel holds MMWS_GPU_SERVER_CTAS SMs (default 8) until
 * mmws_gpu_server_stop (or destroy); while it runs, a device-wide synchronize
 * (cudaDeviceSynchronize, torch.cuda.synchronize, cudaFree) waits for it --
 * synchronise streams instead.  The same holds for the lazy loading
 * (CUDA_MODULE_LOADING=LAZY, the default) of a kernel first launched while it
 * runs: mmws_gpu_init loads all of this library's kernels; other libraries'
 * (torch, NCCL) need CUDA_MODULE_LOADING=EAGER or a warm-up launch first. */
int mmws_gpu_server_start(mmws_gpu_ctx* ctx);
/* Host matrices (any memory); m, n, k <= 96.  *elapsed_s = host wall time of
 * the call (copy in, compute, copy out). */
int mmws_gpu_server_dgemm(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const double* A,
                          int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                          int mode, double* elapsed_s);
int mmws_gpu_server_stop(mmws_gpu_ctx* ctx);

/* ---------------------------------------------------------------- IPC (same-node peers) */
/* Block until everything queued on the context stream has finished. */
int mmws_gpu_synchronize(mmws_gpu_ctx* ctx);
/* Export the device allocation holding `ptr` to another process on this node:
 * 72 bytes = CUDA IPC handle (64) + byte offset of ptr in the allocation (8).
 * Fails for memory that CUDA IPC cannot export (e.g. VMM allocations). */
int mmws_gpu_ipc_export(mmws_gpu_ctx* ctx, const void* ptr, uint8_t out[72]);
/* Map an exported pointer into this process (peer access enabled, mapping
 * cached per allocation until the context is destroyed). */
int mmws_gpu_ipc_open(mmws_gpu_ctx* ctx, const uint8_t in[72], void** ptr);

/* ---------------------------------------------------------------- measurement */
/* Runs one pipe-saturating probe kernel and returns its TFLOP/s. */
int mmws_gpu_peak_probe(mmws_gpu_ctx* ctx, int which, int iters, double* tflops);
/* Calibration of the row-block cost model (the analogue of the reference's
 * `bench calibrate`, bench_main.cpp:64-93, which fits tc/tf to its TCP link):
 * mmws_gpu_gemm_probe times `iters` device-resident n x n multiplies in `mode`
 * (inputs generated on the device, CUDA events) and returns the rate in
 * FLOP/s (2n^3 per multiply). */
int mmws_gpu_gemm_probe(mmws_gpu_ctx* ctx, int64_t n, int mode, int iters, double* flops_per_s);

/* ---------------------------------------------------------------- row-block distribution */
/* The master/worker row decomposition of master_run / worker_run
 * (protocol.hpp:50-147) over NCCL, one rank per GPU.  Bootstrap: rank 0 calls
 * mmws_gpu_nccl_unique_id and ships the 128 bytes to every rank by any means
 * (torch.distributed, the reference's launch.hpp control plane, MPI, ...);
 * every rank then calls mmws_gpu_comm_init. */
int mmws_gpu_nccl_unique_id(uint8_t out[128]);
/* Non-blocking NCCL communicator: returns once all nranks ranks joined, or
 * MMWS_GPU_ERR_TIMEOUT after the deadline (mmws_gpu_set_timeout). */
int mmws_gpu_comm_init(mmws_gpu_ctx* ctx, int nranks, int rank, const uint8_t id[128]);
int mmws_gpu_comm_destroy(mmws_gpu_ctx* ctx);

/* Collective over the context's communicator; every rank calls it with the
 * same m, n, k, mode.  Rank 0 (master) passes device pointers to dense A
 * (m x k), B (k x n) and C (m x n); the other ranks pass NULL.  Rows are split
 * with split_rows(m, nranks); rank r multiplies rows [offset_r, offset_r +
 * rows_r).  Unlike the reference's master (protocol.hpp:3-4) rank 0 also
 * computes its own block -- on a GPU box the master's device is a full worker.
 * Data movement: B broadcast from 0, A-slices 0->r (r >= 1), and each
 * worker's C rows into rank 0's C -- stored directly by the worker's GEMM
 * epilogue through a CUDA IPC mapping of rank 0's C over NVLink (fused
 * gather), or as NCCL C-slice messages when the allocation cannot be
 * IPC-exported; ranks with rows_r == 0 still take part (protocol.hpp:122-123).  *elapsed_s
 * (rank 0, optional) is first send -> last receive measured on the device
 * (the bracket of protocol.hpp:63,105).  Synchronous on return.  The round is
 * queued on the context stream (mmws_gpu_stream): A and B written on another
 * stream must be ordered before the call (an event wait on the context
 * stream, or a synchronisation of the producing stream). */
int mmws_gpu_rowblock_dgemm(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k,
                            const double* A, const double* B, double* C, int mode,
                            double* elapsed_s);
int mmws_gpu_rowblock_sgemm(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k, const float* A,
                            const float* B, float* C, int mode, double* elapsed_s);

/* master_run (protocol.hpp:50-108) for host matrices: rank 0 passes dense host
 * A (m x k), B (k x n) and receives C (m x n); other ranks pass NULL.  The
 * H2D copies of A and B, the round above and the D2H copy of C are all inside
 * *elapsed_s (rank 0).  With no communicator (or nranks == 1) this is the
 * single-GPU host-buffer multiply. */
int mmws_gpu_master_run_host(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k,
                             const double* A, const double* B, double* C, int mode,
                             double* elapsed_s);
int mmws_gpu_master_run_host_f32(mmws_gpu_ctx* ctx, int64_t m, int64_t n, int64_t k,
                                 const float* A, const float* B, float* C, int mode,
                                 double* elapsed_s);
/* The most recent row-block / master_run call: how many ranks multiplied
 * (1 = rank 0 alone or no communicator), how C came back (0 no exchange,
 * 1 fused: worker GEMM epilogues stored into rank 0's C over CUDA IPC,
 * 2 NCCL C-slice messages) and in how many k-panels B was broadcast (> 1:
 * workers multiplied their first rows panel by panel as B landed).  Any
 * output may be NULL. */
int mmws_gpu_last_round(mmws_gpu_ctx* ctx, int* active_ranks, int* gather, int* b_panels);
/* Deadline of one distributed step (communicator bootstrap, a round, a probe):
 * default 30 s (the reference's receive timeout, comm.hpp:144), or
 * MMWS_GPU_TIMEOUT_S at mmws_gpu_init.  When it passes -- or NCCL reports a
 * failed peer -- the communicator is aborted and the call returns
 * MMWS_GPU_ERR_PROTOCOL naming the worker rank(s) that fell behind (from a
 * progress board every rank updates over NVLink), or MMWS_GPU_ERR_TIMEOUT
 * when no rank can be named.  Afterwards every row-block call fails with
 * MMWS_GPU_ERR_STATE until mmws_gpu_comm_destroy + mmws_gpu_comm_init. */
int mmws_gpu_set_timeout(mmws_gpu_ctx* ctx, double seconds);
/* Device time (ms, CUDA events on the launch stream) of this rank's multiply
 * kernel(s) in the most recent row-block / master_run call. */
int mmws_gpu_last_kernel_ms(mmws_gpu_ctx* ctx, double* ms);
/* Kernel configuration (a static, NUL-terminated string, e.g.
 * "dgemm_dmma_kernel<64x64, 4 math warps, 3 CTAs/SM>") the most recent
 * multiply on this context launched; "" before the first one. */
int mmws_gpu_last_plan(mmws_gpu_ctx* ctx, const char** name);

/* Cost model of one row-block round (the analogue of the reference's
 * cost_model.hpp:36-70): predicted seconds given the NVLink bandwidth per
 * direction and the per-GPU multiply rate, plus rank 0's egress (B once + the
 * workers' A rows) and ingress (the workers' C rows) in bytes.  Host-only. */
/* Collective over the context's communicator: `iters` broadcasts of `bytes`
 * from rank 0 (the B broadcast of a round), timed with CUDA events on the
 * communication stream; *bytes_per_s = bytes / time per broadcast on this
 * rank.  Needs mmws_gpu_comm_init. */
int mmws_gpu_link_probe(mmws_gpu_ctx* ctx, int64_t bytes, int iters, double* bytes_per_s);
/* Collective: `iters` point-to-point copies of `bytes` from rank 0 to each
 * worker in turn (the A-slice / C-slice link), timed on the communication
 * stream; *bytes_per_s = the slowest peer's rate on rank 0, the rank's own
 * link on a worker, 0 in a 1-rank world. */
int mmws_gpu_p2p_probe(mmws_gpu_ctx* ctx, int64_t bytes, int iters, double* bytes_per_s);
int mmws_gpu_rowblock_cost(int64_t m, int64_t n, int64_t k, int nranks, int elem_bytes,
                           double link_bytes_per_s, double gemm_flops_per_s, double* seconds,
                           double* root_egress_bytes, double* root_ingress_bytes);

/* Whether a row-block round over nranks GPUs is distributed at all (the north
 * star's "used only where N is large enough to amortise the transfers"):
 * *active = nranks when the cost model above, with fixed planning rates
 * (NVLink 770 GB/s per direction -- the measured B200 peer copy -- and the
 * library's measured 36.3 TFLOP/s fp64 / 62 TFLOP/s fp32 per GPU, 60 us of
 * collective latency per round), predicts the distributed round
 * to beat rank 0 multiplying alone, else 1: rank 0 computes every row and the
 * workers return at once (the reference's idle worker, protocol.hpp:122-123,
 * with no messages at all).  Every rank computes the same answer from its
 * arguments, so no agreement round is needed.  MMWS_GPU_ROWBLOCK_RANKS=all
 * (or =1) in the environment forces the choice.  Host-only. */
int mmws_gpu_rowblock_ranks(int64_t m, int64_t n, int64_t k, int nranks, int elem_bytes,
                            int* active);

/* The message plan rank 0 executes for (m, k, n, nranks), in issue order --
 * the analogue of the reference's Communicator traffic log (comm.hpp:24-32)
 * used by its protocol-shape test (test_protocol.cpp:99-137).  Host-only.
 * Order: one B broadcast, then the A-slices sub-block by sub-block, then the
 * C-slices sub-block by sub-block (offsets/row counts are derived from
 * split_rows on every rank, so there are no scalar metadata messages).  It
 * is the plan of a distributed round (see mmws_gpu_rowblock_ranks).
 * Entry e: peer[e] (-1 = all ranks), tag[e] (1 = assign, 2 = result),
 * kind[e] (1 = fp64/fp32 array), count[e] (elements), row0[e] (first row of
 * A or C the slice covers, -1 for B), dir[e] (0 sent, 1 received,
 * 2 broadcast).  *n_entries in: capacity, out: entries needed; any output
 * array may be NULL. */
int mmws_gpu_rowblock_plan(int64_t m, int64_t n, int64_t k, int nranks, int32_t* peer,
                           int32_t* tag, int32_t* kind, int64_t* count, int64_t* row0,
                           int32_t* dir, int32_t* n_entries);

#ifdef __cplusplus
}
#endif

#endif /* MMWS_GPU_H_ */

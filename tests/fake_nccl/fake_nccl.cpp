// fake_nccl.cpp -- TEST INFRASTRUCTURE ONLY: a loopback stand-in for the
// handful of NCCL entry points libmmws_gpu uses, so that several processes on
// ONE GPU can run the row-block master/worker engine end to end (the worker
// side included) where NCCL itself refuses two ranks on one device.
//
// libmmws_gpu loads it instead of libnccl.so.2 when MMWS_GPU_NCCL_LIB names it
// (csrc/nccl_dl.h).  Every transfer is a device-to-device copy between the
// processes' buffers through CUDA IPC (memory and interprocess events, driver
// API); the rendezvous and the message slots live in POSIX shared memory and
// are driven by the host threads.  No kernel ever waits on another process's
// kernel: ordering across processes is host rendezvous plus stream waits on
// IPC events.  Operations complete in call order per peer pair (the engine
// issues them in the same order on every rank); waits time out (15 s) with
// ncclRemoteError, which is how the dead-worker test sees a peer vanish.
// Not a product component: nothing under paper_1012_2273_b200/ links it.
#include <cuda.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

namespace {

constexpr int MAXR = 8;
constexpr double WAIT_S = 15.0;

struct Msg {
  std::atomic<uint32_t> seq;
  CUipcMemHandle mem;
  uint64_t off, bytes;
  CUipcEventHandle ready;
};
struct Ack {
  std::atomic<uint32_t> seq;
  CUipcEventHandle done;
};
struct Shm {
  std::atomic<int> joined;
  std::atomic<int> gone;
  Msg msg[MAXR][MAXR];  // [src][dst]
  Ack ack[MAXR][MAXR];  // [src][dst]: dst's copy of src's message done
  std::atomic<uint32_t> red_seq[MAXR];   // value of reduction `seq` posted
  std::atomic<uint32_t> red_read[MAXR];  // every value of reduction `seq` read
  int64_t red_val[MAXR];
};

struct Comm {
  int nranks = 0, rank = 0;
  std::string name;
  Shm* shm = nullptr;
  uint32_t sent[MAXR] = {}, recvd[MAXR] = {}, reductions = 0;
  ncclResult_t async = ncclSuccess;
  std::vector<CUevent> events;  // kept until destroy (peers may still open them)
  // per-peer rings of interprocess events, reused: message i to / from a peer
  // uses slot i % RING.  Safe because every send returns only after the
  // peer has queued its wait on the "ready" event, and the sender queues its
  // wait on "done" before the next message of the pair is posted (creating
  // a fresh interprocess event per message ran out after ~6000 of them)
  static constexpr int RING = 4;
  CUevent ready_ring[MAXR][RING] = {}, done_ring[MAXR][RING] = {};
  struct Open {
    CUipcMemHandle h;
    CUdeviceptr base;
  };
  std::vector<Open> opened;
};

bool wait_for(const std::atomic<uint32_t>& a, uint32_t want) {
  const auto t0 = std::chrono::steady_clock::now();
  while (a.load(std::memory_order_acquire) < want) {
    std::this_thread::yield();
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > WAIT_S)
      return false;
  }
  return true;
}

size_t type_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
  }
}

ncclResult_t cu_fail(const char* what, CUresult r, ncclResult_t code) {
  const char* name = nullptr;
  cuGetErrorName(r, &name);
  std::fprintf(stderr, "[fake_nccl] %s failed: %s\n", what, name ? name : "?");
  return code;
}

CUevent new_event(Comm* c) {
  CUevent e = nullptr;
  if (CUresult r = cuEventCreate(&e, CU_EVENT_INTERPROCESS | CU_EVENT_DISABLE_TIMING)) {
    cu_fail("cuEventCreate", r, ncclSystemError);
    return nullptr;
  }
  c->events.push_back(e);
  return e;
}

CUevent ring_event(Comm* c, CUevent* slot) {
  if (!*slot) *slot = new_event(c);
  return *slot;
}

CUdeviceptr open_mem(Comm* c, const CUipcMemHandle& h) {
  for (const auto& o : c->opened)
    if (!std::memcmp(&o.h, &h, sizeof h)) return o.base;
  CUdeviceptr p = 0;
  CUresult r = cuIpcOpenMemHandle(&p, h, CU_IPC_MEM_LAZY_ENABLE_PEER_ACCESS);
  if (r == CUDA_ERROR_ALREADY_MAPPED) {
    // the peer freed a buffer we still map and reallocated at its address:
    // drop the cached mappings (after the copies queued from them) and retry
    cuCtxSynchronize();
    for (auto& o : c->opened) cuIpcCloseMemHandle(o.base);
    c->opened.clear();
    r = cuIpcOpenMemHandle(&p, h, CU_IPC_MEM_LAZY_ENABLE_PEER_ACCESS);
  }
  if (r) {
    cu_fail("cuIpcOpenMemHandle", r, ncclSystemError);
    return 0;
  }
  c->opened.push_back({h, p});
  return p;
}

ncclResult_t fail(Comm* c) {
  c->async = ncclRemoteError;
  return ncclRemoteError;
}

ncclResult_t send(Comm* c, const void* buf, size_t bytes, int peer, CUstream s) {
  CUdeviceptr base = 0;
  size_t size = 0;
  if (cuMemGetAddressRange(&base, &size, reinterpret_cast<CUdeviceptr>(buf)) != CUDA_SUCCESS)
    return ncclInvalidArgument;
  Msg& m = c->shm->msg[c->rank][peer];
  if (CUresult r = cuIpcGetMemHandle(&m.mem, base))
    return cu_fail("cuIpcGetMemHandle", r, ncclSystemError);
  m.off = reinterpret_cast<CUdeviceptr>(buf) - base;
  m.bytes = bytes;
  const uint32_t seq = ++c->sent[peer];
  CUevent ready = ring_event(c, &c->ready_ring[peer][seq % Comm::RING]);
  if (!ready) return ncclSystemError;
  cuEventRecord(ready, s);
  cuIpcGetEventHandle(&m.ready, ready);
  m.seq.store(seq, std::memory_order_release);
  // the peer copies out of buf: wait for its copy before buf may change
  Ack& a = c->shm->ack[c->rank][peer];
  if (!wait_for(a.seq, seq)) return fail(c);
  CUevent done = nullptr;
  if (CUresult r = cuIpcOpenEventHandle(&done, a.done))
    return cu_fail("cuIpcOpenEventHandle(done)", r, ncclSystemError);
  cuStreamWaitEvent(s, done, 0);
  cuEventDestroy(done);
  return ncclSuccess;
}

ncclResult_t recv(Comm* c, void* buf, size_t bytes, int peer, CUstream s) {
  Msg& m = c->shm->msg[peer][c->rank];
  const uint32_t seq = ++c->recvd[peer];
  if (!wait_for(m.seq, seq)) return fail(c);
  if (m.bytes != bytes) return ncclInvalidUsage;
  const CUdeviceptr src = open_mem(c, m.mem);
  if (!src) return ncclSystemError;
  CUevent ready = nullptr;
  if (CUresult r = cuIpcOpenEventHandle(&ready, m.ready))
    return cu_fail("cuIpcOpenEventHandle(ready)", r, ncclSystemError);
  cuStreamWaitEvent(s, ready, 0);
  cuEventDestroy(ready);
  if (bytes)
    if (CUresult r = cuMemcpyDtoDAsync(reinterpret_cast<CUdeviceptr>(buf), src + m.off, bytes, s))
      return cu_fail("cuMemcpyDtoDAsync", r, ncclUnhandledCudaError);
  CUevent done = ring_event(c, &c->done_ring[peer][seq % Comm::RING]);
  if (!done) return ncclSystemError;
  cuEventRecord(done, s);
  Ack& a = c->shm->ack[peer][c->rank];
  cuIpcGetEventHandle(&a.done, done);
  a.seq.store(seq, std::memory_order_release);
  return ncclSuccess;
}

}  // namespace

extern "C" {

const char* ncclGetErrorString(ncclResult_t r) {
  switch (r) {
    case ncclSuccess: return "no error (fake)";
    case ncclRemoteError: return "remote process exited or there was a network error (fake)";
    case ncclInvalidArgument: return "invalid argument (fake)";
    case ncclInvalidUsage: return "invalid usage (fake)";
    default: return "error (fake)";
  }
}

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  std::memset(id->internal, 0, sizeof id->internal);
  std::random_device rd;
  std::snprintf(id->internal, sizeof id->internal, "/mmws_fake_nccl_%08x%08x", rd(), rd());
  return ncclSuccess;
}

ncclResult_t ncclCommInitRankConfig(ncclComm_t* out, int nranks, ncclUniqueId id, int rank,
                                    ncclConfig_t*) {
  if (nranks < 1 || nranks > MAXR || rank < 0 || rank >= nranks) return ncclInvalidArgument;
  cuInit(0);
  auto* c = new Comm();
  c->nranks = nranks;
  c->rank = rank;
  c->name = id.internal;
  const int fd = shm_open(c->name.c_str(), O_CREAT | O_RDWR, 0600);
  if (fd < 0 || ftruncate(fd, sizeof(Shm)) != 0) return ncclSystemError;
  c->shm = static_cast<Shm*>(mmap(nullptr, sizeof(Shm), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0));
  close(fd);
  if (c->shm == MAP_FAILED) return ncclSystemError;
  c->shm->joined.fetch_add(1);
  const auto t0 = std::chrono::steady_clock::now();
  while (c->shm->joined.load() < nranks) {
    std::this_thread::yield();
    if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > WAIT_S)
      return ncclRemoteError;
  }
  *out = reinterpret_cast<ncclComm_t>(c);
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* out, int nranks, ncclUniqueId id, int rank) {
  return ncclCommInitRankConfig(out, nranks, id, rank, nullptr);
}

ncclResult_t ncclCommGetAsyncError(ncclComm_t comm, ncclResult_t* err) {
  *err = reinterpret_cast<Comm*>(comm)->async;
  return ncclSuccess;
}

static ncclResult_t teardown(ncclComm_t comm) {
  auto* c = reinterpret_cast<Comm*>(comm);
  for (auto& o : c->opened) cuIpcCloseMemHandle(o.base);
  if (c->shm->gone.fetch_add(1) + 1 == c->nranks) shm_unlink(c->name.c_str());
  munmap(c->shm, sizeof(Shm));
  for (CUevent e : c->events) cuEventDestroy(e);
  delete c;
  return ncclSuccess;
}

ncclResult_t ncclCommAbort(ncclComm_t comm) { return teardown(comm); }
ncclResult_t ncclCommDestroy(ncclComm_t comm) { return teardown(comm); }
ncclResult_t ncclGroupStart() { return ncclSuccess; }
ncclResult_t ncclGroupEnd() { return ncclSuccess; }

ncclResult_t ncclSend(const void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm,
                      cudaStream_t s) {
  return send(reinterpret_cast<Comm*>(comm), buf, count * type_size(t), peer,
              reinterpret_cast<CUstream>(s));
}

ncclResult_t ncclRecv(void* buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm,
                      cudaStream_t s) {
  return recv(reinterpret_cast<Comm*>(comm), buf, count * type_size(t), peer,
              reinterpret_cast<CUstream>(s));
}

ncclResult_t ncclBroadcast(const void* sendbuf, void* recvbuf, size_t count, ncclDataType_t t,
                           int root, ncclComm_t comm, cudaStream_t s) {
  auto* c = reinterpret_cast<Comm*>(comm);
  const size_t bytes = count * type_size(t);
  auto st = reinterpret_cast<CUstream>(s);
  if (c->rank != root) return recv(c, recvbuf, bytes, root, st);
  if (sendbuf != recvbuf && bytes)
    cuMemcpyDtoDAsync(reinterpret_cast<CUdeviceptr>(recvbuf),
                      reinterpret_cast<CUdeviceptr>(sendbuf), bytes, st);
  for (int r = 0; r < c->nranks; ++r)
    if (r != root)
      if (ncclResult_t e = send(c, recvbuf, bytes, r, st)) return e;
  return ncclSuccess;
}

// One int32 / int64 / double value (the engine's vote and completion barrier).
ncclResult_t ncclAllReduce(const void* sendbuf, void* recvbuf, size_t count, ncclDataType_t t,
                           ncclRedOp_t op, ncclComm_t comm, cudaStream_t s) {
  auto* c = reinterpret_cast<Comm*>(comm);
  if (count != 1 || type_size(t) > 8) return ncclInvalidUsage;
  auto st = reinterpret_cast<CUstream>(s);
  int64_t v = 0;
  cuMemcpyDtoHAsync(&v, reinterpret_cast<CUdeviceptr>(sendbuf), type_size(t), st);
  if (cuStreamSynchronize(st) != CUDA_SUCCESS) return ncclUnhandledCudaError;
  if (t == ncclInt32) v = static_cast<int64_t>(static_cast<int32_t>(v & 0xffffffff));
  const uint32_t seq = ++c->reductions;
  // the previous reduction's values must all have been read before this
  // rank's slot is overwritten
  for (int r = 0; r < c->nranks; ++r)
    if (!wait_for(c->shm->red_read[r], seq - 1)) return fail(c);
  c->shm->red_val[c->rank] = v;
  c->shm->red_seq[c->rank].store(seq, std::memory_order_release);
  int64_t acc = v;
  for (int r = 0; r < c->nranks; ++r) {
    if (!wait_for(c->shm->red_seq[r], seq)) return fail(c);
    const int64_t x = c->shm->red_val[r];
    if (r == c->rank) continue;
    acc = op == ncclMin ? std::min(acc, x) : op == ncclMax ? std::max(acc, x) : acc + x;
  }
  c->shm->red_read[c->rank].store(seq, std::memory_order_release);
  static thread_local int64_t out;
  out = acc;
  cuMemcpyHtoDAsync(reinterpret_cast<CUdeviceptr>(recvbuf), &out, type_size(t), st);
  return cuStreamSynchronize(st) == CUDA_SUCCESS ? ncclSuccess : ncclUnhandledCudaError;
}

}  // extern "C"

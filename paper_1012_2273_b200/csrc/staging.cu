// staging.cu -- host <-> device copies for pageable host buffers.
//
// cudaMemcpy from pageable memory runs at ~11 GB/s on the B200 boxes (the
// driver bounces it through its own pinned buffer on one thread), against
// ~55 GB/s from pinned memory; a plain std::vector / numpy matrix is
// pageable.  Here a pageable transfer is pumped through a ring of pinned
// chunks: a small pool of host threads copies chunk c+1 into pinned memory
// (~50 GB/s with 4 threads, 57-80 GB/s with 8-16, tools/memcpy_probe) while the copy
// engine moves chunk c, so PCIe stays busy.  H2D returns once the last chunk
// is queued (the caller's buffer is no longer needed); D2H (D2hPump) keeps up
// to three chunks in flight across calls and fills the caller's buffers by
// finish().  Measured figures: DESIGN.md 3.6.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "ctx.h"

namespace mmws_impl {

namespace {

constexpr size_t CHUNK = size_t(32) << 20;  // bytes per pinned chunk
constexpr int NSLOT = 4;
// below this a direct pageable cudaMemcpy (the driver's own staging) wins
// over a pinned slot.  With spinning workers (and copies up to 128 KB done
// by the caller alone) the cut sits low: pageable host multiply (min of 40
// back-to-back calls) N=50 29.8 vs 45.3 us with a 2 MB cut, 180 51 vs 69,
// 250 72 vs 112, 350 108 vs 207, 500 199 vs 389; at N=10 (800 B) the
// driver's path is still a little faster
constexpr size_t STAGE_MIN = size_t(4) << 10;

// rows per chunk: at least four chunks per copy (so the host copy of one
// overlaps the DMA of the previous even for mid-size matrices), 1 MB to
// CHUNK bytes each
size_t rows_per_chunk(size_t width, size_t rows) {
  const size_t target = std::clamp(width * rows / 4, size_t(1) << 20, CHUNK);
  return std::clamp<size_t>(target / width, 1, CHUNK / width);
}

// Row-pitched copy split over a persistent pool of host threads (the calling
// thread takes part 0).  A job is published with one atomic generation bump
// and its completion counted down atomically; after a job the workers spin
// for SPIN_NS before they block on the condition variable, so the chunk
// after next of the same transfer (a few tens of microseconds later) finds
// them awake -- a futex wake-up per chunk and thread cost more than copying
// a 2 MB chunk (N=1000 pageable host multiply: 1.3-1.7 ms with blocking
// workers).
class CopyPool {
 public:
  explicit CopyPool(int threads) : n_(threads) {
    for (int t = 1; t < n_; ++t) th_.emplace_back([this, t] { worker(t); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> g(mu_);
      stop_.store(true, std::memory_order_relaxed);
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  // dst/src row-pitched regions of `rows` rows x `width` bytes.
  void copy(char* dst, size_t dpitch, const char* src, size_t spitch, size_t width,
            size_t rows) {
    if (width * rows <= INLINE_MAX) {  // not worth a hand-off: the caller copies it
      for (size_t r = 0; r < rows; ++r) std::memcpy(dst + r * dpitch, src + r * spitch, width);
      return;
    }
    job_ = {dst, dpitch, src, spitch, width, rows};
    pending_.store(n_ - 1, std::memory_order_relaxed);
    {
      std::lock_guard<std::mutex> g(mu_);  // pairs with a worker about to block
      gen_.fetch_add(1, std::memory_order_release);
    }
    cv_.notify_all();
    part(0);
    while (pending_.load(std::memory_order_acquire) != 0) cpu_relax();
  }

 private:
  static constexpr int64_t SPIN_NS = 200000;
  static constexpr size_t INLINE_MAX = size_t(128) << 10;
  struct Job {
    char* dst;
    size_t dpitch;
    const char* src;
    size_t spitch, width, rows;
  };
  static void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
  }
  void part(int t) {
    const Job j = job_;
    if (j.rows == 1 || (j.dpitch == j.width && j.spitch == j.width)) {  // one contiguous run
      const size_t total = j.width * j.rows;
      const size_t lo = total * t / n_, hi = total * (t + 1) / n_;
      if (hi > lo) std::memcpy(j.dst + lo, j.src + lo, hi - lo);
      return;
    }
    const size_t lo = j.rows * t / n_, hi = j.rows * (t + 1) / n_;
    for (size_t r = lo; r < hi; ++r) std::memcpy(j.dst + r * j.dpitch, j.src + r * j.spitch, j.width);
  }
  void worker(int t) {
    uint64_t seen = 0;
    for (;;) {
      const auto t0 = std::chrono::steady_clock::now();
      uint64_t g;
      int spins = 0;
      while ((g = gen_.load(std::memory_order_acquire)) == seen) {
        cpu_relax();
        if (++spins % 256 == 0 &&
            std::chrono::steady_clock::now() - t0 > std::chrono::nanoseconds(SPIN_NS)) {
          std::unique_lock<std::mutex> l(mu_);
          cv_.wait(l, [&] { return gen_.load(std::memory_order_acquire) != seen; });
        }
      }
      seen = g;
      if (stop_.load(std::memory_order_relaxed)) return;
      part(t);
      pending_.fetch_sub(1, std::memory_order_acq_rel);
    }
  }
  int n_;
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_;
  Job job_{};
  std::atomic<int> pending_{0};
  std::atomic<uint64_t> gen_{0};
  std::atomic<bool> stop_{false};
};

// cudaMemcpy2DAsync, as one linear copy when both sides are dense (a 2-D
// copy from pageable memory is much slower than the 1-D one)
cudaError_t copy2d(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                   size_t rows, cudaMemcpyKind kind, cudaStream_t s) {
  if (dpitch == width && spitch == width) return cudaMemcpyAsync(dst, src, width * rows, kind, s);
  return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, kind, s);
}

}  // namespace

struct Stager {
  CopyPool pool;
  char* slot[NSLOT] = {};
  cudaEvent_t ev[NSLOT] = {};
  bool held[NSLOT] = {};  // D2H chunk not yet copied out (D2hPump)
  explicit Stager(int threads) : pool(threads) {}
  // next chunk in round-robin order that no D2hPump still holds (at most
  // NSLOT - 1 are held), once its last transfer has finished
  cudaError_t take(mmws_gpu_ctx* ctx, int* k) {
    do {
      *k = static_cast<int>(ctx->stage_next++ % NSLOT);
    } while (held[*k]);
    return cudaEventSynchronize(ev[*k]);
  }
  ~Stager() {
    for (int s = 0; s < NSLOT; ++s) {
      if (ev[s]) cudaEventDestroy(ev[s]);
      if (slot[s]) cudaFreeHost(slot[s]);
    }
  }
};

namespace {

cudaError_t get_stager(mmws_gpu_ctx* ctx, Stager** out) {
  if (!ctx->stager) {
    const unsigned hw = std::thread::hardware_concurrency();
    // 3/4 of the host's cores, at most 12: 16-core box, N=8192 pageable
    // multiply 56 ms with 8 threads, 46 with 12, 44 with 16 (noisy)
    int threads = static_cast<int>(std::clamp(hw * 3 / 4, 1u, 12u));
    if (ctx->tune.copy_threads > 0) threads = ctx->tune.copy_threads;
    auto* st = new Stager(threads);
    for (int s = 0; s < NSLOT; ++s) {
      cudaError_t e;
      if ((e = cudaHostAlloc(reinterpret_cast<void**>(&st->slot[s]), CHUNK,
                             cudaHostAllocDefault)) != cudaSuccess ||
          (e = cudaEventCreateWithFlags(&st->ev[s], cudaEventDisableTiming)) != cudaSuccess) {
        delete st;
        return e;
      }
    }
    ctx->stager = st;
  }
  *out = static_cast<Stager*>(ctx->stager);
  return cudaSuccess;
}

}  // namespace

bool is_pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();  // clear: an unknown pointer is ordinary host memory
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

void staging_destroy(mmws_gpu_ctx* ctx) {
  delete static_cast<Stager*>(ctx->stager);
  ctx->stager = nullptr;
}

cudaError_t copy_h2d(mmws_gpu_ctx* ctx, void* dst, size_t dpitch, const void* src, size_t spitch,
                     size_t width, size_t rows, cudaStream_t s) {
  if (rows == 0 || width == 0) return cudaSuccess;
  if (width * rows < STAGE_MIN || width > CHUNK || !is_pageable(src))
    return copy2d(dst, dpitch, src, spitch, width, rows, cudaMemcpyHostToDevice, s);
  Stager* st;
  cudaError_t e = get_stager(ctx, &st);
  if (e != cudaSuccess) return e;
  const size_t per = rows_per_chunk(width, rows);
  for (size_t r0 = 0; r0 < rows; r0 += per) {
    const size_t nr = std::min(per, rows - r0);
    int k;
    if ((e = st->take(ctx, &k)) != cudaSuccess) return e;
    st->pool.copy(st->slot[k], width, static_cast<const char*>(src) + r0 * spitch, spitch, width,
                  nr);
    if ((e = copy2d(static_cast<char*>(dst) + r0 * dpitch, dpitch, st->slot[k], width, width, nr,
                    cudaMemcpyHostToDevice, s)) != cudaSuccess ||
        (e = cudaEventRecord(st->ev[k], s)) != cudaSuccess)
      return e;
  }
  return cudaSuccess;
}

D2hPump::D2hPump(mmws_gpu_ctx* ctx, cudaStream_t s) : ctx_(ctx), s_(s) {}

D2hPump::~D2hPump() { finish(); }

cudaError_t D2hPump::drain_one() {
  const Pending p = pending_.front();
  pending_.erase(pending_.begin());
  Stager* st = static_cast<Stager*>(ctx_->stager);
  st->held[p.slot] = false;
  cudaError_t e = cudaEventSynchronize(st->ev[p.slot]);
  if (e != cudaSuccess) return e;
  st->pool.copy(p.dst, p.dpitch, st->slot[p.slot], p.width, p.width, p.rows);
  return cudaSuccess;
}

cudaError_t D2hPump::add(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width,
                         size_t rows) {
  if (rows == 0 || width == 0) return cudaSuccess;
  if (width * rows < STAGE_MIN || width > CHUNK || !is_pageable(dst))
    return copy2d(dst, dpitch, src, spitch, width, rows, cudaMemcpyDeviceToHost, s_);
  Stager* st;
  cudaError_t e = get_stager(ctx_, &st);
  if (e != cudaSuccess) return e;
  const size_t per = rows_per_chunk(width, rows);
  for (size_t r0 = 0; r0 < rows; r0 += per) {
    // keep NSLOT - 1 chunks in flight: copy the oldest out while the rest move
    if (pending_.size() >= NSLOT - 1 && (e = drain_one()) != cudaSuccess) return e;
    const size_t nr = std::min(per, rows - r0);
    int k;
    if ((e = st->take(ctx_, &k)) != cudaSuccess) return e;
    st->held[k] = true;
    if ((e = copy2d(st->slot[k], width, static_cast<const char*>(src) + r0 * spitch, spitch, width,
                    nr, cudaMemcpyDeviceToHost, s_)) != cudaSuccess ||
        (e = cudaEventRecord(st->ev[k], s_)) != cudaSuccess)
      return e;
    pending_.push_back({static_cast<char*>(dst) + r0 * dpitch, dpitch, width, nr, k});
  }
  return cudaSuccess;
}

cudaError_t D2hPump::finish() {
  while (!pending_.empty())
    if (cudaError_t e = drain_one(); e != cudaSuccess) {
      for (const auto& p : pending_) static_cast<Stager*>(ctx_->stager)->held[p.slot] = false;
      pending_.clear();
      return e;
    }
  return cudaSuccess;
}

}  // namespace mmws_impl

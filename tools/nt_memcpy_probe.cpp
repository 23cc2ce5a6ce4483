// Development probe: pageable -> pinned host copy, glibc memcpy vs AVX
// non-temporal (streaming) stores, T threads, at the staging ring's chunk
// sizes -- alone and while the copy engine streams another pinned buffer to
// the GPU (the DMA competes for the same host memory).
//   g++ -O3 -mavx2 -std=c++17 tools/nt_memcpy_probe.cpp -o tools/nt_memcpy_probe \
//       -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart -lpthread
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

static void nt_copy(char* dst, const char* src, size_t n) {
  // head up to 32-byte alignment of dst, streamed body, tail
  size_t head = (32 - (reinterpret_cast<uintptr_t>(dst) & 31)) & 31;
  if (head > n) head = n;
  std::memcpy(dst, src, head);
  dst += head, src += head, n -= head;
  size_t body = n & ~size_t(127);
  for (size_t i = 0; i < body; i += 128) {
    __m256i a = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    __m256i b = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 32));
    __m256i c = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 64));
    __m256i d = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i + 96));
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i), a);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 32), b);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 64), c);
    _mm256_stream_si256(reinterpret_cast<__m256i*>(dst + i + 96), d);
  }
  _mm_sfence();
  std::memcpy(dst + body, src + body, n - body);
}

int main() {
  printf("threads available: %u\n", std::thread::hardware_concurrency());
  const size_t total = size_t(256) << 20;  // 256 MB pageable source
  char* src = static_cast<char*>(malloc(total));
  std::memset(src, 1, total);
  char* pin = nullptr;
  const size_t chunk = size_t(32) << 20;
  cudaHostAlloc(reinterpret_cast<void**>(&pin), 4 * chunk, cudaHostAllocDefault);
  std::memset(pin, 0, 4 * chunk);
  // background DMA source (pinned) and device sink
  char *bg = nullptr, *dbg = nullptr;
  cudaHostAlloc(reinterpret_cast<void**>(&bg), size_t(512) << 20, cudaHostAllocDefault);
  std::memset(bg, 2, size_t(512) << 20);
  cudaMalloc(&dbg, size_t(512) << 20);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int dma = 0; dma < 2; ++dma) {
    for (int T : {4, 8, 12, 16}) {
      for (int nt = 0; nt < 2; ++nt) {
        double best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEvent_t done;
          cudaEventCreate(&done);
          if (dma) {
            for (int i = 0; i < 8; ++i)
              cudaMemcpyAsync(dbg, bg, size_t(512) << 20, cudaMemcpyHostToDevice, s);
            cudaEventRecord(done, s);
          }
          auto t0 = std::chrono::steady_clock::now();
          // 256 MB through the 4 x 32 MB ring, each chunk split over T threads
          for (size_t off = 0; off < total; off += chunk) {
            char* d = pin + (off / chunk % 4) * chunk;
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t)
              th.emplace_back([=] {
                const size_t lo = chunk * t / T, hi = chunk * (t + 1) / T;
                if (nt) nt_copy(d + lo, src + off + lo, hi - lo);
                else std::memcpy(d + lo, src + off + lo, hi - lo);
              });
            for (auto& x : th) x.join();
          }
          const double sec =
              std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          best = std::min(best, sec);
          if (dma) cudaEventSynchronize(done);
          cudaEventDestroy(done);
        }
        printf("dma_bg=%d T=%2d %-8s %.1f GB/s\n", dma, T, nt ? "nt" : "memcpy",
               total / best / 1e9);
        fflush(stdout);
      }
    }
  }
  // DMA alone from pinned
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  for (int i = 0; i < 4; ++i) cudaMemcpyAsync(dbg, bg, size_t(512) << 20, cudaMemcpyHostToDevice, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("H2D from pinned alone: %.1f GB/s\n", 4.0 * (512 << 20) / (ms * 1e-3) / 1e9);
  // D2H into pinned
  cudaEventRecord(e0, s);
  for (int i = 0; i < 4; ++i) cudaMemcpyAsync(bg, dbg, size_t(512) << 20, cudaMemcpyDeviceToHost, s);
  cudaEventRecord(e1, s);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("D2H to pinned alone: %.1f GB/s\n", 4.0 * (512 << 20) / (ms * 1e-3) / 1e9);
  return 0;
}

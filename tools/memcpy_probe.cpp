// Development probe: host memcpy (pageable -> pinned / pageable) with T threads and
// H2D DMA from pinned vs pageable memory.  nvcc -O2 -std=c++17 tools/memcpy_probe.cpp -o tools/memcpy_probe
// host memcpy bandwidth: pageable -> pinned (cudaHostAlloc), T threads
#include <cuda_runtime.h>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <thread>
#include <vector>
int main() {
  const size_t bytes = size_t(512) << 20;
  char* src = static_cast<char*>(malloc(bytes));
  memset(src, 1, bytes);
  char* dst = nullptr;
  cudaHostAlloc(reinterpret_cast<void**>(&dst), bytes, cudaHostAllocDefault);
  memset(dst, 0, bytes);
  char* dst2 = static_cast<char*>(malloc(bytes));
  memset(dst2, 0, bytes);
  for (int T : {1, 2, 4, 8, 12, 16}) {
    for (int which = 0; which < 2; ++which) {
      char* d = which ? dst2 : dst;
      double best = 1e9;
      for (int rep = 0; rep < 3; ++rep) {
        auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
          th.emplace_back([=] {
            const size_t per = bytes / T;
            memcpy(d + t * per, src + t * per, per);
          });
        for (auto& x : th) x.join();
        best = std::min(best, std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
      }
      printf("T=%2d %s %.1f GB/s\n", T, which ? "pageable->pageable" : "pageable->pinned  ", bytes / best / 1e9);
    }
  }
  // DMA from pinned for reference
  void* dev;
  cudaMalloc(&dev, bytes);
  cudaMemcpy(dev, dst, bytes, cudaMemcpyHostToDevice);
  auto t0 = std::chrono::steady_clock::now();
  cudaMemcpy(dev, dst, bytes, cudaMemcpyHostToDevice);
  printf("H2D pinned %.1f GB/s\n", bytes / std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / 1e9);
  t0 = std::chrono::steady_clock::now();
  cudaMemcpy(dev, src, bytes, cudaMemcpyHostToDevice);
  printf("H2D pageable %.1f GB/s\n", bytes / std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() / 1e9);
  return 0;
}

// Development probe: what does pinning a pageable buffer for one transfer
// cost (cudaHostRegister + cudaHostUnregister), against staging it through
// pinned chunks?  Sizes of the paper's mid N (8 MB at N=1000 ... 128 MB at
// N=4096), buffers touched first (as a user's matrix is).
//   g++ -O3 -std=c++17 tools/host_register_probe.cpp -o tools/host_register_probe \
//       -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

using clk = std::chrono::steady_clock;
static double us(clk::time_point a, clk::time_point b) {
  return std::chrono::duration<double, std::micro>(b - a).count();
}

int main() {
  cudaFree(nullptr);
  void* dev = nullptr;
  cudaMalloc(&dev, size_t(128) << 20);
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (size_t mb : {2, 8, 18, 32, 72, 128}) {
    const size_t bytes = mb << 20;
    for (int rep = 0; rep < 4; ++rep) {
      char* p = static_cast<char*>(malloc(bytes + 123) ) + 123;  // unaligned, like any heap block
      std::memset(p, 1, bytes);
      auto t0 = clk::now();
      cudaError_t e = cudaHostRegister(p, bytes, cudaHostRegisterDefault);
      auto t1 = clk::now();
      cudaMemcpyAsync(dev, p, bytes, cudaMemcpyHostToDevice, s);
      cudaStreamSynchronize(s);
      auto t2 = clk::now();
      cudaHostUnregister(p);
      auto t3 = clk::now();
      cudaMemcpy(dev, p, bytes, cudaMemcpyHostToDevice);  // pageable, driver path
      auto t4 = clk::now();
      printf("%4zu MB rep %d: register %8.1f us (%s)  H2D %8.1f us (%.1f GB/s)  unregister %8.1f us"
             "  | pageable cudaMemcpy %8.1f us (%.1f GB/s)\n",
             mb, rep, us(t0, t1), cudaGetErrorString(e), us(t1, t2), bytes / us(t1, t2) / 1e3,
             us(t2, t3), us(t3, t4), bytes / us(t3, t4) / 1e3);
      free(p - 123);
    }
  }
  return 0;
}

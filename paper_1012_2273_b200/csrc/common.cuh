// common.cuh -- shared device helpers for the sm_100a kernels of libmmws_gpu.
//
// Inline PTX for the pieces the kernels build on: mbarriers, TMA tile loads,
// cp.async, the FP64 DMMA (mma.sync m8n8k4) and cache-hinted stores.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define MMWS_DEVICE __device__ __forceinline__

namespace mmws_dev {

MMWS_DEVICE uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------------ mbarrier
MMWS_DEVICE void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

MMWS_DEVICE void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

MMWS_DEVICE void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

MMWS_DEVICE void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

MMWS_DEVICE void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(smem_u32(bar)),
      "r"(bytes)
      : "memory");
}

MMWS_DEVICE void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------------------ TMA
MMWS_DEVICE void tma_prefetch_desc(const CUtensorMap* desc) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(desc)) : "memory");
}

// 2-D tile load global -> shared, completion signalled on `bar` (tx bytes).
MMWS_DEVICE void tma_load_2d(void* smem_dst, const CUtensorMap* desc, uint64_t* bar, int c0,
                             int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(desc)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// ------------------------------------------------------------------ cp.async
MMWS_DEVICE void cp_async_16(void* smem_dst, const void* gsrc, bool pred) {
  const int n = pred ? 16 : 0;  // src-size 0 => zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(smem_dst)),
               "l"(gsrc), "r"(n)
               : "memory");
}
MMWS_DEVICE void cp_async_8(void* smem_dst, const void* gsrc, bool pred) {
  const int n = pred ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(smem_dst)),
               "l"(gsrc), "r"(n)
               : "memory");
}
MMWS_DEVICE void cp_async_4(void* smem_dst, const void* gsrc, bool pred) {
  const int n = pred ? 4 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(smem_dst)),
               "l"(gsrc), "r"(n)
               : "memory");
}
MMWS_DEVICE void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
MMWS_DEVICE void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// ------------------------------------------------------------------ FP64 DMMA
// D(8x8) += A(8x4, row) * B(4x8, col).  Per lane (g = lane>>2, t = lane&3):
// a = A[g][t], b = B[t][g], d = {D[g][2t], D[g][2t+1]}.  One SASS DMMA.8x8x4.
// (volatile only pins source order; stage release relies on basic-block
// boundaries, see dgemm_dmma.cu)
MMWS_DEVICE void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}


}  // namespace mmws_dev

namespace mmws_dev {

// cp.async copy of a ROWS x COLS tile of a row-major matrix g (leading
// dimension ld) starting at (row0, col0) into shared memory s (row pitch SLD
// elements).  Elements outside [0, nrows) x [0, ncols) are zero-filled.
// VEC: 16-byte chunks -- requires a 16-byte aligned base, ld and ncols that
// are multiples of the chunk, so a chunk is either wholly inside or wholly
// outside the matrix.  !VEC: element-sized copies (any alignment).  Every
// thread of the CTA must call it.
template <typename T, int ROWS, int COLS, int SLD, int THREADS, bool VEC>
MMWS_DEVICE void load_tile_async(T* s, const T* __restrict__ g, int64_t ld, int row0, int col0,
                                 int nrows, int ncols) {
  constexpr int CH = VEC ? 16 / sizeof(T) : 1;  // elements per copy
  static_assert(COLS % CH == 0, "tile width must be a whole number of chunks");
  constexpr int CPR = COLS / CH;
  constexpr int TOTAL = ROWS * CPR;
#pragma unroll
  for (int it = 0; it < (TOTAL + THREADS - 1) / THREADS; ++it) {
    const int i = it * THREADS + threadIdx.x;
    if (TOTAL % THREADS != 0 && i >= TOTAL) break;
    const int r = i / CPR, c = (i % CPR) * CH;
    const int gr = row0 + r, gc = col0 + c;
    const bool ok = gr < nrows && gc < ncols;
    const T* src = ok ? g + static_cast<int64_t>(gr) * ld + gc : g;
    if constexpr (VEC)
      cp_async_16(s + r * SLD + c, src, ok);
    else if constexpr (sizeof(T) == 8)
      cp_async_8(s + r * SLD + c, src, ok);
    else
      cp_async_4(s + r * SLD + c, src, ok);
  }
}

}  // namespace mmws_dev

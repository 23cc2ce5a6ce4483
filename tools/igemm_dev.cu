// Development harness: int8 x int8 -> int32 GEMM on the 5th-generation tensor
// cores (tcgen05.mma .kind::i8, TMA-fed, accumulator in TMEM), epilogue
// C mod p -> uint8.  Batched over a third "modulus" dimension.  Checks a small
// case against a CPU reference and times a big one.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/igemm_dev.cu -lcuda -o tools/igemm_dev
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_1012_2273_b200/csrc/common.cuh"

using namespace mmws_dev;

namespace {

constexpr int BM = 128, BN = 256, BK = 128, STAGES = 4, THREADS = 128;
constexpr int A_BYTES = BM * BK, B_BYTES = BN * BK, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t TMEM_COLS = 256;

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// K-major operand, 128-byte swizzle, 8-row core groups 1024 bytes apart.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);          // start address
  d |= static_cast<uint64_t>(0) << 16;                         // LBO (unused, swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;                 // SBO
  d |= static_cast<uint64_t>(1) << 46;                         // version (sm100)
  d |= static_cast<uint64_t>(2) << 61;                         // SWIZZLE_128B
  return d;
}

// s8 x s8 -> s32, K-major A and B, M = 128, N = 256
constexpr uint32_t IDESC = (2u << 4) | (1u << 7) | (1u << 10) | ((BN >> 3) << 17) | ((BM >> 4) << 24);

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(IDESC), "r"(acc));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
    igemm_mod_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     uint8_t* __restrict__ C, int M, int N, int K, const int* __restrict__ mods,
                     int tiles_n) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tm = blockIdx.x / tiles_n, tn = blockIdx.x % tiles_n, z = blockIdx.z;
  const int KB = (K + BK - 1) / BK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0 && lane == 0) {  // TMA producer
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES;
      if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) - 1) & 1);
      uint8_t* sa = smem + s * STAGE_BYTES;
      mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
      tma_load_3d(sa, &tmA, &full[s], kb * BK, tm * BM, z);
      tma_load_3d(sa + A_BYTES, &tmB, &full[s], kb * BK, tn * BN, z);
    }
  } else if (warp == 1 && lane == 0) {  // MMA issuer
    for (int kb = 0; kb < KB; ++kb) {
      const int s = kb % STAGES;
      mbar_wait(&full[s], (kb / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t sa = smem_u32(smem + s * STAGE_BYTES);
      const uint32_t sb = sa + A_BYTES;
#pragma unroll
      for (int kk = 0; kk < BK / 32; ++kk)
        mma_i8(tmem, smem_desc(sa + kk * 32), smem_desc(sb + kk * 32), (kb | kk) != 0);
      mma_commit(&empty[s]);  // smem stage free once these MMAs have read it
    }
    mma_commit(tmem_full);
  }
  __syncwarp();
  // epilogue: lane = row within the warp's 32-row slice; 256 int32 columns
  mbar_wait(tmem_full, 0);
  asm volatile("tcgen05.fence::after_thread_sync;");
  const int row = tm * BM + warp * 32 + lane;
  const int p = mods[z];
  uint8_t* crow = C + (static_cast<size_t>(z) * M + row) * N + tn * BN;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (row < M) {
      uint8_t out[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        int r = static_cast<int>(v[j]) % p;
        out[j] = static_cast<uint8_t>(r < 0 ? r + p : r);
      }
      const int col = tn * BN + c0;
      if (col + 32 <= N) {
#pragma unroll
        for (int q = 0; q < 2; ++q)
          reinterpret_cast<uint4*>(crow + c0)[q] = reinterpret_cast<const uint4*>(out)[q];
      } else {
        for (int j = 0; j < 32 && col + j < N; ++j) crow[c0 + j] = out[j];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                             CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                             CUtensorMapFloatOOBfill);

bool map3(EncodeFn enc, CUtensorMap* m, const void* base, uint64_t k, uint64_t rows, uint64_t batch,
          uint32_t box_rows) {
  const cuuint64_t dims[3] = {k, rows, batch};
  const cuuint64_t strides[2] = {k, k * rows};
  const cuuint32_t box[3] = {BK, box_rows, 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

int main(int argc, char** argv) {
  const int M = argc > 1 ? atoi(argv[1]) : 256, N = argc > 2 ? atoi(argv[2]) : 512,
            K = argc > 3 ? atoi(argv[3]) : 384, Z = argc > 4 ? atoi(argv[4]) : 2;
  const bool check = argc > 5 ? atoi(argv[5]) : 1;
  std::vector<int8_t> A(static_cast<size_t>(Z) * M * K), B(static_cast<size_t>(Z) * N * K);
  uint64_t st = 12345;
  auto rnd = [&] { st = st * 6364136223846793005ULL + 1442695040888963407ULL; return static_cast<int8_t>(st >> 56); };
  for (auto& x : A) x = rnd();
  for (auto& x : B) x = rnd();
  std::vector<int> mods = {251, 256, 253, 241, 239, 233, 229, 227, 223, 211, 199, 197, 193, 191, 181, 179};
  mods.resize(Z);
  int8_t *dA, *dB;
  uint8_t* dC;
  int* dM;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dC, static_cast<size_t>(Z) * M * N);
  cudaMalloc(&dM, Z * sizeof(int));
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dM, mods.data(), Z * sizeof(int), cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(fn);
  CUtensorMap ta, tb;
  if (!map3(enc, &ta, dA, K, M, Z, BM) || !map3(enc, &tb, dB, K, N, Z, BN)) {
    printf("tensor map failed\n");
    return 1;
  }
  cudaFuncSetAttribute(igemm_mod_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  dim3 grid(tiles_m * tiles_n, 1, Z);
  igemm_mod_kernel<<<grid, THREADS, SMEM>>>(ta, tb, dC, M, N, K, dM, tiles_n);
  cudaError_t e = cudaDeviceSynchronize();
  printf("first launch: %s\n", cudaGetErrorString(e));
  if (e != cudaSuccess) return 1;
  if (check) {
    std::vector<uint8_t> C(static_cast<size_t>(Z) * M * N);
    cudaMemcpy(C.data(), dC, C.size(), cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int z = 0; z < Z; ++z)
      for (int i = 0; i < M; ++i)
        for (int j = 0; j < N; ++j) {
          long long s = 0;
          for (int k = 0; k < K; ++k)
            s += static_cast<long long>(A[(static_cast<size_t>(z) * M + i) * K + k]) *
                 B[(static_cast<size_t>(z) * N + j) * K + k];
          long long r = s % mods[z];
          if (r < 0) r += mods[z];
          if (C[(static_cast<size_t>(z) * M + i) * N + j] != r) {
            if (bad < 5) printf("mismatch z=%d i=%d j=%d got %d want %lld\n", z, i, j,
                                C[(static_cast<size_t>(z) * M + i) * N + j], r);
            ++bad;
          }
        }
    printf("check: %ld mismatches of %ld\n", bad, static_cast<long>(C.size()));
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e9;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    igemm_mod_kernel<<<grid, THREADS, SMEM>>>(ta, tb, dC, M, N, K, dM, tiles_n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  printf("M=%d N=%d K=%d Z=%d: %.3f ms, %.1f TOPS\n", M, N, K, Z, best,
         2.0 * M * N * K * Z / (best * 1e-3) / 1e12);
  return 0;
}

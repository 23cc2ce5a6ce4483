// ozaki.cu -- fp64 GEMM emulated exactly on the int8 tensor cores
// (MMWS_GPU_MODE_OZAKI; an opt-in mode, AUTO stays on DMMA).
//
// The FP64 tensor pipe (DMMA) peaks at 37 TFLOP/s on B200; the int8 tcgen05
// pipe at ~4.5 POPS.  The Ozaki scheme (Ozaki, Uchino, Imamura: "Ozaki Scheme
// II: a GEMM-oriented emulation of floating-point matrix multiplication using
// an integer modular technique") trades one fp64 GEMM for s exact int8 GEMMs:
//   1. scale every row of A and column of B by a power of two so its largest
//      magnitude is just below 2^t and round to integers A', B' (|A'|, |B'| <
//      2^t; the only rounding of the whole scheme, relative 2^-t per element);
//   2. for s pairwise-coprime moduli p_l <= 256, take signed residues
//      A'_l = A' mod p_l, B'_l = B' mod p_l (int8) and compute the exact int32
//      products A'_l B'_l on the tensor cores (|.| <= k * 128^2 < 2^31), kept
//      mod p_l as uint8;
//   3. rebuild C' = A'B' exactly from its residues by the Chinese remainder
//      theorem (P = prod p_l >= 4 k 2^(2t), 128-bit integers) and scale back:
//      C = C' * 2^-(e_i + f_j), one rounding to double.
// With s = 14 moduli (P ~ 2^110) and k <= 16384, t = 47: the normwise error is
// ~1.4 * 2^-47 ~ 1e-14 for random inputs (bound 1e-12), and integer-valued
// inputs come out bit-exact (C' is then the exact integer product).  Each
// element's result depends only on its row of A and column of B, so row
// slices give the same bits as the whole problem.  Inputs must be finite; a
// row or column holding Inf/NaN yields NaN in the affected outputs.  fp32
// operands go through the same kernels with 30-bit scaling (~10 moduli).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>

#include "common.cuh"
#include "kernels.h"

namespace mmws_impl {
namespace {

using namespace mmws_dev;

constexpr int OZ_MAX_MODULI = 16;
constexpr int OZ_NONFINITE = 1 << 20;  // exponent marker: row / column holds Inf or NaN
constexpr int OZ_GROUPS = 4;           // moduli groups pipelined residues -> GEMMs

// pairwise-coprime moduli, largest first (log2 of the product: 8, 16, 24, ...)
constexpr int kModuli[OZ_MAX_MODULI] = {256, 255, 253, 251, 247, 241, 239, 233,
                                        229, 227, 223, 211, 199, 197, 193, 191};

// CRT constants, passed to every kernel by value (__grid_constant__) -- no
// constant-memory upload, so concurrent calls and CUDA-graph replays each
// carry their own
struct CrtConst {
  int p[OZ_MAX_MODULI];
  int w[OZ_MAX_MODULI];          // (P / p_l)^-1 mod p_l
  uint64_t m_lo[OZ_MAX_MODULI];  // P / p_l, 128-bit
  uint64_t m_hi[OZ_MAX_MODULI];
  uint64_t P_lo, P_hi;
  double P_d, inv_P;
  // reconstruction (crt_kernel): fp32 forms of p_l, 1/p_l, w_l and the two
  // offsets of its (y w) mod p_l step, and D = -256 sum_l P/p_l mod P in
  // 32-bit limbs (cancels the +256 that keeps every residue term positive)
  float pf[OZ_MAX_MODULI], invf[OZ_MAX_MODULI], wf[OZ_MAX_MODULI];
  float c0[OZ_MAX_MODULI], c1[OZ_MAX_MODULI];
  uint32_t d[4];
  double pd[OZ_MAX_MODULI], invd[OZ_MAX_MODULI];  // residue kernels: p_l, fl(1 / p_l)
  int s;
};

// ---------------------------------------------------------------- scaling exponents
// e_i: amax_i * 2^e_i < 2^t for row i of A (frexp: amax = f 2^x, f in [0.5, 1))
template <class T>
__global__ void row_exponent_kernel(const T* __restrict__ A, int64_t lda, int m, int k, int t,
                                    int* __restrict__ e) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= m) return;
  const T* row = A + static_cast<int64_t>(warp) * lda;
  double amax = 0.0;
  bool finite = true;
  for (int j = lane; j < k; j += 32) {
    const double v = static_cast<double>(row[j]);
    finite = finite && isfinite(v);
    amax = fmax(amax, fabs(v));
  }
  for (int o = 16; o; o >>= 1) {
    amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
    finite = __all_sync(0xffffffffu, finite);
  }
  if (lane == 0) {
    int x = 0;
    frexp(amax, &x);
    e[warp] = !finite ? OZ_NONFINITE : (amax == 0.0 ? 0 : t - x);
  }
}

// f_j for column j of B (k x n, row-major).  |v| as a bit pattern orders
// like |v| (and Inf < NaN patterns sit above every finite value), so column
// maxima are atomicMax over 64-bit patterns from a 2-D grid of row blocks;
// col_exponent_finalize turns them into exponents.
constexpr int OZ_COL_ROWS = 256;  // rows per block of col_absmax_kernel
template <class T>
__global__ void col_absmax_kernel(const T* __restrict__ B, int64_t ldb, int k, int n,
                                  unsigned long long* __restrict__ colmax) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int r0 = blockIdx.y * OZ_COL_ROWS, r1 = min(k, r0 + OZ_COL_ROWS);
  unsigned long long mx = 0;
  for (int r = r0; r < r1; ++r) {
    const unsigned long long bits =
        static_cast<unsigned long long>(
            __double_as_longlong(static_cast<double>(B[static_cast<int64_t>(r) * ldb + j]))) &
        0x7fffffffffffffffULL;
    mx = bits > mx ? bits : mx;
  }
  atomicMax(colmax + j, mx);
}

__global__ void col_exponent_finalize(const unsigned long long* __restrict__ colmax, int n, int t,
                                      int* __restrict__ f) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const unsigned long long bits = colmax[j];
  if (bits >= 0x7ff0000000000000ULL) {
    f[j] = OZ_NONFINITE;
    return;
  }
  const double amax = __longlong_as_double(static_cast<long long>(bits));
  int x = 0;
  frexp(amax, &x);
  f[j] = amax == 0.0 ? 0 : t - x;
}

// signed residue of an integer-valued double (|x| < 2^52), on the FP64 pipe
// without conversions: q = rint(x / p) from one DFMA against 1.5 * 2^52
// (|x / p| < 2^45, so the sum lands where the ulp is 1), r = x - q p exactly
// (one DFMA), and r's two's-complement low word read off r + 1.5 * 2^52.  The
// estimate x * fl(1/p) is within 0.006 of x / p, so |r| <= p/2 + 1 and r > 127
// only for p in {255, 256}: one subtraction of p brings every case into int8.
// Any representative is fine: the GEMM epilogue reduces mod p.
constexpr double OZ_MAGIC = 6755399441055744.0;  // 1.5 * 2^52
MMWS_DEVICE uint32_t sresidue(double x, double pd, double inv) {
  const double q = __dadd_rn(__fma_rn(x, inv, OZ_MAGIC), -OZ_MAGIC);
  const double r = __fma_rn(-q, pd, x);
  int ri = static_cast<int>(__double2loint(__dadd_rn(r, OZ_MAGIC)));
  ri -= ri > 127 ? static_cast<int>(pd) : 0;
  return static_cast<uint32_t>(ri) & 0xffu;
}

// rint(v 2^ex), |result| < 2^52: one DMUL by an exact power of two where it is
// normal (the product is then exact or, for far-below-one results, rounds to
// a value whose rint is the same zero), ldexp otherwise
MMWS_DEVICE double scaled_int(double v, int ex) {
  if (ex == OZ_NONFINITE) return 0.0;
  const double y = (ex > -1023 && ex < 1024)
                       ? v * __longlong_as_double(static_cast<long long>(1023 + ex) << 52)
                       : ldexp(v, ex);
  return rint(y);
}

// residues of A' = rint(A 2^e): res[l][i][j], j < kpad (zero padding).
// A thread takes 8 consecutive j and stores one 8-byte word per modulus.
template <class T>
__global__ void residue_a_kernel(const T* __restrict__ A, int64_t lda, int m, int k, int kpad,
                                 const int* __restrict__ e, int8_t* __restrict__ res, int l0,
                                 int l1, const __grid_constant__ CrtConst c_crt) {
  const int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * 8;
  if (j0 >= kpad) return;
  for (int i = blockIdx.y; i < m; i += gridDim.y) {
    const int ex = e[i];
    const T* row = A + static_cast<int64_t>(i) * lda;
    double x[8];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      x[q] = j0 + q < k ? scaled_int(static_cast<double>(row[j0 + q]), ex) : 0.0;
    const int64_t plane = static_cast<int64_t>(m) * kpad;
    const int64_t o = static_cast<int64_t>(i) * kpad + j0;
    for (int l = l0; l < l1; ++l) {
      const double pd = c_crt.pd[l], inv = c_crt.invd[l];
      uint32_t lo = 0, hi = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        lo |= sresidue(x[q], pd, inv) << (8 * q);
        hi |= sresidue(x[q + 4], pd, inv) << (8 * q);
      }
      *reinterpret_cast<uint2*>(res + l * plane + o) = make_uint2(lo, hi);
    }
  }
}

// residues of B' = rint(B 2^f) transposed (K-major operand): res[l][j][r],
// r < kpad.  A block stages a 64 (k) x 32 (column) tile of scaled B through
// shared memory; thread t then owns column t/8 and 8 consecutive k, so each
// 8-thread group writes 64 contiguous bytes of one output row per modulus.
constexpr int OZ_BT_K = 64;
template <class T>
__global__ void __launch_bounds__(256) residue_bt_kernel(const T* __restrict__ B, int64_t ldb,
                                                         int k, int n, int kpad,
                                                         const int* __restrict__ f,
                                                         int8_t* __restrict__ res, int l0, int l1,
                                                         const __grid_constant__ CrtConst c_crt) {
  __shared__ double tile[OZ_BT_K][33];
  const int r0 = blockIdx.y * OZ_BT_K, c0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // load phase: 32 x 8
  {
    const int c = c0 + tx;
    const int fc = c < n ? f[c] : 0;
    for (int i = ty; i < OZ_BT_K; i += 8) {
      const int r = r0 + i;
      tile[i][tx] =
          (r < k && c < n)
              ? scaled_int(static_cast<double>(B[static_cast<int64_t>(r) * ldb + c]), fc)
              : 0.0;
    }
  }
  __syncthreads();
  const int col = threadIdx.x >> 3, kq = (threadIdx.x & 7) * 8;  // store phase
  const int c = c0 + col, rq = r0 + kq;
  if (c >= n || rq >= kpad) return;
  double x[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) x[q] = tile[kq + q][col];
  const int64_t plane = static_cast<int64_t>(n) * kpad;
  const int64_t o = static_cast<int64_t>(c) * kpad + rq;
  for (int l = l0; l < l1; ++l) {
    const double pd = c_crt.pd[l], inv = c_crt.invd[l];
    uint32_t lo = 0, hi = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      lo |= sresidue(x[q], pd, inv) << (8 * q);
      hi |= sresidue(x[q + 4], pd, inv) << (8 * q);
    }
    *reinterpret_cast<uint2*>(res + l * plane + o) = make_uint2(lo, hi);
  }
}

// ---------------------------------------------------------------- int8 tensor-core GEMM
// C_l = (A_l B_l^T) mod p_l for every modulus l, A_l: m x kpad, B_l: n x
// kpad (both K-major int8), C_l: m x n uint8.  256 x 256 tiles:
// tcgen05.mma.kind::i8 (M=128, N=256, K=32) issued by one thread, two per
// k-step sharing the B operand (64 KB per 128-byte k-block for 256x256
// outputs; 128x256 tiles needed 48 KB for half the outputs and ran 7 %
// slower), operands TMA-staged (128-byte swizzle, 3-stage ring), int32
// accumulators in TMEM (all 512 columns), epilogue tcgen05.ld -> mod p ->
// 16-byte stores.
constexpr int IG_BM = 256, IG_BN = 256, IG_BK = 128, IG_STAGES = 3;
constexpr int IG_HALVES = IG_BM / 128;                 // M=128 MMAs per k-step
constexpr int IG_NBUF = 512 / (IG_HALVES * IG_BN);    // TMEM accumulator buffers
constexpr int IG_EPI_WARPS = 4, IG_THREADS = (2 + IG_EPI_WARPS) * 32;
constexpr int IG_A_BYTES = IG_BM * IG_BK, IG_B_BYTES = IG_BN * IG_BK;
constexpr int IG_STAGE = IG_A_BYTES + IG_B_BYTES;
constexpr int IG_SMEM = IG_STAGES * IG_STAGE + 1024 + 256;
constexpr uint32_t IG_TMEM_COLS = 512;  // all of TMEM: IG_NBUF x IG_HALVES x 256 columns
// instruction descriptor: s32 accumulate, s8 x s8, K-major A and B, N = 256, M = 128
constexpr uint32_t IG_IDESC =
    (2u << 4) | (1u << 7) | (1u << 10) | ((IG_BN >> 3) << 17) | ((128 >> 4) << 24);

MMWS_DEVICE void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                             int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row core
// groups 1024 bytes apart (SBO), sm100 descriptor version 1
MMWS_DEVICE uint64_t umma_desc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFF) | (static_cast<uint64_t>(1024 >> 4) << 32) |
         (static_cast<uint64_t>(1) << 46) | (static_cast<uint64_t>(2) << 61);
}

MMWS_DEVICE void umma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(IG_IDESC), "r"(accumulate));
}

MMWS_DEVICE void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

// Persistent: one CTA per SM walks work items (modulus z, tile) z-major, with
// grouped rasterisation inside a modulus.  Warp 0 = TMA producer, warp 1 =
// MMA issuer, warps 2..5 = epilogue (TMEM lane quarter = warp % 4).  Two
// 256-column TMEM accumulators: the MMAs of item i+1 run while the epilogue
// drains item i (tmem_full / tmem_empty mbarriers).
__global__ void __launch_bounds__(IG_THREADS, 1)
    igemm_mod_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB,
                     uint8_t* __restrict__ C, int m, int n, int kpad, int tiles_m, int tiles_n,
                     int z0, int nz, const __grid_constant__ CrtConst c_crt) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + IG_STAGES * IG_STAGE);
  uint64_t* empty = full + IG_STAGES;
  uint64_t* tmem_full = empty + IG_STAGES;       // [IG_NBUF]
  uint64_t* tmem_empty = tmem_full + IG_NBUF;   // [IG_NBUF]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + IG_NBUF);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int KB = (kpad + IG_BK - 1) / IG_BK;
  const int tiles = tiles_m * tiles_n;
  const int items = tiles * nz;
  auto item_at = [&](int w, int& z, int& tm, int& tn) {
    z = z0 + w / tiles;
    const int tile = w % tiles;
    constexpr int GROUP = 8;  // 8 tile rows advance together (A/B panels shared in L2)
    const int per_group = GROUP * tiles_n;
    const int first_m = (tile / per_group) * GROUP;
    const int gm = min(tiles_m - first_m, GROUP);
    tm = first_m + (tile % per_group) % gm;
    tn = (tile % per_group) / gm;
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < IG_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < IG_NBUF; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], IG_EPI_WARPS);
    }
    fence_barrier_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(IG_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
      int kg = 0;  // stage counter across items
      for (int w = blockIdx.x; w < items; w += gridDim.x) {
        int z, tm, tn;
        item_at(w, z, tm, tn);
        for (int kb = 0; kb < KB; ++kb, ++kg) {
          const int s = kg % IG_STAGES;
          if (kg >= IG_STAGES) mbar_wait(&empty[s], ((kg / IG_STAGES) - 1) & 1);
          uint8_t* sa = smem + s * IG_STAGE;
          mbar_arrive_expect_tx(&full[s], IG_STAGE);
          tma_load_3d(sa, &tmA, &full[s], kb * IG_BK, tm * IG_BM, z);
          tma_load_3d(sa + IG_A_BYTES, &tmB, &full[s], kb * IG_BK, tn * IG_BN, z);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int kg = 0, it = 0;
      for (int w = blockIdx.x; w < items; w += gridDim.x, ++it) {
        const int b = it % IG_NBUF, use = it / IG_NBUF;
        mbar_wait(&tmem_empty[b], (use & 1) ^ 1);  // epilogue has drained buffer b
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t acc = tmem + b * IG_HALVES * IG_BN;
        for (int kb = 0; kb < KB; ++kb, ++kg) {
          const int s = kg % IG_STAGES;
          mbar_wait(&full[s], (kg / IG_STAGES) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;");
          const uint32_t sa = smem_u32(smem + s * IG_STAGE), sb = sa + IG_A_BYTES;
#pragma unroll
          for (int kk = 0; kk < IG_BK / 32; ++kk)  // K = 32 bytes per MMA, inside the swizzle row
#pragma unroll
            for (int h = 0; h < IG_HALVES; ++h)    // rows 128h.., accumulator columns 256h..
              umma_i8(acc + h * IG_BN, umma_desc(sa + h * 128 * IG_BK + kk * 32),
                      umma_desc(sb + kk * 32), (kb | kk) != 0);
          umma_commit(&empty[s]);  // the stage is free once these MMAs have read it
        }
        umma_commit(&tmem_full[b]);
      }
    }
  } else {  // epilogue warps 2..5: TMEM lanes 32*(warp%4) .. +31 = tile rows
    const int quarter = warp & 3;
    int it = 0;
    for (int w = blockIdx.x; w < items; w += gridDim.x, ++it) {
      int z, tm, tn;
      item_at(w, z, tm, tn);
      const int b = it % IG_NBUF, use = it / IG_NBUF;
      mbar_wait(&tmem_full[b], use & 1);
      asm volatile("tcgen05.fence::after_thread_sync;");
      const int p = c_crt.p[z];
#pragma unroll 1
      for (int h = 0; h < IG_HALVES; ++h) {
        const int row = tm * IG_BM + h * 128 + quarter * 32 + lane;
        uint8_t* crow = C + (static_cast<size_t>(z) * m + row) * n;
#pragma unroll 1
        for (int c0 = 0; c0 < IG_BN; c0 += 32) {
          uint32_t v[32];
          const uint32_t taddr = tmem + (static_cast<uint32_t>(quarter * 32) << 16) +
                                 (b * IG_HALVES + h) * IG_BN + c0;
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
              "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
              "%28, %29, %30, %31}, [%32];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
                "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
                "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
                "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
                "=r"(v[31])
              : "r"(taddr));
          asm volatile("tcgen05.wait::ld.sync.aligned;");
          if (h + 1 == IG_HALVES && c0 + 32 == IG_BN) {  // last read of buffer b: hand it back
            asm volatile("tcgen05.fence::before_thread_sync;");
            __syncwarp();
            if (lane == 0) mbar_arrive(&tmem_empty[b]);
          }
          const int col = tn * IG_BN + c0;
          if (row >= m || col >= n) continue;
          uint32_t packed[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            uint32_t word = 0;
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
              int r = static_cast<int>(v[4 * q + bb]) % p;  // C mod p in [0, p)
              r += r < 0 ? p : 0;
              word |= static_cast<uint32_t>(r) << (8 * bb);
            }
            packed[q] = word;
          }
          if (col + 32 <= n && (n % 16) == 0) {
            uint4* dst = reinterpret_cast<uint4*>(crow + col);
            dst[0] = make_uint4(packed[0], packed[1], packed[2], packed[3]);
            dst[1] = make_uint4(packed[4], packed[5], packed[6], packed[7]);
          } else {
            const uint8_t* bytes = reinterpret_cast<const uint8_t*>(packed);
            for (int j = 0; j < 32 && col + j < n; ++j) crow[col + j] = bytes[j];
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(IG_TMEM_COLS));
}

// ---------------------------------------------------------------- reconstruction
// C'_ij = sum_l ((y_l w_l) mod p_l) (P / p_l)  mod P, lifted to (-P/2, P/2],
// then C_ij = C' 2^-(e_i + f_j).  Grid (column blocks, rows); a thread takes 4
// consecutive columns (one 4-byte load per modulus, all s loads issued before
// any arithmetic).
//
// Per residue y (a byte), on the FP32 pipe and exact throughout:
//   Y  = 2^23 + y                     one PRMT (byte into a float's mantissa)
//   t  = Y w + (2^23 + 256 - 2^23 w)  = y w + 2^23 + 256   (one FFMA, exact)
//   q ~ rint(t / p - (2^23 + 256) / p) = rint(y w / p)     (error < 0.01)
//   r  = t - q p                      = 2^23 + 256 + z, z = y w - q p, |z| < p/2 + 2
//   u  = mantissa(r) & 0x1ff          = z + 256 in [1, 511]
// and u (P / p_l) is summed in four 32-bit limbs (IMAD.WIDE), D folding the
// +256 back out.  The sum stays below 44 P (< 2^124 for the s <= 15 the
// plans use); the nearest multiple of P comes from a double estimate, and the
// remainder is the signed C' itself (|C'| <= P/4 by the plan).
// acc += a * b (32 x 32 -> 64 bits) as one IMAD.WIDE.U32: written out so the
// compiler does not re-associate the four limb products into 64-bit multiplies
MMWS_DEVICE void mad_wide(uint64_t& acc, uint32_t a, uint32_t b) {
  asm("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(a), "r"(b));
}

MMWS_DEVICE double u128_to_double(unsigned __int128 v) {  // at most one extra rounding
  return static_cast<double>(static_cast<uint64_t>(v >> 64)) * 18446744073709551616.0 +
         static_cast<double>(static_cast<uint64_t>(v));
}

// S: the number of moduli as a compile-time count (the plans use 8..15; other
// counts run as S = 16 with zero terms: make_crt leaves P / p_l = 0 there)
template <class TO, int S>
__global__ void __launch_bounds__(128) crt_kernel(const uint8_t* __restrict__ Cres, int m, int n,
                                                  const int* __restrict__ e,
                                                  const int* __restrict__ f, TO* __restrict__ C,
                                                  int64_t ldc,
                                                  const __grid_constant__ CrtConst c_crt) {
  const int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (j0 >= n) return;
  const int64_t plane = static_cast<int64_t>(m) * n;
  const int s = c_crt.s;
  const bool vec = (n % 4) == 0;  // 4-byte aligned words (planes and rows)
  static_assert(S >= 1 && S <= OZ_MAX_MODULI, "moduli count");
  const unsigned __int128 P =
      (static_cast<unsigned __int128>(c_crt.P_hi) << 64) | static_cast<unsigned __int128>(c_crt.P_lo);
  for (int i = blockIdx.y; i < m; i += gridDim.y) {
    const int64_t base = static_cast<int64_t>(i) * n + j0;
    uint32_t word[S];
#pragma unroll
    for (int l = 0; l < S; ++l) {
      word[l] = 0;
      if (l < s) {
        if (vec) {
          word[l] = __ldcs(reinterpret_cast<const unsigned int*>(Cres + l * plane + base));
        } else {
          for (int q = 0; q < 4 && j0 + q < n; ++q)
            word[l] |= static_cast<uint32_t>(Cres[l * plane + base + q]) << (8 * q);
        }
      }
    }
    uint64_t limb[4][4];
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int b = 0; b < 4; ++b) limb[q][b] = c_crt.d[b];
#pragma unroll
    for (int l = 0; l < S; ++l) {
      {
        const float pf = c_crt.pf[l], inv = c_crt.invf[l], wf = c_crt.wf[l];
        const float c0 = c_crt.c0[l], c1 = c_crt.c1[l];
        const uint32_t m0 = static_cast<uint32_t>(c_crt.m_lo[l]);
        const uint32_t m1 = static_cast<uint32_t>(c_crt.m_lo[l] >> 32);
        const uint32_t m2 = static_cast<uint32_t>(c_crt.m_hi[l]);
        const uint32_t m3 = static_cast<uint32_t>(c_crt.m_hi[l] >> 32);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          // byte q of the word under exponent byte 0x4B: 2^23 + y
          const float Y = __uint_as_float(__byte_perm(word[l], 0x4B000000u, 0x7540u + q));
          const float t = __fmaf_rn(Y, wf, c0);
          const float qf = __fsub_rn(__fadd_rn(__fmaf_rn(t, inv, -c1), 12582912.0f), 12582912.0f);
          const float r = __fmaf_rn(-qf, pf, t);
          const uint32_t u = __float_as_uint(r) & 0x1ffu;
          mad_wide(limb[q][0], u, m0);
          mad_wide(limb[q][1], u, m1);
          mad_wide(limb[q][2], u, m2);
          mad_wide(limb[q][3], u, m3);
        }
      }
    }
    const int ex = e[i];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + q;
      if (j >= n) break;
      TO* out = C + static_cast<int64_t>(i) * ldc + j;
      const int fx = f[j];
      if (ex == OZ_NONFINITE || fx == OZ_NONFINITE) {
        *out = static_cast<TO>(__longlong_as_double(0x7ff8000000000000LL));
        continue;
      }
      const unsigned __int128 acc = static_cast<unsigned __int128>(limb[q][0]) +
                                    (static_cast<unsigned __int128>(limb[q][1]) << 32) +
                                    (static_cast<unsigned __int128>(limb[q][2]) << 64) +
                                    (static_cast<unsigned __int128>(limb[q][3]) << 96);
      // nearest multiple of P (the quotient is < 64)
      const uint32_t qt = __double2uint_rn(u128_to_double(acc) * c_crt.inv_P);
      const __int128 r = static_cast<__int128>(acc - static_cast<unsigned __int128>(qt) * P);
      const bool neg = r < 0;
      const double d = u128_to_double(static_cast<unsigned __int128>(neg ? -r : r));
      const int sh = ex + fx;  // C = C' 2^-sh: one DMUL by an exact power of two when it is normal
      const double v = neg ? -d : d;
      const double res = (sh > -1023 && sh < 1023)
                             ? v * __longlong_as_double(static_cast<long long>(1023 - sh) << 52)
                             : ldexp(v, -sh);
      *out = static_cast<TO>(res);
    }
  }
}

bool map3_u8(const Launch& L, CUtensorMap* map, const void* base, int64_t kpad, int64_t rows,
             int64_t batch, int box_rows) {
  const cuuint64_t dims[3] = {static_cast<cuuint64_t>(kpad), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(batch)};
  const cuuint64_t strides[2] = {static_cast<cuuint64_t>(kpad),
                                 static_cast<cuuint64_t>(kpad * rows)};
  const cuuint32_t box[3] = {IG_BK, static_cast<cuuint32_t>(box_rows), 1};
  const cuuint32_t es[3] = {1, 1, 1};
  return L.encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void*>(base), dims, strides,
                  box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// host: CRT constants for the first s moduli
void make_crt(int s, CrtConst* c) {
  c->s = s;
  unsigned __int128 P = 1;
  for (int l = 0; l < s; ++l) P *= static_cast<unsigned>(kModuli[l]);
  unsigned __int128 sumM = 0;
  for (int l = 0; l < OZ_MAX_MODULI; ++l) {
    const int p = kModuli[l];
    const unsigned __int128 M = l < s ? P / static_cast<unsigned>(p) : 0;
    int w = 1;
    if (l < s) {
      const int mr = static_cast<int>(M % static_cast<unsigned>(p));
      while ((mr * w) % p != 1) ++w;  // p <= 256: brute force
      sumM = (sumM + M) % P;
    }
    c->p[l] = p;
    c->w[l] = w;
    c->m_lo[l] = static_cast<uint64_t>(M);
    c->m_hi[l] = static_cast<uint64_t>(M >> 64);
    c->pd[l] = static_cast<double>(p);
    c->invd[l] = 1.0 / static_cast<double>(p);
    c->pf[l] = static_cast<float>(p);
    c->invf[l] = 1.0f / static_cast<float>(p);
    c->wf[l] = static_cast<float>(w);
    // exact: 256 (2^15 (1 - w) + 1), 24 significant bits at most
    c->c0[l] = 8388864.0f - 8388608.0f * static_cast<float>(w);
    c->c1[l] = 8388864.0f * c->invf[l];
  }
  // D = (-256 sum M_l) mod P
  unsigned __int128 k256 = sumM;  // 256 sumM mod P by doubling (P < 2^126: no overflow)
  for (int b = 0; b < 8; ++b) k256 = (k256 * 2u) % P;
  const unsigned __int128 D = k256 == 0 ? 0 : P - k256;
  for (int b = 0; b < 4; ++b) c->d[b] = static_cast<uint32_t>(D >> (32 * b));
  c->P_lo = static_cast<uint64_t>(P);
  c->P_hi = static_cast<uint64_t>(P >> 64);
  c->P_d = static_cast<double>(c->P_hi) * 18446744073709551616.0 + static_cast<double>(c->P_lo);
  c->inv_P = 1.0 / c->P_d;
}

}  // namespace

// Plan: number of moduli and integer bits for an inner dimension k; the
// smallest s whose product leaves at least `target` bits per operand.
void ozaki_plan_bits(int64_t k, int target, int* s_out, int* t_out) {
  const double logk = std::ceil(std::log2(static_cast<double>(std::max<int64_t>(k, 2))));
  double logP = 0;
  int s = 0, t = 0;
  for (s = 1; s <= OZ_MAX_MODULI; ++s) {
    logP += std::log2(static_cast<double>(kModuli[s - 1]));
    t = static_cast<int>(std::floor((logP - 2.0 - logk) / 2.0));
    if (t >= target) break;
  }
  if (s > OZ_MAX_MODULI) s = OZ_MAX_MODULI;
  *s_out = s;
  *t_out = std::min(t, 52);
}

// fp64: t >= 46 (~1.4 * 2^-46 ~ 2e-14 normwise for random inputs)
void ozaki_plan(int64_t k, int* s, int* t) { ozaki_plan_bits(k, 46, s, t); }

namespace {

template <class T>
void plan_for(int64_t k, int* s, int* t) {
  if constexpr (sizeof(T) == 8)
    ozaki_plan_bits(k, 46, s, t);  // fp64: t >= 46 (~1.4 * 2^-46 ~ 2e-14 normwise)
  else
    ozaki_plan_bits(k, 30, s, t);  // fp32: 1.4 * 2^-30 ~ 1e-9, far below fp32 rounding
}

template <class T>
size_t workspace_bytes(int64_t m, int64_t n, int64_t k) {
  int s, t;
  plan_for<T>(k, &s, &t);
  const int64_t kpad = (k + 15) / 16 * 16;
  return static_cast<size_t>(s) * (m * kpad + n * kpad + m * n) + sizeof(int) * (m + n) +
         sizeof(unsigned long long) * n + 1024;
}

// Workspace layout.  B's part (residues, column exponents and maxima) comes
// first and does not depend on m, so one prepared B serves row panels of any
// height: [bres s*n*kpad | colmax n | fx n | pad to 256] [ares s*m*kpad |
// cres s*m*n | pad 16 | ex m].  Every TMA base stays 16-byte aligned (kpad is
// a multiple of 16).
struct OzWs {
  int8_t* bres;
  unsigned long long* colmax;
  int* fx;
  int8_t* ares;
  uint8_t* cres;
  int* ex;
};

OzWs layout(void* ws, int64_t m, int64_t n, int64_t kpad, int s) {
  OzWs w;
  uintptr_t p = reinterpret_cast<uintptr_t>(ws);
  w.bres = reinterpret_cast<int8_t*>(p);
  p += s * n * kpad;
  p = (p + 15) & ~uintptr_t(15);
  w.colmax = reinterpret_cast<unsigned long long*>(p);
  p += sizeof(unsigned long long) * n;
  w.fx = reinterpret_cast<int*>(p);
  p += sizeof(int) * n;
  p = (p + 255) & ~uintptr_t(255);
  w.ares = reinterpret_cast<int8_t*>(p);
  p += s * m * kpad;
  w.cres = reinterpret_cast<uint8_t*>(p);
  p += s * m * n;
  p = (p + 15) & ~uintptr_t(15);
  w.ex = reinterpret_cast<int*>(p);
  return w;
}

// B's column exponents; the residue passes take moduli [l0, l1)
template <class T>
cudaError_t scale_b(cudaStream_t st, int64_t N, int64_t K, const T* B, int64_t ldb, const OzWs& w,
                    int t) {
  const int n = static_cast<int>(N), k = static_cast<int>(K);
  cudaError_t e = cudaMemsetAsync(w.colmax, 0, sizeof(unsigned long long) * N, st);
  if (e != cudaSuccess) return e;
  col_absmax_kernel<T><<<dim3(static_cast<unsigned>((N + 255) / 256),
                              static_cast<unsigned>((K + OZ_COL_ROWS - 1) / OZ_COL_ROWS)),
                         256, 0, st>>>(B, ldb, k, n, w.colmax);
  col_exponent_finalize<<<static_cast<unsigned>((N + 255) / 256), 256, 0, st>>>(w.colmax, n, t,
                                                                                 w.fx);
  return cudaSuccess;
}

template <class T>
void residues_b(cudaStream_t st, int64_t N, int64_t K, int64_t kpad, const T* B, int64_t ldb,
                const OzWs& w, int l0, int l1, const CrtConst& cc) {
  residue_bt_kernel<T><<<dim3(static_cast<unsigned>((N + 31) / 32),
                              static_cast<unsigned>((kpad + OZ_BT_K - 1) / OZ_BT_K)),
                         256, 0, st>>>(B, ldb, static_cast<int>(K), static_cast<int>(N),
                                       static_cast<int>(kpad), w.fx, w.bres, l0, l1, cc);
}

template <class T>
void residues_a(cudaStream_t st, int64_t M, int64_t K, int64_t kpad, const T* A, int64_t lda,
                const OzWs& w, int l0, int l1, const CrtConst& cc) {
  const unsigned rows_y = static_cast<unsigned>(std::min<int64_t>(M, 65535));
  residue_a_kernel<T><<<dim3(static_cast<unsigned>((kpad / 8 + 127) / 128), rows_y), 128, 0, st>>>(
      A, lda, static_cast<int>(M), static_cast<int>(K), static_cast<int>(kpad), w.ex, w.ares, l0,
      l1, cc);
}

cudaError_t igemm(const Launch& L, cudaStream_t st, int64_t M, int64_t N, int64_t kpad, int s,
                  const OzWs& w, int l0, int l1, const CrtConst& cc) {
  CUtensorMap ta, tb;
  if (!map3_u8(L, &ta, w.ares, kpad, M, s, IG_BM) || !map3_u8(L, &tb, w.bres, kpad, N, s, IG_BN))
    return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(igemm_mod_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       IG_SMEM);
  if (e != cudaSuccess) return e;
  const int tiles_m = static_cast<int>((M + IG_BM - 1) / IG_BM);
  const int tiles_n = static_cast<int>((N + IG_BN - 1) / IG_BN);
  const int grid = static_cast<int>(
      std::min<int64_t>(static_cast<int64_t>(tiles_m) * tiles_n * (l1 - l0), L.num_sms));
  igemm_mod_kernel<<<grid, IG_THREADS, IG_SMEM, st>>>(ta, tb, w.cres, static_cast<int>(M),
                                                      static_cast<int>(N), static_cast<int>(kpad),
                                                      tiles_m, tiles_n, l0, l1 - l0, cc);
  return cudaSuccess;
}

template <class T>
void crt(cudaStream_t st, int64_t M, int64_t N, const OzWs& w, T* C, int64_t ldc,
         const CrtConst& cc) {
  const unsigned rows_y = static_cast<unsigned>(std::min<int64_t>(M, 65535));
  const dim3 grid(static_cast<unsigned>((N / 4 + 1 + 127) / 128), rows_y);
  const int m = static_cast<int>(M), n = static_cast<int>(N);
  switch (cc.s) {
#define MMWS_CRT_CASE(S_)                                                        \
  case S_:                                                                       \
    crt_kernel<T, S_><<<grid, 128, 0, st>>>(w.cres, m, n, w.ex, w.fx, C, ldc, cc); \
    break;
    MMWS_CRT_CASE(8)
    MMWS_CRT_CASE(9)
    MMWS_CRT_CASE(10)
    MMWS_CRT_CASE(11)
    MMWS_CRT_CASE(12)
    MMWS_CRT_CASE(13)
    MMWS_CRT_CASE(14)
    MMWS_CRT_CASE(15)
#undef MMWS_CRT_CASE
    default:
      crt_kernel<T, OZ_MAX_MODULI><<<grid, 128, 0, st>>>(w.cres, m, n, w.ex, w.fx, C, ldc, cc);
  }
}

template <class T>
cudaError_t prepare_b(const Launch& L, int64_t N, int64_t K, const T* B, int64_t ldb, void* ws) {
  int s, t;
  plan_for<T>(K, &s, &t);
  CrtConst cc;
  make_crt(s, &cc);
  const int64_t kpad = (K + 15) / 16 * 16;
  const OzWs w = layout(ws, 0, N, kpad, s);
  cudaError_t e = scale_b<T>(L.stream, N, K, B, ldb, w, t);
  if (e != cudaSuccess) return e;
  residues_b<T>(L.stream, N, K, kpad, B, ldb, w, 0, s, cc);
  for (int i = 0; i < 3; ++i) L.count();
  return cudaGetLastError();
}

template <class T>
cudaError_t panel(const Launch& L, int64_t M, int64_t N, int64_t K, const T* A, int64_t lda, T* C,
                  int64_t ldc, void* ws) {
  int s, t;
  plan_for<T>(K, &s, &t);
  CrtConst cc;
  make_crt(s, &cc);
  const int64_t kpad = (K + 15) / 16 * 16;
  const OzWs w = layout(ws, M, N, kpad, s);
  cudaStream_t st = L.stream;
  row_exponent_kernel<T><<<static_cast<unsigned>((M * 32 + 255) / 256), 256, 0, st>>>(
      A, lda, static_cast<int>(M), static_cast<int>(K), t, w.ex);
  residues_a<T>(st, M, K, kpad, A, lda, w, 0, s, cc);
  cudaError_t e = igemm(L, st, M, N, kpad, s, w, 0, s, cc);
  if (e != cudaSuccess) return e;
  crt<T>(st, M, N, w, C, ldc, cc);
  for (int i = 0; i < 4; ++i) L.count();
  return cudaGetLastError();
}

template <class T>
cudaError_t launch_gemm_ozaki(const Launch& L, int64_t M, int64_t N, int64_t K, const T* A,
                              int64_t lda, const T* B, int64_t ldb, T* C, int64_t ldc, void* ws,
                              cudaStream_t aux, cudaEvent_t* ev) {
  // Large problems: B prepared once, then A's one panel (the GEMMs fill the SMs).
  // Below ~1.4e11 multiply-adds the residues and tensor-core GEMMs run in
  // moduli groups: the (FP64-ALU bound) residues of group g+1 on `st` while
  // the int8 GEMMs of group g run on `aux`, their blocks sharing the SMs.
  // Measured: N=4096 3.0 -> 2.0 ms with 4 groups; from N ~ 8192 up the extra
  // passes over A and B cost more than the overlap saves (N=16384: 64.5 vs
  // 66.9 ms).
  const double work = static_cast<double>(M) * N * K;
  int s, t;
  plan_for<T>(K, &s, &t);
  const int groups = work <= 1.4e11 ? std::min(s, OZ_GROUPS) : 1;
  if (groups == 1) {
    cudaError_t e = prepare_b<T>(L, N, K, B, ldb, ws);
    return e == cudaSuccess ? panel<T>(L, M, N, K, A, lda, C, ldc, ws) : e;
  }
  CrtConst cc;
  make_crt(s, &cc);
  const int64_t kpad = (K + 15) / 16 * 16;
  const OzWs w = layout(ws, M, N, kpad, s);
  cudaStream_t st = L.stream;
  cudaError_t e;
  row_exponent_kernel<T><<<static_cast<unsigned>((M * 32 + 255) / 256), 256, 0, st>>>(
      A, lda, static_cast<int>(M), static_cast<int>(K), t, w.ex);
  if ((e = scale_b<T>(st, N, K, B, ldb, w, t)) != cudaSuccess) return e;
  for (int g = 0; g < groups; ++g) {
    const int l0 = s * g / groups, l1 = s * (g + 1) / groups;
    residues_a<T>(st, M, K, kpad, A, lda, w, l0, l1, cc);
    residues_b<T>(st, N, K, kpad, B, ldb, w, l0, l1, cc);
    if ((e = cudaEventRecord(ev[g], st)) != cudaSuccess ||
        (e = cudaStreamWaitEvent(aux, ev[g], 0)) != cudaSuccess ||
        (e = igemm(L, aux, M, N, kpad, s, w, l0, l1, cc)) != cudaSuccess)
      return e;
  }
  // ---- reconstruction after the last GEMM
  if ((e = cudaEventRecord(ev[groups], aux)) != cudaSuccess ||
      (e = cudaStreamWaitEvent(st, ev[groups], 0)) != cudaSuccess)
    return e;
  crt<T>(st, M, N, w, C, ldc, cc);
  for (int i = 0; i < 4 + 3 * groups; ++i) L.count();
  return cudaGetLastError();
}

}  // namespace

size_t ozaki_workspace_bytes(int64_t m, int64_t n, int64_t k) {
  return workspace_bytes<double>(m, n, k);
}
size_t ozaki_workspace_bytes_f32(int64_t m, int64_t n, int64_t k) {
  return workspace_bytes<float>(m, n, k);
}

// fp32 through the same integer scheme: 30-bit scaling needs ~10 moduli at
// k = 32768
void ozaki_plan_f32(int64_t k, int* s, int* t) { ozaki_plan_bits(k, 30, s, t); }

cudaError_t launch_dgemm_ozaki(const Launch& L, int64_t M, int64_t N, int64_t K, const double* A,
                               int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                               void* ws, cudaStream_t aux, cudaEvent_t* ev) {
  return launch_gemm_ozaki<double>(L, M, N, K, A, lda, B, ldb, C, ldc, ws, aux, ev);
}

cudaError_t launch_sgemm_ozaki(const Launch& L, int64_t M, int64_t N, int64_t K, const float* A,
                               int64_t lda, const float* B, int64_t ldb, float* C, int64_t ldc,
                               void* ws, cudaStream_t aux, cudaEvent_t* ev) {
  return launch_gemm_ozaki<float>(L, M, N, K, A, lda, B, ldb, C, ldc, ws, aux, ev);
}

cudaError_t launch_ozaki_prepare_b(const Launch& L, int64_t N, int64_t K, const double* B,
                                   int64_t ldb, void* ws) {
  return prepare_b<double>(L, N, K, B, ldb, ws);
}
cudaError_t launch_ozaki_prepare_b(const Launch& L, int64_t N, int64_t K, const float* B,
                                   int64_t ldb, void* ws) {
  return prepare_b<float>(L, N, K, B, ldb, ws);
}
cudaError_t launch_ozaki_panel(const Launch& L, int64_t M, int64_t N, int64_t K, const double* A,
                               int64_t lda, double* C, int64_t ldc, void* ws) {
  return panel<double>(L, M, N, K, A, lda, C, ldc, ws);
}
cudaError_t launch_ozaki_panel(const Launch& L, int64_t M, int64_t N, int64_t K, const float* A,
                               int64_t lda, float* C, int64_t ldc, void* ws) {
  return panel<float>(L, M, N, K, A, lda, C, ldc, ws);
}

template <class T>
cudaError_t preload_crt() {
  return preload_kernels(crt_kernel<T, 8>, crt_kernel<T, 9>, crt_kernel<T, 10>, crt_kernel<T, 11>,
                         crt_kernel<T, 12>, crt_kernel<T, 13>, crt_kernel<T, 14>,
                         crt_kernel<T, 15>, crt_kernel<T, OZ_MAX_MODULI>);
}

cudaError_t preload_ozaki() {
  cudaError_t e = preload_kernels(row_exponent_kernel<double>, col_absmax_kernel<double>,
                                  col_exponent_finalize, residue_a_kernel<double>,
                                  residue_bt_kernel<double>, igemm_mod_kernel,
                                  row_exponent_kernel<float>, col_absmax_kernel<float>,
                                  residue_a_kernel<float>, residue_bt_kernel<float>);
  if (e == cudaSuccess) e = preload_crt<double>();
  if (e == cudaSuccess) e = preload_crt<float>();
  return e;
}

}  // namespace mmws_impl

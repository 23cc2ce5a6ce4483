/*
 * mmws_oracle.c -- CPU restatement of the reference's dense-matmul hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_1012_2273_b200/,
 * include/) links, loads or calls this file.  It is the checker that tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg compare the CUDA path
 * against.  It is pinned against the reference itself (oracle/_ref, built from
 * /root/reference/proj/include by oracle/Makefile) and against the golden
 * vectors in tests/golden/ (see tests/test_oracle.py).
 *
 * Build: gcc -O3 -ffp-contract=off -fno-fast-math (the reference builds with
 * -ffp-contract=off, proj/CMakeLists.txt:12-15, so a*b and +acc are two
 * separate roundings and every per-element chain is ascending in the inner
 * index from +0.0).
 *
 * Every function names the reference file:line it restates.  Paths are
 * relative to /root/reference/proj/.
 */
#define _GNU_SOURCE
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define ORACLE_OK 0
#define ORACLE_ERR_DIM 1
#define ORACLE_ERR_DOMAIN 2

/* ---------------------------------------------------------------------------
 * splitmix64 stream -- include/mmws/matrix.hpp:23-28 (splitmix64_next) and
 * :31-33 (to_unit_double).  random_matrix (matrix.hpp:101-107) seeds the state
 * with `seed` and advances once per element in row-major order, so element i
 * (0-based) of a matrix is mix(seed + (i + 1) * GOLDEN): counter-based, which
 * lets both this oracle and the device generator produce any element
 * independently.
 * ------------------------------------------------------------------------- */
static const uint64_t GOLDEN = 0x9E3779B97F4A7C15ULL;

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t oracle_splitmix64_draw(uint64_t seed, uint64_t index) {
  return mix64(seed + (index + 1) * GOLDEN);
}

/* Distributions (frozen here and in the device generator):
 *   0 UNIT       u = (bits >> 11) * 2^-53 in [0,1)      matrix.hpp:31-33
 *   1 UNIFORM    2u - 1 in [-1,1)  (exact: 2m-2^53 is an integer < 2^54)
 *   2 INT_PM8    ((bits >> 11) * 17 >> 53) - 8 in [-8,8], integer-valued
 *   3 NORMAL     fp32 Box-Muller from draws 2i, 2i+1 (host libm; see below)  */
static inline double draw_to_double(int dist, uint64_t bits) {
  const uint64_t m = bits >> 11;
  switch (dist) {
    case 0: return (double)m * 0x1.0p-53;
    case 1: return 2.0 * ((double)m * 0x1.0p-53) - 1.0;
    case 2: return (double)((int64_t)((m * 17ULL) >> 53) - 8);
    default: return 0.0;
  }
}

typedef struct {
  int dist;
  uint64_t seed, first, count;
  double* out_d;
  float* out_f;
} fill_job;

static void* fill_worker(void* p) {
  fill_job* j = (fill_job*)p;
  for (uint64_t e = 0; e < j->count; ++e) {
    const uint64_t i = j->first + e;
    if (j->dist == 3) {
      const double u1 = (double)(oracle_splitmix64_draw(j->seed, 2 * i) >> 11) * 0x1.0p-53;
      const double u2 = (double)(oracle_splitmix64_draw(j->seed, 2 * i + 1) >> 11) * 0x1.0p-53;
      const double z = sqrt(-2.0 * log(1.0 - u1)) * cos(6.283185307179586 * u2);
      j->out_f[e] = (float)z;
    } else {
      const double x = draw_to_double(j->dist, oracle_splitmix64_draw(j->seed, i));
      if (j->out_d) j->out_d[e] = x;
      else j->out_f[e] = (float)x;
    }
  }
  return NULL;
}

static int n_threads_for(uint64_t work, int want) {
  long hw = sysconf(_SC_NPROCESSORS_ONLN);
  int t = want > 0 ? want : (int)(hw > 0 ? hw : 1);
  if (t > 256) t = 256;
  if ((uint64_t)t > work / 65536 + 1) t = (int)(work / 65536 + 1);
  return t < 1 ? 1 : t;
}

/* Fill `count` elements starting at flat index `first` (row-major order).
 * Exactly one of out_d / out_f is non-NULL.  dist 3 requires out_f. */
int oracle_fill(int dist, uint64_t seed, uint64_t first, uint64_t count, double* out_d,
                float* out_f, int threads) {
  if (dist < 0 || dist > 3 || (!out_d && !out_f) || (dist == 3 && !out_f))
    return ORACLE_ERR_DOMAIN;
  const int t = n_threads_for(count, threads);
  pthread_t tid[256];
  fill_job jobs[256];
  uint64_t start = 0;
  for (int w = 0; w < t; ++w) {
    const uint64_t len = count / t + ((uint64_t)w < count % t ? 1 : 0);
    jobs[w] = (fill_job){dist, seed, first + start, len, out_d ? out_d + start : NULL,
                         out_f ? out_f + start : NULL};
    start += len;
  }
  for (int w = 1; w < t; ++w) pthread_create(&tid[w], NULL, fill_worker, &jobs[w]);
  fill_worker(&jobs[0]);
  for (int w = 1; w < t; ++w) pthread_join(tid[w], NULL);
  return ORACLE_OK;
}

/* ---------------------------------------------------------------------------
 * matmul_seq -- include/mmws/matrix.hpp:112-126.  For i, for k (output
 * column): acc = +0.0; for j ascending: acc += a(i,j) * b(j,k).  Row-major with
 * explicit leading dimensions (the reference's Matrix is ld == cols).
 * Dimension errors mirror matrix.hpp:113-116 (zero dims: matrix.hpp:72-78).
 * ------------------------------------------------------------------------- */
int oracle_matmul_seq(int64_t m, int64_t n, int64_t k, const double* a, int64_t lda,
                      const double* b, int64_t ldb, double* c, int64_t ldc) {
  if (m <= 0 || n <= 0 || k <= 0 || lda < k || ldb < n || ldc < n) return ORACLE_ERR_DIM;
  for (int64_t i = 0; i < m; ++i) {
    for (int64_t kk = 0; kk < n; ++kk) {
      double acc = 0.0;
      for (int64_t j = 0; j < k; ++j) acc += a[i * lda + j] * b[j * ldb + kk];
      c[i * ldc + kk] = acc;
    }
  }
  return ORACLE_OK;
}

/* worker_run's loop order -- include/mmws/protocol.hpp:132-141 (k outer, i
 * middle, j inner, acc from 0.0).  Per element identical to matmul_seq. */
int oracle_worker_block(int64_t rows, int64_t n, int64_t k, const double* a_slice,
                        const double* b, double* c_slice) {
  if (rows < 0 || n <= 0 || k <= 0) return ORACLE_ERR_DIM;
  for (int64_t kk = 0; kk < n; ++kk) {
    for (int64_t i = 0; i < rows; ++i) {
      double acc = 0.0;
      for (int64_t j = 0; j < k; ++j) acc += a_slice[i * k + j] * b[j * n + kk];
      c_slice[i * n + kk] = acc;
    }
  }
  return ORACLE_OK;
}

/* ---------------------------------------------------------------------------
 * Row-sampled oracle.  C(i, :) depends only on row i of A and all of B, so a
 * subset of rows is bitwise what matmul_seq would produce on those rows
 * (SURVEY.md s8(c) fact 2).  The loop is i / j / k with a row of
 * accumulators: element (i,k) still sees acc = +0.0, then acc += a(i,j)*b(j,k)
 * for j ascending with separate roundings -- the same chain as matrix.hpp:
 * 120-122 -- but B is streamed row by row instead of walked by column.
 * Threads split the output columns; each thread owns disjoint accumulators.
 * The *_f32w variant widens fp32 inputs to double first (the fp64 reference
 * for the fp32 config).
 * ------------------------------------------------------------------------- */
typedef struct {
  int64_t n_rows;
  const int64_t* rows;
  int64_t n, k, col0, col1;
  const double* a_d;
  const double* b_d;
  const float* a_f;
  const float* b_f;
  int64_t lda, ldb;
  double* out; /* n_rows x n, row-major */
} rows_job;

static void* rows_worker(void* p) {
  rows_job* J = (rows_job*)p;
  const int64_t w = J->col1 - J->col0;
  if (w <= 0) return NULL;
  double* acc = (double*)malloc((size_t)w * sizeof(double));
  for (int64_t r = 0; r < J->n_rows; ++r) {
    const int64_t i = J->rows[r];
    for (int64_t c = 0; c < w; ++c) acc[c] = 0.0;
    for (int64_t j = 0; j < J->k; ++j) {
      const double aij = J->a_d ? J->a_d[i * J->lda + j] : (double)J->a_f[i * J->lda + j];
      if (J->b_d) {
        const double* brow = J->b_d + j * J->ldb + J->col0;
        for (int64_t c = 0; c < w; ++c) {
          const double prod = aij * brow[c];
          acc[c] = acc[c] + prod;
        }
      } else {
        const float* brow = J->b_f + j * J->ldb + J->col0;
        for (int64_t c = 0; c < w; ++c) {
          const double prod = aij * (double)brow[c];
          acc[c] = acc[c] + prod;
        }
      }
    }
    memcpy(J->out + r * J->n + J->col0, acc, (size_t)w * sizeof(double));
  }
  free(acc);
  return NULL;
}

static int matmul_rows_impl(int64_t n_rows, const int64_t* rows, int64_t m, int64_t n,
                            int64_t k, const double* a_d, const float* a_f, int64_t lda,
                            const double* b_d, const float* b_f, int64_t ldb, double* out,
                            int threads) {
  if (m <= 0 || n <= 0 || k <= 0 || lda < k || ldb < n || n_rows < 0) return ORACLE_ERR_DIM;
  for (int64_t r = 0; r < n_rows; ++r)
    if (rows[r] < 0 || rows[r] >= m) return ORACLE_ERR_DIM;
  long hw = sysconf(_SC_NPROCESSORS_ONLN);
  int t = threads > 0 ? threads : (int)(hw > 0 ? hw : 1);
  if (t > 256) t = 256;
  if (t > n / 64 + 1) t = (int)(n / 64 + 1);
  pthread_t tid[256];
  rows_job jobs[256];
  int64_t start = 0;
  for (int w = 0; w < t; ++w) {
    const int64_t len = n / t + (w < n % t ? 1 : 0);
    jobs[w] = (rows_job){n_rows, rows, n, k, start, start + len, a_d, b_d, a_f, b_f, lda, ldb, out};
    start += len;
  }
  for (int w = 1; w < t; ++w) pthread_create(&tid[w], NULL, rows_worker, &jobs[w]);
  rows_worker(&jobs[0]);
  for (int w = 1; w < t; ++w) pthread_join(tid[w], NULL);
  return ORACLE_OK;
}

int oracle_matmul_rows(int64_t n_rows, const int64_t* rows, int64_t m, int64_t n, int64_t k,
                       const double* a, int64_t lda, const double* b, int64_t ldb, double* out,
                       int threads) {
  return matmul_rows_impl(n_rows, rows, m, n, k, a, NULL, lda, b, NULL, ldb, out, threads);
}

int oracle_matmul_rows_f32w(int64_t n_rows, const int64_t* rows, int64_t m, int64_t n,
                            int64_t k, const float* a, int64_t lda, const float* b, int64_t ldb,
                            double* out, int threads) {
  return matmul_rows_impl(n_rows, rows, m, n, k, NULL, a, lda, NULL, b, ldb, out, threads);
}

/* ---------------------------------------------------------------------------
 * Partitions.
 * static_partition -- include/mmws/workshare.hpp:33-46: the first
 *   (iterations % workers) workers get one extra iteration; workers == 0 is a
 *   DomainError.
 * split_rows -- include/mmws/protocol.hpp:33-46: averow = n/W, extra = n%W,
 *   first `extra` workers get +1, offsets accumulate; W < 1 or n < 0 is a
 *   DomainError.
 * op_count -- include/mmws/matrix.hpp:130-134: N^2 (2N - 1), N < 1 DomainError.
 * ------------------------------------------------------------------------- */
int oracle_static_partition(uint64_t iterations, uint32_t workers, uint64_t* start,
                            uint64_t* len) {
  if (workers == 0) return ORACLE_ERR_DOMAIN;
  const uint64_t base = iterations / workers, extra = iterations % workers;
  uint64_t s = 0;
  for (uint32_t w = 0; w < workers; ++w) {
    start[w] = s;
    len[w] = base + (w < extra ? 1 : 0);
    s += len[w];
  }
  return ORACLE_OK;
}

int oracle_split_rows(int64_t n_rows, int32_t n_workers, int64_t* offset, int64_t* rows) {
  if (n_workers < 1 || n_rows < 0) return ORACLE_ERR_DOMAIN;
  const int64_t averow = n_rows / n_workers, extra = n_rows % n_workers;
  int64_t off = 0;
  for (int32_t w = 0; w < n_workers; ++w) {
    offset[w] = off;
    rows[w] = averow + (w < extra ? 1 : 0);
    off += rows[w];
  }
  return ORACLE_OK;
}

int oracle_op_count(int64_t n, uint64_t* out) {
  if (n < 1) return ORACLE_ERR_DOMAIN;
  const uint64_t un = (uint64_t)n;
  *out = un * un * (2 * un - 1);
  return ORACLE_OK;
}

/* matmul_threads -- include/mmws/workshare.hpp:98-113: rows split by
 * static_partition, each worker runs matmul_seq's per-element loop on its
 * rows.  Bitwise equal to oracle_matmul_seq. */
typedef struct {
  int64_t r0, r1, n, k;
  const double* a;
  const double* b;
  double* c;
} thr_job;

static void* thr_worker(void* p) {
  thr_job* J = (thr_job*)p;
  for (int64_t i = J->r0; i < J->r1; ++i)
    for (int64_t kk = 0; kk < J->n; ++kk) {
      double acc = 0.0;
      for (int64_t j = 0; j < J->k; ++j) acc += J->a[i * J->k + j] * J->b[j * J->n + kk];
      J->c[i * J->n + kk] = acc;
    }
  return NULL;
}

int oracle_matmul_threads(int64_t m, int64_t n, int64_t k, const double* a, const double* b,
                          double* c, uint32_t workers) {
  if (m <= 0 || n <= 0 || k <= 0) return ORACLE_ERR_DIM;
  if (workers == 0) return ORACLE_ERR_DOMAIN;
  if (workers > 256) workers = 256;
  uint64_t st[256], ln[256];
  oracle_static_partition((uint64_t)m, workers, st, ln);
  pthread_t tid[256];
  thr_job jobs[256];
  for (uint32_t w = 0; w < workers; ++w)
    jobs[w] = (thr_job){(int64_t)st[w], (int64_t)(st[w] + ln[w]), n, k, a, b, c};
  for (uint32_t w = 1; w < workers; ++w)
    if (ln[w]) pthread_create(&tid[w], NULL, thr_worker, &jobs[w]);
  thr_worker(&jobs[0]);
  for (uint32_t w = 1; w < workers; ++w)
    if (ln[w]) pthread_join(tid[w], NULL);
  return ORACLE_OK;
}

/* bitwise_equal / first_difference -- include/mmws/matrix.hpp:136-157:
 * memcmp per element, so -0.0 != +0.0 and NaN payloads must match.
 * Returns -1 when equal, else the first differing flat index. */
int64_t oracle_first_difference(const double* x, const double* y, int64_t count) {
  for (int64_t i = 0; i < count; ++i)
    if (memcmp(&x[i], &y[i], sizeof(double)) != 0) return i;
  return -1;
}

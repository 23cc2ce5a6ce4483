// ref_shim.cpp -- C entry points over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against
// /root/reference/proj/include (by include path; no reference source is copied
// into this repo) into oracle/_ref/libmmws_ref.so.  Used to pin the C oracle
// (tests/test_oracle.py), to generate the golden fixtures
// (tests/golden/gen_golden.py), and as bench.py's CPU baseline / reference arm
// (the reference's own matmul_seq / matmul_threads code path, timed with the
// reference's time_model bracket semantics, include/mmws/bench.hpp:92-129).
//
// Status codes: 0 ok, 1 DimensionError, 2 DomainError, 9 any other exception.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "mmws/error.hpp"
#include "mmws/matrix.hpp"
#include "mmws/workshare.hpp"
#ifdef MMWS_REF_WITH_PROTOCOL
#include "mmws/bench.hpp"
#include "mmws/protocol.hpp"
#endif

namespace {

int status_of(const std::exception_ptr& e) {
  try {
    std::rethrow_exception(e);
  } catch (const mmws::DimensionError&) {
    return 1;
  } catch (const mmws::DomainError&) {
    return 2;
  } catch (...) {
    return 9;
  }
}

mmws::Matrix wrap(std::int64_t rows, std::int64_t cols, const double* data) {
  std::vector<double> v(data, data + rows * cols);
  return mmws::Matrix(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols),
                      std::move(v));
}

void unwrap(const mmws::Matrix& m, double* out) {
  const auto d = m.data();
  std::memcpy(out, d.data(), d.size() * sizeof(double));
}

// wall_time semantics: steady_clock seconds (include/mmws/net.hpp:88-90).
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

}  // namespace

extern "C" {

int ref_random_matrix(std::int64_t rows, std::int64_t cols, std::uint64_t seed, double* out) {
  try {
    unwrap(mmws::random_matrix(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols),
                               seed),
           out);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int ref_identity(std::int64_t n, double* out) {
  try {
    unwrap(mmws::identity(static_cast<std::size_t>(n)), out);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// C (m x n) = A (m x k) . B (kb x n); kb != k exercises the DimensionError path.
int ref_matmul_seq(std::int64_t m, std::int64_t k, std::int64_t kb, std::int64_t n,
                   const double* a, const double* b, double* c) {
  try {
    const mmws::Matrix A = wrap(m, k, a), B = wrap(kb, n, b);
    unwrap(mmws::matmul_seq(A, B), c);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int ref_matmul_threads(std::int64_t m, std::int64_t k, std::int64_t kb, std::int64_t n,
                       const double* a, const double* b, double* c, unsigned workers) {
  try {
    const mmws::Matrix A = wrap(m, k, a), B = wrap(kb, n, b);
    unwrap(mmws::matmul_threads(A, B, workers), c);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

// time_model bracket (bench.hpp:99-111): clock around the call only, min of
// `repeats`.  Inputs are wrapped into mmws::Matrix outside the bracket.
// workers == 0 selects matmul_seq, otherwise matmul_threads(workers).
int ref_time_matmul(std::int64_t m, std::int64_t k, std::int64_t n, const double* a,
                    const double* b, unsigned workers, int repeats, double* best_s,
                    double* c_out) {
  try {
    const mmws::Matrix A = wrap(m, k, a), B = wrap(k, n, b);
    double best = 0.0;
    for (int r = 0; r < repeats; ++r) {
      const double t0 = now_s();
      mmws::Matrix C = workers == 0 ? mmws::matmul_seq(A, B) : mmws::matmul_threads(A, B, workers);
      const double el = now_s() - t0;
      if (r == 0 || el < best) best = el;
      if (c_out && r == repeats - 1) unwrap(C, c_out);
    }
    *best_s = best;
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int ref_static_partition(std::uint64_t iterations, unsigned workers, std::uint64_t* start,
                         std::uint64_t* len) {
  try {
    const auto p = mmws::static_partition(iterations, workers);
    for (std::size_t w = 0; w < p.assignments.size(); ++w) {
      start[w] = p.assignments[w].start;
      len[w] = p.assignments[w].len;
    }
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int ref_op_count(std::int64_t n, std::uint64_t* out) {
  try {
    *out = mmws::op_count(n);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
}

int ref_has_protocol(void) {
#ifdef MMWS_REF_WITH_PROTOCOL
  return 1;
#else
  return 0;
#endif
}

int ref_split_rows(std::int64_t n_rows, int n_workers, std::int64_t* offset,
                   std::int64_t* rows) {
#ifdef MMWS_REF_WITH_PROTOCOL
  try {
    const auto s = mmws::split_rows(n_rows, n_workers);
    for (std::size_t w = 0; w < s.size(); ++w) {
      offset[w] = s[w].offset;
      rows[w] = s[w].rows;
    }
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
#else
  (void)n_rows; (void)n_workers; (void)offset; (void)rows;
  return 9;
#endif
}

// bench.hpp:83-86 (derive_seed) and :70-78 (mflops); 9 when the harness
// header could not be built.
int ref_derive_seed(std::uint64_t seed, std::int64_t n, int which, std::uint64_t* out) {
#ifdef MMWS_REF_WITH_PROTOCOL
  *out = mmws::detail::derive_seed(seed, n, which);
  return 0;
#else
  (void)seed; (void)n; (void)which; (void)out;
  return 9;
#endif
}

int ref_mflops(std::int64_t n, double elapsed, double* out) {
#ifdef MMWS_REF_WITH_PROTOCOL
  try {
    *out = mmws::mflops(n, elapsed);
    return 0;
  } catch (...) {
    return status_of(std::current_exception());
  }
#else
  (void)n; (void)elapsed; (void)out;
  return 9;
#endif
}

}  // extern "C"

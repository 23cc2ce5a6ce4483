// C++ drop-in adapter test (include/mmws_gpu.hpp over libmmws_gpu.so).
// Mirrors the reference's own Catch2 cases where they apply to the hot path
// (test_matrix.cpp, test_workshare.cpp, test_protocol.cpp).  Usage:
//   test_adapter cpu   -- host-only checks (no GPU needed)
//   test_adapter gpu   -- multiply checks on device 0
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "mmws_gpu.hpp"

using mmws::gpu::MatrixF32;
using mmws::gpu::MatrixF64;
namespace G = mmws::gpu;

static int g_fail = 0;
#define CHECK(cond)                                                      \
  do {                                                                   \
    if (!(cond)) {                                                       \
      std::fprintf(stderr, "CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++g_fail;                                                          \
    }                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, type)                                      \
  do {                                                                   \
    bool thrown_ = false;                                                \
    try { (void)(expr); } catch (const type&) { thrown_ = true; } catch (...) {} \
    if (!thrown_) {                                                      \
      std::fprintf(stderr, "CHECK_THROWS_AS failed %s:%d: %s\n", __FILE__, __LINE__, #expr); \
      ++g_fail;                                                          \
    }                                                                    \
  } while (0)

// test-local splitmix64 uniform [0,1) fill, the reference's random_matrix stream
static MatrixF64 random_matrix(std::size_t r, std::size_t c, std::uint64_t seed) {
  std::vector<double> v(r * c);
  std::uint64_t s = seed;
  for (double& x : v) {
    std::uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    z ^= z >> 31;
    x = static_cast<double>(z >> 11) * 0x1.0p-53;
  }
  return MatrixF64(r, c, std::move(v));
}

// test-local sequential product in the reference's order (ascending j from +0.0)
static MatrixF64 seq(const MatrixF64& a, const MatrixF64& b) {
  MatrixF64 c(a.rows(), b.cols());
  for (std::size_t i = 0; i < a.rows(); ++i)
    for (std::size_t k = 0; k < b.cols(); ++k) {
      volatile double acc = 0.0;
      for (std::size_t j = 0; j < a.cols(); ++j) {
        volatile double p = a(i, j) * b(j, k);
        acc = acc + p;
      }
      c(i, k) = acc;
    }
  return c;
}

static bool bitwise_equal(const MatrixF64& x, const MatrixF64& y) {
  return x.rows() == y.rows() && x.cols() == y.cols() &&
         std::memcmp(x.data().data(), y.data().data(), x.size() * sizeof(double)) == 0;
}

// In-process two-rank control plane with the reference Communicator's
// send_i64/recv_i64 surface (comm.hpp:49-77), for share_unique_id.
struct FakeComm {
  int rank, world;
  std::vector<std::int64_t>* wire;  // rank 0 -> rank 1, FIFO
  std::size_t* cursor;
  int my_rank() const { return rank; }
  int world_size() const { return world; }
  void send_i64(int, std::uint32_t, std::int64_t v) { wire->push_back(v); }
  std::int64_t recv_i64(int, std::uint32_t) { return (*wire)[(*cursor)++]; }
};

static void cpu_checks() {
  CHECK((G::split_rows(4, 3) == std::vector<G::WorkAssignment>{{0, 2}, {2, 1}, {3, 1}}));
  CHECK((G::split_rows(6, 3) == std::vector<G::WorkAssignment>{{0, 2}, {2, 2}, {4, 2}}));
  CHECK((G::split_rows(2, 3) == std::vector<G::WorkAssignment>{{0, 1}, {1, 1}, {2, 0}}));
  CHECK_THROWS_AS(G::split_rows(4, 0), mmws::DomainError);
  CHECK_THROWS_AS(G::split_rows(-1, 2), mmws::DomainError);
  CHECK((G::static_partition(10, 3) == std::vector<G::Range>{{0, 4}, {4, 3}, {7, 3}}));
  CHECK_THROWS_AS(G::static_partition(3, 0), mmws::DomainError);
  CHECK(G::op_count(1) == 1);
  CHECK(G::op_count(100) == 1'990'000);
  CHECK(G::op_count(1000) == 1'999'000'000);
  CHECK_THROWS_AS(G::op_count(0), mmws::DomainError);
  CHECK_THROWS_AS(MatrixF64(0, 3), mmws::DimensionError);
  CHECK_THROWS_AS(MatrixF64(2, 2, {1, 2, 3}), mmws::DimensionError);
  // no CPU fallback: without an sm_100 device the context cannot be created
  CHECK_THROWS_AS(G::Context(0), G::GpuError);
  // the 128-byte NCCL id travels as 16 int64 scalars over the control plane
  std::vector<std::int64_t> wire;
  std::size_t cursor = 0;
  FakeComm root{0, 2, &wire, &cursor}, worker{1, 2, &wire, &cursor};
  const auto id0 = G::share_unique_id(root);
  const auto id1 = G::share_unique_id(worker);
  CHECK(wire.size() == 16 && id0.size() == 128 && id0 == id1);
  // status codes map to the reference's exception types (error.hpp)
  CHECK_THROWS_AS(G::check(MMWS_GPU_ERR_TIMEOUT), mmws::TimeoutError);
  CHECK_THROWS_AS(G::check(MMWS_GPU_ERR_PROTOCOL), mmws::ProtocolError);
  CHECK_THROWS_AS(G::check(MMWS_GPU_ERR_RANK), mmws::RankError);
  CHECK_THROWS_AS(G::check(MMWS_GPU_ERR_NCCL), G::GpuError);
  // the drop-in's master_run defaults to the reference's bitwise contract
  CHECK(G::contract_mode<MatrixF64>() == G::Mode::exact);
  CHECK(G::contract_mode<MatrixF32>() == G::Mode::ffma);
}

static void gpu_checks() {
  G::Context ctx(0);
  // test_matrix.cpp:105-120
  const MatrixF64 a2(2, 2, {1, 2, 3, 4}), b2(2, 2, {5, 6, 7, 8});
  for (G::Mode m : {G::Mode::exact, G::Mode::dmma, G::Mode::automatic}) {
    const MatrixF64 c = G::matmul(ctx, a2, b2, m);
    CHECK(c(0, 0) == 19.0 && c(0, 1) == 22.0 && c(1, 0) == 43.0 && c(1, 1) == 50.0);
  }
  CHECK(G::matmul_seq(ctx, MatrixF64(1, 1, {3.25}), MatrixF64(1, 1, {-2.0}))(0, 0) == 3.25 * -2.0);
  // bitwise contract of matmul_seq / matmul_threads (test_workshare.cpp:140-172)
  for (auto [m, k, n] : {std::tuple{5, 5, 5}, {50, 50, 50}, {3, 3, 3}, {4, 7, 3}, {130, 257, 65}}) {
    const MatrixF64 a = random_matrix(m, k, 21 + m), b = random_matrix(k, n, 22 + n);
    const MatrixF64 want = seq(a, b);
    CHECK(bitwise_equal(G::matmul_seq(ctx, a, b), want));
    for (unsigned w : {1u, 2u, 8u}) CHECK(bitwise_equal(G::matmul_threads(ctx, a, b, w), want));
    const MatrixF64 d = G::matmul(ctx, a, b);
    double num = 0, den = 0;
    for (std::size_t i = 0; i < d.size(); ++i) {
      num += (d.data()[i] - want.data()[i]) * (d.data()[i] - want.data()[i]);
      den += want.data()[i] * want.data()[i];
    }
    CHECK(std::sqrt(num / den) <= 1e-12);
  }
  const MatrixF64 r23 = random_matrix(2, 3, 29), r22 = random_matrix(2, 2, 30);
  CHECK_THROWS_AS(G::matmul_threads(ctx, r23, r22, 2), mmws::DimensionError);
  CHECK_THROWS_AS(G::matmul_threads(ctx, r22, r22, 0), mmws::DomainError);
  CHECK_THROWS_AS(G::matmul_seq(ctx, r23, r22), mmws::DimensionError);
  // master_run in a one-rank world (rank 0 is master and worker); the
  // default mode keeps the reference's bitwise contract
  const MatrixF64 a = random_matrix(33, 33, 3033), b = random_matrix(33, 33, 4033);
  auto [c, elapsed] = G::master_run(ctx, a, b, G::Mode::exact);
  CHECK(bitwise_equal(c, seq(a, b)));
  CHECK(elapsed > 0.0);
  auto [c_default, el2] = G::master_run(ctx, random_matrix(130, 257, 5), random_matrix(257, 65, 6));
  CHECK(bitwise_equal(c_default, seq(random_matrix(130, 257, 5), random_matrix(257, 65, 6))));
  CHECK(el2 > 0.0);
  CHECK_THROWS_AS(G::worker_run(ctx, 4, 4, 4), mmws::RankError);
  // fp32 configuration type
  MatrixF32 af(3, 2, {1, 2, 3, 4, 5, 6}), bf(2, 2, {1, 0, 0, 1});
  const MatrixF32 cf = G::matmul(ctx, af, bf);
  CHECK(cf(2, 0) == 5.f && cf(2, 1) == 6.f);
  CHECK(ctx.launches() > 0);
  // the same calls served by the resident latency server: same bits
  ctx.server_start();
  for (auto [m, k, n] : {std::tuple{5, 5, 5}, {50, 50, 50}, {96, 96, 96}, {4, 7, 3}}) {
    const MatrixF64 a = random_matrix(m, k, 21 + m), b = random_matrix(k, n, 22 + n);
    CHECK(bitwise_equal(G::matmul_seq(ctx, a, b), seq(a, b)));
    CHECK(bitwise_equal(G::matmul_threads(ctx, a, b, 4), seq(a, b)));
  }
  ctx.server_stop();
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  try {
    if (mode == "gpu") gpu_checks();
    else cpu_checks();
  } catch (const std::exception& e) {
    std::fprintf(stderr, "uncaught: %s\n", e.what());
    return 2;
  }
  std::printf("%s: %s\n", mode.c_str(), g_fail ? "FAILED" : "ok");
  return g_fail ? 1 : 0;
}

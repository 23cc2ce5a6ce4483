// Host-side pieces of include/mmws_gpu_bench.hpp, printed as JSON for
// tests/test_harness.py to compare with the reference's own values
// (tests/golden/ref_small.json): derive_seed (bench.hpp:83-86), mflops
// (bench.hpp:70-73), random_matrix's first draws, and the CSV format.
#include <cinttypes>
#include <cstdio>
#include <string>
#include <vector>

#include "mmws_gpu_bench.hpp"

namespace G = mmws::gpu;

int main(int argc, char** argv) {
  if (argc > 1) {  // emit_plots on fixed records (plots.hpp:145-198 analogue)
    std::vector<G::BenchRecord> recs = {
        {"gpu", 500, 1, 0.002, 1.0e5, 30.0, 0.0},
        {"gpu", 100, 1, 0.0001, 2.0e4, 4.0, 0.0},
        {"gpu-exact", 100, 1, 0.0002, 1.0e4, std::nullopt, 0.0},
        {"gpu-rowblock", 4096, 4, 0.01, 1.3e7, std::nullopt, 0.0},
        {"gpu-rowblock", 2048, 4, 0.003, 5.7e6, std::nullopt, 0.0}};
    G::CostFit fit;
    fit.link_bytes_per_s = 500e9;
    fit.gemm_flops_per_s = 3.0e13;
    G::emit_plots(recs, argv[1], fit);
    bool threw = false;
    try {
      G::emit_plots({}, argv[1]);
    } catch (const mmws::DomainError&) {
      threw = true;
    }
    // a regular file where the directory should be: IoError (test_plots.cpp:204-212)
    const std::string blocker = std::string(argv[1]) + "/blocker";
    { std::FILE* f = std::fopen(blocker.c_str(), "w"); if (f) std::fclose(f); }
    bool io_threw = false;
    try {
      G::emit_plots(recs, blocker + "/sub");
    } catch (const mmws::IoError&) {
      io_threw = true;
    }
    std::remove(blocker.c_str());
    std::printf("{\"empty_throws\": %s, \"io_error\": %s}\n", threw ? "true" : "false",
                io_threw ? "true" : "false");
    return 0;
  }
  std::printf("{\"derive_seed\": {");
  bool first = true;
  for (std::uint64_t s : {0ULL, 42ULL, (1ULL << 63) + 5})
    for (std::int64_t n : {1, 100, 1000, 16384})
      for (int w : {0, 1}) {
        std::printf("%s\"%" PRIu64 ",%lld,%d\": %" PRIu64, first ? "" : ", ", s,
                    static_cast<long long>(n), w, G::bench_detail::derive_seed(s, n, w));
        first = false;
      }
  std::printf("}, \"mflops\": {");
  first = true;
  for (std::int64_t n : {100, 500, 1000, 2000})
    for (double t : {0.03, 2.09, 22.52, 240.97}) {
      std::printf("%s\"%lld,%s\": %.17g", first ? "" : ", ", static_cast<long long>(n),
                  G::bench_detail::format_g6(t).c_str(), G::mflops(n, t));
      first = false;
    }
  const G::MatrixF64 r = G::bench_detail::random_matrix(1, 1, 0);
  std::printf("}, \"random0\": %.17g", r(0, 0));
  G::BenchRecord a{"gpu", 1000, 1, 0.000123456789, 16191.2345, std::nullopt, 0.0};
  G::BenchRecord b{"gpu-exact", 1000, 1, 0.5, 3998.0, 2.5, 0.0};
  std::string csv = G::csv({a, b});
  for (auto& ch : csv)
    if (ch == '\n') ch = '|';
  std::printf(", \"csv\": \"%s\"", csv.c_str());
  bool threw = false;
  try {
    G::mflops(10, 0.0);
  } catch (const mmws::DomainError&) {
    threw = true;
  }
  std::printf(", \"mflops_zero_throws\": %s}\n", threw ? "true" : "false");
  return 0;
}

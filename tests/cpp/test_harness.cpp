// Host-side pieces of include/mmws_gpu_bench.hpp, printed as JSON for
// tests/test_harness.py to compare with the reference's own values
// (tests/golden/ref_small.json): derive_seed (bench.hpp:83-86), mflops
// (bench.hpp:70-73), random_matrix's first draws, and the CSV format.
#include <cinttypes>
#include <cstdio>
#include <string>

#include "mmws_gpu_bench.hpp"

namespace G = mmws::gpu;

int main() {
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

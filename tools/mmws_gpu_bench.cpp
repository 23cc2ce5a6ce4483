// mmws_gpu_bench -- the reference's `bench` CLI (tools/bench_main.cpp) for the
// GPU models: sweeps N, gates every product, prints the table and writes the
// reference's CSV format.
//
//   mmws_gpu_bench --dims 100,500,1000 [--models gpu,gpu-exact] [--repeats 3]
//                  [--seed 42] [--csv out.csv] [--tolerance 1e-12] [--server]
//                  [--plots DIR] [--calibrate]
//
// Build: g++ -std=c++20 -O2 -Iinclude tools/mmws_gpu_bench.cpp
//            -Lpaper_1012_2273_b200 -lmmws_gpu -Wl,-rpath,<repo>/paper_1012_2273_b200
// (add -I<reference>/proj/include to gate small N against mmws::matmul_seq).
#include <cstdio>
#include <cstdlib>
#include <sstream>
#include <string>
#include <vector>

#include "mmws_gpu_bench.hpp"

namespace {

std::vector<std::string> split(const std::string& s) {
  std::vector<std::string> out;
  std::stringstream ss(s);
  std::string item;
  while (std::getline(ss, item, ','))
    if (!item.empty()) out.push_back(item);
  return out;
}

int usage() {
  std::fprintf(stderr,
               "usage: mmws_gpu_bench --dims N1,N2,... [--models gpu,gpu-exact,gpu-rowblock] "
               "[--repeats R] [--seed S] [--tolerance T] [--csv PATH] [--device D] [--server] [--plots DIR] [--calibrate]\n");
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  mmws::gpu::BenchConfig config;
  std::string csv_path, plots_dir;
  bool calibrate = false;  // bench_main.cpp:64-93 analogue: fit the row-block cost model
  int device = 0;
  bool server = false;  // resident latency server for N <= 96 (mmws_gpu_server_start)
  try {
    for (int i = 1; i < argc; ++i) {
      const std::string arg = argv[i];
      auto value = [&]() -> std::string {
        if (i + 1 >= argc) throw mmws::DomainError("missing value for " + arg);
        return argv[++i];
      };
      if (arg == "--dims") {
        for (const auto& d : split(value())) config.dims.push_back(std::stoll(d));
      } else if (arg == "--models") {
        config.models.clear();
        for (const auto& m : split(value())) config.models.push_back(mmws::gpu::model_from_name(m));
      } else if (arg == "--repeats") {
        config.repeats = std::stoi(value());
      } else if (arg == "--seed") {
        config.seed = std::stoull(value());
      } else if (arg == "--tolerance") {
        config.tolerance = std::stod(value());
      } else if (arg == "--csv") {
        csv_path = value();
      } else if (arg == "--device") {
        device = std::stoi(value());
      } else if (arg == "--plots") {
        plots_dir = value();
      } else if (arg == "--calibrate") {
        calibrate = true;
      } else if (arg == "--server") {
        server = true;
      } else {
        return usage();
      }
    }
    if (config.dims.empty()) return usage();
    mmws::gpu::Context ctx(device);
    if (server) ctx.server_start();
    const auto records = mmws::gpu::run_suite(ctx, config);
    std::printf("%-13s %8s %8s %14s %14s %12s\n", "model", "n", "gpus", "elapsed_s", "mflops",
                "rel_err");
    for (const auto& r : records)
      std::printf("%-13s %8lld %8d %14.6g %14.6g %12.3g\n", r.model.c_str(),
                  static_cast<long long>(r.n), r.workers, r.elapsed, r.mflops, r.rel_err);
    if (!csv_path.empty()) mmws::gpu::emit_csv(records, csv_path);
    std::optional<mmws::gpu::CostFit> fit;
    if (calibrate) {
      fit = mmws::gpu::calibrate(ctx);
      std::printf("calibration: link %.6g B/s (%s), gemm %.6g FLOP/s\n", fit->link_bytes_per_s,
                  fit->link_measured ? "measured" : "nominal NVLink 5", fit->gemm_flops_per_s);
    }
    if (!plots_dir.empty()) mmws::gpu::emit_plots(records, plots_dir, fit);
  } catch (const mmws::gpu::GateError& e) {
    std::fprintf(stderr, "mmws_gpu_bench: %s\n", e.what());
    return 2;  // bench_main.cpp:175-177
  } catch (const std::exception& e) {
    std::fprintf(stderr, "mmws_gpu_bench: %s\n", e.what());
    return 1;
  }
  return 0;
}

// mmws_gpu_bench -- the reference's `bench` CLI (tools/bench_main.cpp) for the
// GPU models: sweeps N, gates every product, prints the table and writes the
// reference's CSV format.
//
//   mmws_gpu_bench --dims 100,500,1000 [--models gpu,gpu-exact] [--repeats 3]
//                  [--seed 42] [--csv out.csv] [--tolerance 1e-12] [--server]
//                  [--plots DIR] [--calibrate] [--gpus P]
//                  [--cpu-models seq,threads] [--cpu-repeats R]
//
// --cpu-models (needs the reference headers): the reference's own run_suite
// (bench.hpp:133-188) times its seq / threads models on this host first, with
// its own gate; their records join the CSV / table / plots and the seq times
// give every GPU record its speedup column -- the paper's comparison in one
// run.
//
// --gpus P (gpu-rowblock over P GPUs of this node, one process per GPU): rank
// 0 spawns ranks 1..P-1 -- this binary in worker mode -- with the reference's
// own launcher (launch_with_master / connect_from_env, launch.hpp), ships the
// NCCL id over its TCP Communicator (mmws::gpu::comm_init_from), and every
// rank then takes part in each gpu-rowblock round (worker_run on ranks >= 1,
// replaying the master's sweep from the same arguments).  Needs the
// reference headers at build time.
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

#if __has_include(<mmws/launch.hpp>) && __has_include(<json.hpp>)
#include <mmws/launch.hpp>
#define MMWS_GPU_BENCH_HAVE_LAUNCHER 1
#endif
#if __has_include(<mmws/bench.hpp>) && __has_include(<json.hpp>)
#include <mmws/bench.hpp>
#define MMWS_GPU_BENCH_HAVE_REF_SUITE 1
#endif

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
               "[--repeats R] [--seed S] [--tolerance T] [--csv PATH] [--device D] [--server] [--plots DIR] [--calibrate] [--gpus P] "
               "[--cpu-models seq,threads] [--cpu-repeats R]\n");
  return 2;
}

}  // namespace

#ifdef MMWS_GPU_BENCH_HAVE_LAUNCHER
// Rank >= 1 of a --gpus run: the same rounds as the master's gpu-rowblock
// records (run_suite order: per N, `repeats` timed rounds), as worker_run.
int run_worker(const mmws::gpu::BenchConfig& config, bool calibrate) {
  mmws::Communicator comm = mmws::connect_from_env();
  // one process per GPU; MMWS_BENCH_ONE_GPU_WORLD=1 (tests: every rank on GPU
  // 0 with the loopback NCCL stand-in, MMWS_GPU_NCCL_LIB) keeps them on one
  mmws::gpu::Context ctx(std::getenv("MMWS_BENCH_ONE_GPU_WORLD") ? 0 : comm.my_rank());
  mmws::gpu::comm_init_from(ctx, comm);
  bool rowblock = false;
  for (auto m : config.models) rowblock = rowblock || m == mmws::gpu::GpuModel::gpu_rowblock;
  if (rowblock)
    for (const std::int64_t n : config.dims)
      for (int r = 0; r < config.repeats; ++r)
        mmws::gpu::worker_run(ctx, n, n, n, mmws::gpu::Mode::automatic);  // the master's mode (time_model)
  if (calibrate) mmws::gpu::calibrate(ctx);  // its link probe is collective
  return 0;
}
#endif

int main(int argc, char** argv) {
  mmws::gpu::BenchConfig config;
  std::string csv_path, plots_dir;
  bool calibrate = false;  // bench_main.cpp:64-93 analogue: fit the row-block cost model
  int device = 0;
  bool server = false;  // resident latency server for N <= 96 (mmws_gpu_server_start)
  int gpus = 0;  // 0: no --gpus, plain single-context run
  bool worker = false;
  std::vector<std::string> cpu_models;  // the reference's own seq / threads models
  int cpu_repeats = 1;
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
      } else if (arg == "--gpus") {
        gpus = std::stoi(value());
      } else if (arg == "--worker") {
        worker = true;
      } else if (arg == "--server") {
        server = true;
      } else if (arg == "--cpu-models") {
        cpu_models = split(value());
      } else if (arg == "--cpu-repeats") {
        cpu_repeats = std::stoi(value());
      } else {
        return usage();
      }
    }
    if (config.dims.empty()) return usage();
#ifdef MMWS_GPU_BENCH_HAVE_LAUNCHER
    if (worker) return run_worker(config, calibrate);
    std::optional<mmws::MsgWorld> world;
    if (gpus >= 1) {  // even P = 1 goes through the launcher and a 1-rank NCCL world
      std::vector<std::string> child_args(argv + 1, argv + argc);
      child_args.push_back("--worker");
      world.emplace(mmws::launch_with_master("/proc/self/exe", child_args, gpus));
    }
#else
    if (gpus > 1 || worker)
      throw mmws::DomainError("--gpus > 1 needs the reference headers (its launcher) at build time");
#endif
    mmws::gpu::Context ctx(device);
#ifdef MMWS_GPU_BENCH_HAVE_LAUNCHER
    if (world) mmws::gpu::comm_init_from(ctx, world->comm);
#endif
    if (server) ctx.server_start();
    std::vector<mmws::gpu::BenchRecord> records;
    std::vector<std::pair<std::int64_t, double>> seq_times;
    if (!cpu_models.empty()) {
#ifdef MMWS_GPU_BENCH_HAVE_REF_SUITE
      mmws::BenchConfig ref;
      ref.dims = config.dims;
      ref.models.clear();
      for (const auto& m : cpu_models) {
        const mmws::Model model = mmws::model_from_name(m);
        if (model == mmws::Model::msg)
          throw mmws::DomainError("--cpu-models: msg is the TCP protocol, not a CPU model here");
        ref.models.push_back(model);
      }
      ref.repeats = cpu_repeats;
      ref.seed = config.seed;
      for (const auto& r : mmws::run_suite(ref)) {  // the reference's harness, unchanged
        mmws::gpu::BenchRecord rec;
        rec.model = mmws::model_name(r.model);
        rec.n = r.n;
        rec.workers = r.workers;
        rec.elapsed = r.elapsed;
        rec.mflops = r.mflops;
        rec.speedup = r.speedup;
        if (r.model == mmws::Model::seq) seq_times.emplace_back(r.n, r.elapsed);
        records.push_back(std::move(rec));
      }
#else
      (void)cpu_repeats;
      throw mmws::DomainError("--cpu-models needs the reference headers at build time");
#endif
    }
    for (auto& r : mmws::gpu::run_suite(ctx, config, seq_times)) records.push_back(std::move(r));
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
                  fit->link_measured ? "measured" : "B200 peer-copy reference",
                  fit->gemm_flops_per_s);
      if (fit->link_measured)
        std::printf("calibration: broadcast %.6g B/s, point-to-point %.6g B/s\n",
                    fit->broadcast_bytes_per_s, fit->p2p_bytes_per_s);
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

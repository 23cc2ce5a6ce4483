// mmws_gpu_bench.hpp -- the reference's benchmark harness (include/mmws/bench.hpp)
// extended with GPU execution models: "gpu" (FP64 tensor path), "gpu-exact"
// (bitwise matmul_seq) and "gpu-rowblock" (master/worker over the context's
// NCCL world).  Header-only, on top of mmws_gpu.hpp.
//
// Mirrors bench.hpp: model names and parsing (:30-46), the record and config
// (:48-67), mflops / speedup (:70-78), derive_seed (:83-86), time_model's
// min-of-repeats bracket (:92-129), run_suite's correctness gate (:161-168)
// and the CSV format (:190-212); plus the SVG charts of plots.hpp (:145-198:
// runtime / mflops / speedup vs N, one series per model, machine-checkable
// data-series / data-points attributes, dashed cost-model overlay) and the
// `bench calibrate` step (bench_main.cpp:64-93) re-aimed at the row-block
// cost model's two rates.  The gate is bitwise for gpu-exact and
// normwise (config.tolerance, default 1e-12) for the tensor-path models, whose
// accumulation order differs from matmul_seq's; the gate's reference product
// is mmws::matmul_seq itself when the reference headers are on the include
// path and n <= config.cpu_gate_max, else the GPU exact-order product (bitwise
// matmul_seq by construction, tests/test_gpu_parity.py).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "mmws_gpu.hpp"

#if __has_include(<mmws/matrix.hpp>)
#include <mmws/matrix.hpp>
#define MMWS_GPU_BENCH_HAVE_REFERENCE 1
#endif

namespace mmws {
namespace gpu {

struct GateError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

enum class GpuModel { gpu, gpu_exact, gpu_rowblock };

inline const char* model_name(GpuModel m) {
  switch (m) {
    case GpuModel::gpu: return "gpu";
    case GpuModel::gpu_exact: return "gpu-exact";
    case GpuModel::gpu_rowblock: return "gpu-rowblock";
  }
  return "?";
}

inline GpuModel model_from_name(const std::string& name) {
  if (name == "gpu") return GpuModel::gpu;
  if (name == "gpu-exact") return GpuModel::gpu_exact;
  if (name == "gpu-rowblock") return GpuModel::gpu_rowblock;
  throw DomainError("unknown model '" + name + "' (want gpu, gpu-exact or gpu-rowblock)");
}

struct BenchRecord {
  std::string model;
  std::int64_t n = 0;
  int workers = 1;          // GPUs
  double elapsed = 0.0;     // seconds, host matrices in -> host matrix out
  double mflops = 0.0;
  std::optional<double> speedup;
  double rel_err = 0.0;     // normwise vs the gate reference (0 for bitwise-equal)
};

struct BenchConfig {
  std::vector<std::int64_t> dims;
  std::vector<GpuModel> models = {GpuModel::gpu, GpuModel::gpu_exact};
  int repeats = 3;
  std::uint64_t seed = 42;
  double tolerance = 1e-12;
  std::int64_t cpu_gate_max = 256;  // largest N gated against mmws::matmul_seq on the host
};

// bench.hpp:70-78
inline double mflops(std::int64_t n, double elapsed) {
  if (elapsed <= 0.0) throw DomainError("mflops: elapsed must be positive");
  return static_cast<double>(op_count(n)) / elapsed / 1e6;
}

inline double speedup(double t_seq, double t_par) {
  if (t_seq <= 0.0 || t_par <= 0.0) throw DomainError("speedup: times must be positive");
  return t_seq / t_par;
}

namespace bench_detail {

inline std::uint64_t splitmix64_next(std::uint64_t& state) {  // matrix.hpp:23-28
  std::uint64_t z = (state += 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

// bench.hpp:83-86
inline std::uint64_t derive_seed(std::uint64_t seed, std::int64_t n, int which) {
  std::uint64_t state =
      seed ^ (static_cast<std::uint64_t>(n) * 2 + static_cast<std::uint64_t>(which));
  return splitmix64_next(state);
}

// random_matrix (matrix.hpp:101-107): uniform [0,1), row-major stream
inline MatrixF64 random_matrix(std::size_t rows, std::size_t cols, std::uint64_t seed) {
  std::vector<double> v(rows * cols);
  std::uint64_t state = seed;
  for (double& x : v) x = static_cast<double>(splitmix64_next(state) >> 11) * 0x1.0p-53;
  return MatrixF64(rows, cols, std::move(v));
}

inline std::string format_g6(double v) {  // bench.hpp:194-198
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.6g", v);
  return buf;
}

}  // namespace bench_detail

// One model at one dimension, `repeats` times; min elapsed and the last product
// (time_model, bench.hpp:92-129).  The bracket is the whole host-level call:
// H2D of A and B, the multiply (or master/worker round), D2H of C.
inline std::pair<MatrixF64, double> time_model(Context& ctx, GpuModel model, const MatrixF64& a,
                                               const MatrixF64& b, int repeats) {
  double best = 0.0;
  std::optional<MatrixF64> last;
  for (int r = 0; r < repeats; ++r) {
    std::vector<double> out(a.rows() * b.cols());
    double elapsed = 0.0;
    const auto m = static_cast<std::int64_t>(a.rows());
    const auto n = static_cast<std::int64_t>(b.cols());
    const auto k = static_cast<std::int64_t>(a.cols());
    if (model == GpuModel::gpu_rowblock)
      check(mmws_gpu_master_run_host(ctx.handle(), m, n, k, a.data().data(), b.data().data(),
                                     out.data(), MMWS_GPU_MODE_AUTO, &elapsed));
    else
      check(mmws_gpu_matmul_host(ctx.handle(), m, n, k, a.data().data(), b.data().data(),
                                 out.data(),
                                 model == GpuModel::gpu_exact ? MMWS_GPU_MODE_EXACT
                                                              : MMWS_GPU_MODE_AUTO,
                                 &elapsed));
    if (r == 0 || elapsed < best) best = elapsed;
    last.emplace(a.rows(), b.cols(), std::move(out));
  }
  return {std::move(*last), best};
}

inline double normwise_error(const MatrixF64& x, const MatrixF64& ref) {
  double num = 0.0, den = 0.0;
  for (std::size_t i = 0; i < ref.size(); ++i) {
    const double d = x.data()[i] - ref.data()[i];
    num += d * d;
    den += ref.data()[i] * ref.data()[i];
  }
  return den > 0.0 ? std::sqrt(num / den) : std::sqrt(num);
}

inline bool bitwise_equal(const MatrixF64& x, const MatrixF64& y) {
  return x.rows() == y.rows() && x.cols() == y.cols() &&
         std::memcmp(x.data().data(), y.data().data(), x.size() * sizeof(double)) == 0;
}

// run_suite (bench.hpp:134-188) for the GPU models; seq_times pairs
// (N, seconds) of a reference sequential run give the speedup column.
inline std::vector<BenchRecord> run_suite(
    Context& ctx, const BenchConfig& config,
    const std::vector<std::pair<std::int64_t, double>>& seq_times = {}) {
  if (config.dims.empty()) throw DomainError("run_suite: no dimensions configured");
  if (config.repeats < 1) throw DomainError("run_suite: repeats must be >= 1");
  std::vector<BenchRecord> records;
  const GpuModel order[] = {GpuModel::gpu, GpuModel::gpu_exact, GpuModel::gpu_rowblock};
  for (GpuModel model : order) {
    bool wanted = false;
    for (GpuModel m : config.models) wanted = wanted || m == model;
    if (!wanted) continue;
    for (const std::int64_t n : config.dims) {
      if (n < 1) throw DomainError("run_suite: dimensions must be >= 1");
      const auto dim = static_cast<std::size_t>(n);
      const MatrixF64 a = bench_detail::random_matrix(dim, dim, bench_detail::derive_seed(config.seed, n, 0));
      const MatrixF64 b = bench_detail::random_matrix(dim, dim, bench_detail::derive_seed(config.seed, n, 1));
      auto [c, elapsed] = time_model(ctx, model, a, b, config.repeats);

      // correctness gate (bench.hpp:161-168)
      std::optional<MatrixF64> reference;
#ifdef MMWS_GPU_BENCH_HAVE_REFERENCE
      if (n <= config.cpu_gate_max) {
        const mmws::Matrix ra(dim, dim, a.data()), rb(dim, dim, b.data());
        const mmws::Matrix rc = mmws::matmul_seq(ra, rb);
        const auto d = rc.data();
        reference.emplace(dim, dim, std::vector<double>(d.begin(), d.end()));
      }
#endif
      if (!reference) reference.emplace(matmul(ctx, a, b, Mode::exact));
      BenchRecord rec;
      rec.model = model_name(model);
      rec.n = n;
      rec.workers = model == GpuModel::gpu_rowblock ? ctx.world_size() : 1;
      rec.elapsed = elapsed;
      rec.mflops = mflops(n, elapsed);
      if (model == GpuModel::gpu_exact) {
        if (!bitwise_equal(c, *reference))
          throw GateError(std::string("correctness gate: model=") + rec.model + " n=" +
                          std::to_string(n) + " differs bitwise from matmul_seq");
      } else {
        rec.rel_err = normwise_error(c, *reference);
        if (!(rec.rel_err <= config.tolerance))
          throw GateError(std::string("correctness gate: model=") + rec.model + " n=" +
                          std::to_string(n) + " normwise error " +
                          bench_detail::format_g6(rec.rel_err) + " > " +
                          bench_detail::format_g6(config.tolerance));
      }
      for (const auto& [sn, st] : seq_times)
        if (sn == n) rec.speedup = speedup(st, elapsed);
      records.push_back(std::move(rec));
    }
  }
  return records;
}

inline constexpr const char* kCsvHeader = "model,n,workers,elapsed_s,mflops,speedup";

// emit_csv (bench.hpp:200-212): same header, %.6g numbers, empty speedup when
// there is no sequential baseline at that N.
inline std::string csv(const std::vector<BenchRecord>& records) {
  std::string out = std::string(kCsvHeader) + "\n";
  for (const auto& rec : records)
    out += rec.model + ',' + std::to_string(rec.n) + ',' + std::to_string(rec.workers) + ',' +
           bench_detail::format_g6(rec.elapsed) + ',' + bench_detail::format_g6(rec.mflops) +
           ',' + (rec.speedup ? bench_detail::format_g6(*rec.speedup) : std::string{}) + "\n";
  return out;
}

inline void emit_csv(const std::vector<BenchRecord>& records, const std::string& path) {
  std::ofstream f(path);
  if (!f) throw IoError("cannot write " + path);
  f << csv(records);
  if (!f.flush()) throw IoError("short write to " + path);
}

// ---------------------------------------------------------------- calibration
// The reference's `bench calibrate` fits tc / tf (seconds per datum moved over
// its TCP link) for cost_model.hpp.  The GPU row-block round has two rates:
// rank 0's NVLink egress (the B broadcast and the point-to-point A-slices) and
// the per-GPU multiply rate (mmws_gpu_rowblock_cost).  With a communicator of
// more than one rank both links are measured (collective: every rank must
// call it) and the slower one is the model's link rate; a 1-rank world has no
// link to measure, so the rate is the B200 peer-copy reference of 770 GB/s
// per direction (B200_PROFILING.md) and marked as not measured in this run.
struct CostFit {
  double link_bytes_per_s = 770e9;
  double broadcast_bytes_per_s = 0.0;  // measured (world > 1)
  double p2p_bytes_per_s = 0.0;        // measured (world > 1)
  double gemm_flops_per_s = 0.0;
  bool link_measured = false;
};

inline CostFit calibrate(Context& ctx, std::int64_t gemm_n = 4096,
                         std::int64_t link_bytes = std::int64_t{1} << 28) {
  CostFit fit;
  check(mmws_gpu_gemm_probe(ctx.handle(), gemm_n, MMWS_GPU_MODE_AUTO, 3, &fit.gemm_flops_per_s));
  if (ctx.world_size() > 1) {
    check(mmws_gpu_link_probe(ctx.handle(), link_bytes, 5, &fit.broadcast_bytes_per_s));
    check(mmws_gpu_p2p_probe(ctx.handle(), link_bytes, 5, &fit.p2p_bytes_per_s));
    fit.link_bytes_per_s = fit.p2p_bytes_per_s > 0.0
                               ? std::min(fit.broadcast_bytes_per_s, fit.p2p_bytes_per_s)
                               : fit.broadcast_bytes_per_s;
    fit.link_measured = true;
  }
  return fit;
}

// Predicted seconds of one gpu-rowblock round of an n x n fp64 multiply.
inline double predicted_seconds(const CostFit& fit, std::int64_t n, int workers) {
  double t = 0.0;
  check(mmws_gpu_rowblock_cost(n, n, n, workers, 8, fit.link_bytes_per_s, fit.gemm_flops_per_s,
                               &t, nullptr, nullptr));
  return t;
}

// ---------------------------------------------------------------- plots
struct PlotSeries {
  std::string name;
  std::string color;
  bool dashed = false;
  std::vector<std::pair<double, double>> points;  // (N, value), ascending N
};

namespace plot_detail {

inline std::string num(double v) { return bench_detail::format_g6(v); }

// One linear-axis line chart: title, y label, every series as a polyline
// carrying data-series="name" and data-points="n:v;n:v" (the values, not the
// pixels), a marker per point and a legend; x ticks at the measured N.
inline std::string line_chart(const std::string& title, const std::string& y_label,
                              const std::vector<PlotSeries>& series,
                              const std::string& comment) {
  const double W = 720, H = 480, left = 80, right = 24, top = 48, bottom = 56;
  const double pw = W - left - right, ph = H - top - bottom;
  std::vector<double> xs;
  double ymax = 0.0;
  for (const auto& s : series)
    for (const auto& [x, y] : s.points) {
      xs.push_back(x);
      ymax = std::max(ymax, y);
    }
  std::sort(xs.begin(), xs.end());
  xs.erase(std::unique(xs.begin(), xs.end()), xs.end());
  const double x0 = xs.empty() ? 0.0 : xs.front();
  const double x1 = xs.empty() || xs.back() == x0 ? x0 + 1.0 : xs.back();
  ymax = ymax > 0.0 ? ymax * 1.08 : 1.0;
  auto X = [&](double x) { return left + (x - x0) / (x1 - x0) * pw; };
  auto Y = [&](double y) { return top + ph * (1.0 - y / ymax); };
  auto text = [](std::ostringstream& o, double x, double y, const char* anchor, int size,
                 const std::string& body, const std::string& extra = {}) {
    o << "<text x=\"" << x << "\" y=\"" << y << "\" text-anchor=\"" << anchor
      << "\" font-size=\"" << size << "\" font-family=\"sans-serif\"" << extra << ">" << body
      << "</text>\n";
  };
  std::ostringstream o;
  o << "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"" << W << "\" height=\"" << H
    << "\" viewBox=\"0 0 " << W << ' ' << H << "\">\n";
  if (!comment.empty()) o << "<!-- " << comment << " -->\n";
  o << "<rect width=\"100%\" height=\"100%\" fill=\"white\"/>\n";
  text(o, W / 2, 26, "middle", 16, title);
  o << "<path d=\"M" << left << ' ' << top << "V" << top + ph << "H" << left + pw
    << "\" fill=\"none\" stroke=\"black\"/>\n";
  for (int t = 0; t <= 5; ++t) {
    const double v = ymax * t / 5.0;
    o << "<path d=\"M" << left - 4 << ' ' << Y(v) << "H" << left << "\" stroke=\"black\"/>\n";
    text(o, left - 8, Y(v) + 4, "end", 11, num(v));
  }
  for (double x : xs) {
    o << "<path d=\"M" << X(x) << ' ' << top + ph << "V" << top + ph + 4
      << "\" stroke=\"black\"/>\n";
    text(o, X(x), top + ph + 18, "middle", 11, num(x));
  }
  text(o, W / 2, H - 12, "middle", 12, "matrix dimension N");
  std::ostringstream rot;
  rot << " transform=\"rotate(-90 18 " << top + ph / 2 << ")\"";
  text(o, 18, top + ph / 2, "middle", 12, y_label, rot.str());
  double ly = top + 10;
  for (const auto& s : series) {
    std::string data, pts;
    for (const auto& [x, y] : s.points) {
      data += (data.empty() ? "" : ";") + num(x) + ":" + num(y);
      std::ostringstream p;
      p << (pts.empty() ? "" : " ") << X(x) << ',' << Y(y);
      pts += p.str();
    }
    const std::string dash = s.dashed ? " stroke-dasharray=\"6 3\"" : "";
    o << "<polyline fill=\"none\" stroke=\"" << s.color << "\" stroke-width=\"2\"" << dash
      << " data-series=\"" << s.name << "\" data-points=\"" << data << "\" points=\"" << pts
      << "\"/>\n";
    for (const auto& [x, y] : s.points)
      o << "<circle cx=\"" << X(x) << "\" cy=\"" << Y(y) << "\" r=\"3\" fill=\"" << s.color
        << "\"/>\n";
    o << "<path d=\"M" << left + pw - 150 << ' ' << ly << "h24\" stroke=\"" << s.color
      << "\" stroke-width=\"2\"" << dash << "/>\n";
    text(o, left + pw - 120, ly + 4, "start", 12, s.name);
    ly += 18;
  }
  o << "</svg>\n";
  return o.str();
}

inline void write_file(const std::string& path, const std::string& body) {
  std::ofstream f(path);
  if (!f) throw IoError("cannot write " + path);
  f << body;
  if (!f.flush()) throw IoError("short write to " + path);
}

inline const char* model_color(const std::string& model) {
  if (model == "seq") return "#9467bd";      // the reference's CPU models
  if (model == "threads") return "#ff7f0e";
  if (model == "gpu") return "#1f77b4";
  if (model == "gpu-exact") return "#555555";
  if (model == "gpu-rowblock") return "#d62728";
  return "#000000";
}

}  // namespace plot_detail

// emit_plots (plots.hpp:145-198): runtime.svg, mflops.svg and speedup.svg in
// `dir`, one series per model in seq / threads (the reference's CPU models,
// when present) / gpu / gpu-exact / gpu-rowblock order.  With
// a CostFit and gpu-rowblock records, runtime.svg gains the dashed
// "cost-model" series of predicted round times.
inline void emit_plots(const std::vector<BenchRecord>& records, const std::string& dir,
                       const std::optional<CostFit>& fit = std::nullopt) {
  if (records.empty()) throw DomainError("emit_plots: no records");
  std::error_code ec;
  std::filesystem::create_directories(dir, ec);
  if (ec) throw IoError("cannot create " + dir + ": " + ec.message());
  auto series_of = [&](auto value_of) {
    std::vector<PlotSeries> out;
    for (const char* name : {"seq", "threads", "gpu", "gpu-exact", "gpu-rowblock"}) {
      PlotSeries s{name, plot_detail::model_color(name), false, {}};
      for (const auto& r : records)
        if (r.model == name)
          if (const std::optional<double> v = value_of(r))
            s.points.emplace_back(static_cast<double>(r.n), *v);
      std::sort(s.points.begin(), s.points.end());
      if (!s.points.empty()) out.push_back(std::move(s));
    }
    return out;
  };
  auto runtime = series_of([](const BenchRecord& r) { return std::optional<double>(r.elapsed); });
  std::string comment;
  if (fit) {
    PlotSeries model{"cost-model", "#2ca02c", true, {}};
    for (const auto& r : records)
      if (r.model == "gpu-rowblock")
        model.points.emplace_back(static_cast<double>(r.n), predicted_seconds(*fit, r.n, r.workers));
    std::sort(model.points.begin(), model.points.end());
    if (!model.points.empty()) {
      runtime.push_back(std::move(model));
      comment = "cost-model overlay: link=" + plot_detail::num(fit->link_bytes_per_s) +
                " B/s (" + (fit->link_measured ? "measured" : "B200 peer-copy reference") +
                "), gemm=" + plot_detail::num(fit->gemm_flops_per_s) +
                " FLOP/s; predicted seconds = mmws_gpu_rowblock_cost";
    }
  }
  plot_detail::write_file(dir + "/runtime.svg",
                          plot_detail::line_chart("Running time vs matrix dimension",
                                                  "elapsed seconds", runtime, comment));
  plot_detail::write_file(
      dir + "/mflops.svg",
      plot_detail::line_chart("Throughput vs matrix dimension", "MFLOPS",
                              series_of([](const BenchRecord& r) {
                                return std::optional<double>(r.mflops);
                              }),
                              {}));
  plot_detail::write_file(
      dir + "/speedup.svg",
      plot_detail::line_chart("Speedup over sequential vs matrix dimension", "speedup",
                              series_of([](const BenchRecord& r) { return r.speedup; }), {}));
}

}  // namespace gpu
}  // namespace mmws

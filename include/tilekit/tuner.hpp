// tilekit/tuner.hpp -- per-shape tuner and tuning DB (drop-in API).
//
// Same surface and selection semantics as the reference tuner
// (tuner.hpp:36-694): Problem, ParamSpace, stock_gemm_configs,
// enumerate_gemm_configs / enumerate_conv_configs (filtered by the device
// budgets, name-sorted), benchmark_config (inputs seeded from
// fnv1a(problem.key()) ^ seed, median / min / mean, GFLOP/s = flops /
// median ns, verification on a capped proxy shape), select_best (median,
// then registers, local memory, name), tune, and the NDJSON tuning DB with
// the reference's nine keys (save_db / load_db / lookup_best).
//
// What changes on the B200:
//   * the clock: samples are device durations (CUDA events around the
//     kernel on resident inputs, tk_bench_gemm / tk_bench_conv2d) instead of
//     host wall time; BenchOptions::time_one stays as the test seam;
//   * the search space: besides the reference's h/w/r/c/loc/db (the exact
//     FP32 kernel) and conv algorithms, b200::tune explores precision
//     (exact FP32, TF32, BF16) and the tensor-core N tile.  Extended
//     candidates are named "<reference name>@<precision>[_n<tile>]"
//     (e.g. "im2col@tf32", "gemm@bf16_n128") so DB records stay one flat
//     config string and the reference grammars are untouched.
// The records carry extra keys (precision, tflops, frac_peak) that the
// reference's load_db ignores (it reads with j.at).
#pragma once

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdint>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <optional>
#include <random>
#include <sstream>
#include <string>
#include <tuple>
#include <utility>
#include <vector>

#include "tilekit/b200.hpp"
#include "tilekit/config.hpp"
#include "tilekit/conv.hpp"
#include "tilekit/device.hpp"
#include "tilekit/errors.hpp"
#include "tilekit/gemm.hpp"
#include "tilekit/numeric.hpp"
#include "tilekit/tensor.hpp"
#include "tilekit/winograd.hpp"

namespace tilekit {

// ---- problems and spaces ----------------------------------------------------

struct Problem {
  enum class Kind { Gemm, Conv };
  Kind kind = Kind::Gemm;
  GemmShape gemm;
  ConvShape conv;

  static Problem of(const GemmShape& s) {
    Problem p;
    p.kind = Kind::Gemm;
    p.gemm = s;
    return p;
  }
  static Problem of(const ConvShape& s) {
    Problem p;
    p.kind = Kind::Conv;
    p.conv = s;
    return p;
  }
  std::string key() const { return kind == Kind::Gemm ? gemm.key() : conv.key(); }
  std::uint64_t flops() const { return kind == Kind::Gemm ? gemm.flops() : conv_flops(conv); }
};

struct ParamSpace {
  std::vector<std::size_t> reg_rows{1, 2, 4, 8};
  std::vector<std::size_t> reg_cols{1, 2, 4, 8};
  std::vector<std::size_t> wg_rows{4, 8, 16};
  std::vector<std::size_t> wg_cols{4, 8, 16};
  std::vector<bool> use_local{false, true};
  std::vector<bool> double_buffer{false, true};
  std::vector<std::size_t> tile_rows{1, 2, 3, 4, 5};
  std::vector<std::size_t> tile_cols{1, 2, 3, 4, 5};
  std::vector<std::size_t> channel_vectors{1, 2, 4, 8};
  std::vector<std::size_t> feature_vectors{1, 2, 4, 8};
  std::vector<ConvAlgo> algos{ConvAlgo::Naive, ConvAlgo::Tiled, ConvAlgo::Im2col,
                              ConvAlgo::Winograd};
  // B200 axes (b200::tune only)
  std::vector<b200::Precision> precisions{b200::Precision::Fp32Exact, b200::Precision::Tf32,
                                          b200::Precision::Bf16};
  std::vector<int> tc_tiles{0};  // GEMM N tile, 0 = library choice
  std::vector<int> tc_stages{0};     // shared-memory ring depth, 0 = library choice
  std::vector<int> tc_clusters{0};   // 1 = one SM, 2 = CTA pair, 0 = library choice
  std::vector<b200::TcMode> tc_modes{b200::TcMode::Auto};  // conv operand path
};

inline std::vector<GemmConfig> stock_gemm_configs() {
  std::vector<GemmConfig> out;
  for (const char* n : {"4x4_8x8_loc", "4x4_16x16_loc", "8x4_8x16_loc", "8x2_4x16_loc",
                        "8x4_8x16_noloc", "8x4_4x8_noloc", "4x4_8x8_noloc"})
    out.push_back(parse_gemm_config(n));
  return out;
}

namespace detail {

template <typename T, typename Key>
void sort_by_name(std::vector<T>& v, Key key) {
  std::sort(v.begin(), v.end(), [&](const T& a, const T& b) { return key(a) < key(b); });
}

// The constraint that filtered the most candidates ("[name] kind: ...").
inline std::string binding_constraint(const std::vector<std::string>& rejected) {
  if (rejected.empty()) return "no constraint";
  std::map<std::string, std::size_t> tally;
  for (const std::string& r : rejected) {
    const std::size_t from = r.find("] ") == std::string::npos ? 0 : r.find("] ") + 2;
    const std::size_t colon = r.find(": ", from);
    ++tally[colon == std::string::npos ? r : r.substr(from, colon - from)];
  }
  auto best = tally.begin();
  for (auto it = tally.begin(); it != tally.end(); ++it)
    if (it->second > best->second) best = it;
  return "binding constraint: " + best->first + " (rejected " + std::to_string(best->second) +
         " of " + std::to_string(rejected.size()) + " candidates)";
}

}  // namespace detail

inline std::vector<GemmConfig> enumerate_gemm_configs(const ParamSpace& space,
                                                      const DeviceSpec& dev,
                                                      const GemmShape& shape,
                                                      std::vector<std::string>* rejected = nullptr) {
  std::vector<GemmConfig> out;
  for (std::size_t h : space.reg_rows)
    for (std::size_t w : space.reg_cols)
      for (std::size_t r : space.wg_rows)
        for (std::size_t c : space.wg_cols)
          for (bool loc : space.use_local)
            for (bool db : space.double_buffer) {
              if (db && !loc) continue;  // no "noloc_db" in the grammar
              GemmConfig cfg;
              cfg.reg_rows = h;
              cfg.reg_cols = w;
              cfg.wg_rows = r;
              cfg.wg_cols = c;
              cfg.use_local_memory = loc;
              cfg.double_buffer = db;
              const ConfigVerdict v = validate_config(cfg, dev, shape);
              if (v.ok) out.push_back(cfg);
              else if (rejected) rejected->push_back("[" + cfg.name() + "] " + v.summary());
            }
  detail::sort_by_name(out, [](const GemmConfig& c) { return c.name(); });
  return out;
}

inline std::vector<ConvAlgoParams> enumerate_conv_configs(
    const ParamSpace& space, const ConvShape& shape,
    std::vector<std::string>* rejected = nullptr) {
  std::vector<ConvAlgoParams> out;
  auto reject = [&](const ConvAlgoParams& p, const std::string& why) {
    if (rejected) rejected->push_back("[" + p.name() + "] " + why);
  };
  auto has = [](const std::vector<std::size_t>& v, std::size_t x) {
    return std::find(v.begin(), v.end(), x) != v.end();
  };
  for (ConvAlgo algo : space.algos) {
    ConvAlgoParams p;
    p.algo = algo;
    if (algo == ConvAlgo::Naive || algo == ConvAlgo::Im2col) {
      out.push_back(p);
    } else if (algo == ConvAlgo::Tiled) {
      for (std::size_t tr : space.tile_rows)
        for (std::size_t tc : space.tile_cols)
          for (std::size_t cv : space.channel_vectors)
            for (std::size_t fv : space.feature_vectors) {
              p.tile_rows = tr;
              p.tile_cols = tc;
              p.channel_vector = cv;
              p.feature_vector = fv;
              if (!valid_vector_width(cv) || !valid_vector_width(fv))
                reject(p, "vector constraint: widths must be in {1,2,4,8}");
              else if (tr == 0 || tc == 0)
                reject(p, "tile constraint: tile dims must be >= 1");
              else if (shape.stride != 1 && shape.stride != 2)
                reject(p, "stride constraint: tiled kernel handles strides 1 and 2");
              else
                out.push_back(p);
            }
    } else {
      for (std::size_t t : {std::size_t{2}, std::size_t{4}}) {
        p.tile_rows = p.tile_cols = t;
        if (!has(space.tile_rows, t) || !has(space.tile_cols, t)) continue;
        if (shape.stride != 1)
          reject(p, "stride constraint: fast convolution requires stride 1");
        else if (shape.window_rows != 3 || shape.window_cols != 3)
          reject(p, "window constraint: no transform plan for " +
                        std::to_string(shape.window_rows) + "x" +
                        std::to_string(shape.window_cols) + " windows");
        else
          out.push_back(p);
      }
    }
  }
  detail::sort_by_name(out, [](const ConvAlgoParams& c) { return c.name(); });
  return out;
}

// ---- records and benchmarking ---------------------------------------------------

struct TuningRecord {
  std::string problem;
  std::string config;
  std::string device;
  int samples = 0;
  std::int64_t median_ns = 0;
  std::int64_t min_ns = 0;
  std::int64_t mean_ns = 0;
  double gflops = 0.0;
  bool valid = true;
  // B200 additions (extra NDJSON keys the reference's load_db ignores):
  // the throughput as a fraction of the precision's nominal dense peak
  // (tensor pipe for TF32/BF16, the FMUL+FADD issue cap for exact FP32) and
  // the compulsory-traffic bandwidth (operands once, result once; the
  // analysis.hpp model) over the median time.
  double frac_of_peak = 0.0;
  double algo_gbs = 0.0;

  bool operator==(const TuningRecord&) const = default;
};

struct BenchOptions {
  int warmup = 5;
  int samples = 20;
  std::uint64_t seed = 0;
  // Test seams (reference tuner.hpp:275-279): time_one replaces the clock
  // (it receives the kernel invocation), verify_override the oracle check.
  std::function<std::int64_t(const std::function<void()>&)> time_one;
  std::function<bool()> verify_override;
  // B200 additions: the precision / tensor-core tile the candidate runs
  // with, and a replacement for the kernel invocation (host-only tests).
  b200::ExecOptions exec;
  std::function<void()> run_override;
};

namespace detail {

inline std::uint64_t fnv1a(const std::string& text) {
  std::uint64_t h = 1469598103934665603ull;
  for (unsigned char ch : text) {
    h ^= ch;
    h *= 1099511628211ull;
  }
  return h;
}

inline void fill_random(std::vector<float>& v, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
  for (float& x : v) x = dist(rng);
}

inline void check_bench_options(const BenchOptions& o) {
  if (o.samples < 3) throw ContractError("benchmark_config: samples must be >= 3");
  if (o.warmup < 1) throw ContractError("benchmark_config: warmup must be >= 1");
}

// Median (rounded-down midpoint for even counts), min and mean.
inline void summarize_times(std::vector<std::int64_t> t, TuningRecord& rec) {
  std::sort(t.begin(), t.end());
  const std::size_t n = t.size();
  rec.min_ns = t.front();
  rec.median_ns = (n % 2) ? t[n / 2] : (t[n / 2 - 1] + t[n / 2]) / 2;
  std::int64_t sum = 0;
  for (std::int64_t x : t) sum += x;
  rec.mean_ns = sum / static_cast<std::int64_t>(n);
}

inline GemmShape gemm_proxy(GemmShape s) {
  s.m = std::min<std::size_t>(s.m, 128);
  s.n = std::min<std::size_t>(s.n, 128);
  s.k = std::min<std::size_t>(s.k, 128);
  return s;
}

inline ConvShape conv_proxy(ConvShape s) {
  s.batch = std::min<std::size_t>(s.batch, 2);
  s.in_rows = std::max(s.window_rows, std::min<std::size_t>(s.in_rows, 24));
  s.in_cols = std::max(s.window_cols, std::min<std::size_t>(s.in_cols, 24));
  // Channel / feature counts pick the tensor-core operand path (slab
  // alignment, halo vs pixel boxes): keep them, so a candidate is verified
  // on the path it was timed on.
  s.channels = std::min<std::size_t>(s.channels, 512);
  s.features = std::min<std::size_t>(s.features, 512);
  return s;
}

// Tolerance of a precision under the metric the reference uses for it.
inline double tolerance(b200::Precision p) {
  switch (p) {
    case b200::Precision::Fp32Exact: return 1e-4;  // elementwise (we are bit-exact)
    case b200::Precision::Tf32: return 1e-3;       // scaled
    case b200::Precision::Bf16: return 5e-3;       // scaled
    default: return 1e-3;
  }
}

inline Matrix sized(std::size_t r, std::size_t c, std::uint64_t seed) {
  Matrix m(r, c);
  fill_random(m.data, seed);
  return m;
}

inline Tensor4 sized(Tensor4Layout l, std::size_t a, std::size_t b, std::size_t c, std::size_t d,
                     std::uint64_t seed) {
  Tensor4 t(l, a, b, c, d);
  fill_random(t.data, seed);
  return t;
}

// Nominal dense peaks of a B200 (TF/s) per precision.
inline double nominal_peak_tflops(b200::Precision p) {
  switch (p) {
    case b200::Precision::Tf32: return 1125.0;
    case b200::Precision::Bf16: return 2250.0;
    case b200::Precision::Tf32x3: return 375.0;
    default: return 148 * 128 * 1.965e-3;  // one FMUL + one FADD per MAC: half of FFMA
  }
}

inline double compulsory_bytes(const Problem& p) {
  if (p.kind == Problem::Kind::Gemm) {
    const double m = (double)p.gemm.m, n = (double)p.gemm.n, k = (double)p.gemm.k;
    return 4.0 * (m * k + k * n + m * n * (p.gemm.beta != 0.0f ? 2.0 : 1.0));
  }
  const ConvShape& c = p.conv;
  return 4.0 * ((double)c.batch * c.in_rows * c.in_cols * c.channels +
                (double)c.window_rows * c.window_cols * c.channels * c.features +
                (double)c.batch * c.out_rows() * c.out_cols() * c.features);
}

template <typename Bench>
TuningRecord run_bench(const Problem& problem, const std::string& config,
                       const DeviceSpec& dev, const BenchOptions& opts,
                       const std::function<void()>& host_run, Bench&& device_bench) {
  TuningRecord rec;
  rec.problem = problem.key();
  rec.config = config;
  rec.device = dev.name;
  rec.samples = opts.samples;
  std::vector<std::int64_t> t(static_cast<std::size_t>(opts.samples));
  if (opts.time_one) {
    const std::function<void()> run = opts.run_override ? opts.run_override : host_run;
    for (int i = 0; i < opts.warmup; ++i) run();
    for (auto& x : t) x = opts.time_one(run);
  } else {
    device_bench(t.data());
  }
  summarize_times(std::move(t), rec);
  const double ns = static_cast<double>(std::max<std::int64_t>(rec.median_ns, 1));
  rec.gflops = static_cast<double>(problem.flops()) / ns;
  rec.frac_of_peak = rec.gflops / (1e3 * nominal_peak_tflops(opts.exec.precision));
  rec.algo_gbs = compulsory_bytes(problem) / ns;
  return rec;
}

}  // namespace detail

// GEMM candidate: device-timed B200 kernel on seeded inputs; verified on
// a proxy shape against gemm_naive.
inline TuningRecord benchmark_config(const Problem& problem, const GemmConfig& cfg,
                                     const DeviceSpec& dev, const BenchOptions& opts = {}) {
  if (problem.kind != Problem::Kind::Gemm)
    throw ContractError("benchmark_config: GEMM config given a non-GEMM problem");
  detail::check_bench_options(opts);
  const GemmShape& s = problem.gemm;
  const std::uint64_t seed = detail::fnv1a(problem.key()) ^ opts.seed;
  const bool ta = s.op_a == Op::Transpose, tb = s.op_b == Op::Transpose;
  const Matrix a = detail::sized(ta ? s.k : s.m, ta ? s.m : s.k, seed);
  const Matrix b = detail::sized(tb ? s.n : s.k, tb ? s.k : s.n, seed + 1);
  const Matrix c = detail::sized(s.m, s.n, seed + 2);
  const bool exact = opts.exec.precision == b200::Precision::Fp32Exact;
  if (exact) {  // the budget check gemm_tiled makes before any launch
    const ConfigVerdict v = validate_config(cfg, dev, s);
    if (!v.ok)
      throw ConfigError("gemm_tiled: config \"" + cfg.name() + "\" rejected: " + v.summary());
  }
  const std::string name =
      exact ? cfg.name() : "gemm@" + b200::precision_name(opts.exec.precision) + opts.exec.suffix();
  TuningRecord rec = detail::run_bench(
      problem, name, dev, opts, [&] { gemm_tiled(a, b, c, s, cfg, dev); },
      [&](std::int64_t* out) {
        const tk_gemm_shape cs = detail::to_c(s);
        const tk_gemm_config cc = detail::to_c(cfg);
        const tk_exec_options eo = opts.exec.c();
        detail::check_status(tk_bench_gemm(&cs, &cc, &eo, a.data.data(), b.data.data(),
                                           c.data.data(), opts.warmup, opts.samples, out));
      });
  if (opts.verify_override) {
    rec.valid = opts.verify_override();
  } else {
    const GemmShape px = detail::gemm_proxy(s);
    const Matrix pa = detail::sized(ta ? px.k : px.m, ta ? px.m : px.k, seed + 3);
    const Matrix pb = detail::sized(tb ? px.n : px.k, tb ? px.k : px.n, seed + 4);
    const Matrix pc = detail::sized(px.m, px.n, seed + 5);
    const Matrix want = gemm_naive(pa, pb, pc, px);
    if (exact) {
      rec.valid = max_rel_error(gemm_tiled(pa, pb, pc, px, cfg, dev).data, want.data) <= 1e-4;
    } else {
      rec.valid = max_scaled_error(b200::gemm(pa, pb, pc, px, opts.exec).data, want.data) <=
                  detail::tolerance(opts.exec.precision);
    }
  }
  return rec;
}

// Convolution candidate (algorithm + precision), verified against
// conv2d_naive on a proxy shape with the reference tolerances (Winograd and
// tensor-core precisions under max_scaled_error).
inline TuningRecord benchmark_config(const Problem& problem, const ConvAlgoParams& params,
                                     const DeviceSpec& dev, const BenchOptions& opts = {}) {
  if (problem.kind != Problem::Kind::Conv)
    throw ContractError("benchmark_config: conv params given a non-conv problem");
  detail::check_bench_options(opts);
  const ConvShape& s = problem.conv;
  const std::uint64_t seed = detail::fnv1a(problem.key()) ^ opts.seed;
  const Tensor4 in = detail::sized(Tensor4Layout::InputNhwc, s.batch, s.in_rows, s.in_cols,
                                   s.channels, seed);
  const Tensor4 filt = detail::sized(Tensor4Layout::FilterHwck, s.window_rows, s.window_cols,
                                     s.channels, s.features, seed + 1);
  const bool exact = opts.exec.precision == b200::Precision::Fp32Exact;
  const std::string name =
      exact ? params.name()
            : params.name() + "@" + b200::precision_name(opts.exec.precision) + opts.exec.suffix();
  TuningRecord rec = detail::run_bench(
      problem, name, dev, opts,
      [&] {
        if (exact) conv2d(in, filt, s, params);
        else b200::conv2d(in, filt, s, params, opts.exec);
      },
      [&](std::int64_t* out) {
        const tk_conv_shape cs = detail::to_c(s);
        const tk_conv_params cp = detail::to_c(params);
        const tk_exec_options eo = opts.exec.c();
        detail::check_status(tk_bench_conv2d(&cs, &cp, &eo, in.data.data(), filt.data.data(),
                                             opts.warmup, opts.samples, out));
      });
  if (opts.verify_override) {
    rec.valid = opts.verify_override();
  } else {
    const ConvShape px = detail::conv_proxy(s);
    const Tensor4 pin = detail::sized(Tensor4Layout::InputNhwc, px.batch, px.in_rows, px.in_cols,
                                      px.channels, seed + 2);
    const Tensor4 pf = detail::sized(Tensor4Layout::FilterHwck, px.window_rows, px.window_cols,
                                     px.channels, px.features, seed + 3);
    const Tensor4 want = conv2d_naive(pin, pf, px);
    const Tensor4 got = exact ? conv2d(pin, pf, px, params) : b200::conv2d(pin, pf, px, params, opts.exec);
    if (params.algo == ConvAlgo::Winograd || !exact) {
      const double tol = std::max(params.algo == ConvAlgo::Winograd ? 1e-3 : 0.0,
                                  exact ? 0.0 : detail::tolerance(opts.exec.precision)) *
                         (params.algo == ConvAlgo::Winograd && params.tile_rows == 4 && !exact
                              ? 10.0
                              : 1.0);
      rec.valid = max_scaled_error(got.data, want.data) <= tol;
    } else {
      rec.valid = max_rel_error(got.data, want.data) <= (params.algo == ConvAlgo::Im2col ? 1e-5 : 1e-4);
    }
  }
  return rec;
}

// ---- selection ------------------------------------------------------------------

namespace detail {

// Tie-break keys recoverable from the config name (reference tuner.hpp:482-507).
struct SelectionRank {
  std::size_t registers = 1;
  std::size_t local_mem = 0;
};

inline SelectionRank selection_rank(const std::string& name) {
  SelectionRank r;
  const std::string base = name.substr(0, name.find('@'));
  try {
    const GemmConfig c = parse_gemm_config(base);
    r.registers = c.register_tile();
    if (c.use_local_memory)
      r.local_mem = (c.double_buffer ? 2 : 1) * (c.block_rows() + c.block_cols());
    return r;
  } catch (const ParseError&) {
  }
  try {
    const ConvAlgoParams p = parse_conv_params(base);
    r.registers = p.tile_rows * p.tile_cols * p.channel_vector * p.feature_vector;
  } catch (const ParseError&) {
  }
  return r;
}

}  // namespace detail

inline std::optional<TuningRecord> select_best(const std::vector<TuningRecord>& records) {
  std::optional<TuningRecord> best;
  auto key = [](const TuningRecord& r) {
    const detail::SelectionRank k = detail::selection_rank(r.config);
    return std::make_tuple(r.median_ns, k.registers, k.local_mem, r.config);
  };
  for (const TuningRecord& r : records) {
    if (!r.valid) continue;
    if (!best || key(r) < key(*best)) best = r;
  }
  return best;
}

struct TuneResult {
  TuningRecord best;
  std::vector<TuningRecord> records;
};

namespace detail {

inline TuneResult finish(std::vector<TuningRecord> records) {
  const std::optional<TuningRecord> best = select_best(records);
  if (!best) {
    std::string why;
    for (const TuningRecord& r : records) why += (why.empty() ? "[" : "; [") + r.config + "] oracle mismatch";
    throw TuningError("tune: no config passed verification (" + why + ")");
  }
  return TuneResult{*best, std::move(records)};
}

}  // namespace detail

inline TuneResult tune(const Problem& problem, const std::vector<GemmConfig>& candidates,
                       const DeviceSpec& dev, const BenchOptions& opts = {}) {
  std::vector<TuningRecord> records;
  std::vector<std::string> rejected;
  for (const GemmConfig& cfg : candidates) {
    const ConfigVerdict v = validate_config(cfg, dev, problem.gemm);
    if (!v.ok) {
      rejected.push_back("[" + cfg.name() + "] " + v.summary());
      continue;
    }
    records.push_back(benchmark_config(problem, cfg, dev, opts));
  }
  if (records.empty())
    throw TuningError("tune: no feasible config for device \"" + dev.name + "\"; " +
                      detail::binding_constraint(rejected));
  return detail::finish(std::move(records));
}

inline TuneResult tune(const Problem& problem, const ParamSpace& space, const DeviceSpec& dev,
                       const BenchOptions& opts = {}) {
  std::vector<std::string> rejected;
  std::vector<TuningRecord> records;
  if (problem.kind == Problem::Kind::Gemm) {
    const auto cfgs = enumerate_gemm_configs(space, dev, problem.gemm, &rejected);
    if (cfgs.empty())
      throw TuningError("tune: empty GEMM config space for device \"" + dev.name + "\"; " +
                        detail::binding_constraint(rejected));
    for (const GemmConfig& c : cfgs) records.push_back(benchmark_config(problem, c, dev, opts));
  } else {
    const auto cfgs = enumerate_conv_configs(space, problem.conv, &rejected);
    if (cfgs.empty())
      throw TuningError("tune: empty conv config space; " + detail::binding_constraint(rejected));
    for (const ConvAlgoParams& p : cfgs) records.push_back(benchmark_config(problem, p, dev, opts));
  }
  return detail::finish(std::move(records));
}

// ---- tuning DB (NDJSON, one flat object per line) ----------------------------------

namespace detail {

inline std::string json_escape(const std::string& s) {
  std::string o;
  for (char ch : s) {
    if (ch == '"' || ch == '\\') o += '\\';
    o += ch;
  }
  return o;
}

// Parses one flat JSON object of string / number / bool values.
inline std::map<std::string, std::string> parse_flat_json(const std::string& line,
                                                          const std::string& where) {
  std::map<std::string, std::string> kv;
  std::size_t i = 0;
  auto bad = [&](const std::string& why) -> void {
    throw ParseError(where + ": malformed tuning record: " + why);
  };
  auto ws = [&] {
    while (i < line.size() && std::isspace(static_cast<unsigned char>(line[i]))) ++i;
  };
  auto str = [&]() -> std::string {
    if (i >= line.size() || line[i] != '"') bad("expected a string");
    std::string out;
    for (++i; i < line.size() && line[i] != '"'; ++i) {
      if (line[i] == '\\' && i + 1 < line.size()) ++i;
      out += line[i];
    }
    if (i >= line.size()) bad("unterminated string");
    ++i;
    return out;
  };
  ws();
  if (i >= line.size() || line[i] != '{') bad("expected '{'");
  ++i;
  ws();
  if (i < line.size() && line[i] == '}') return kv;
  while (true) {
    ws();
    const std::string key = str();
    ws();
    if (i >= line.size() || line[i] != ':') bad("expected ':'");
    ++i;
    ws();
    std::string val;
    if (i < line.size() && line[i] == '"') {
      val = "\"" + str();
    } else {
      const std::size_t b = i;
      while (i < line.size() && line[i] != ',' && line[i] != '}') ++i;
      val = line.substr(b, i - b);
      while (!val.empty() && std::isspace(static_cast<unsigned char>(val.back()))) val.pop_back();
      if (val.empty()) bad("missing value for \"" + key + "\"");
    }
    kv[key] = val;
    ws();
    if (i < line.size() && line[i] == ',') {
      ++i;
      continue;
    }
    if (i < line.size() && line[i] == '}') {
      ++i;
      break;
    }
    bad("expected ',' or '}'");
  }
  ws();
  if (i != line.size()) bad("trailing characters");
  return kv;
}

}  // namespace detail

inline void save_db(const std::vector<TuningRecord>& records, const std::string& path) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw IoError("save_db: cannot open " + path + " for writing");
  out.precision(17);
  for (const TuningRecord& r : records) {
    out << "{\"problem\":\"" << detail::json_escape(r.problem) << "\",\"config\":\""
        << detail::json_escape(r.config) << "\",\"device\":\"" << detail::json_escape(r.device)
        << "\",\"samples\":" << r.samples << ",\"median_ns\":" << r.median_ns
        << ",\"min_ns\":" << r.min_ns << ",\"mean_ns\":" << r.mean_ns << ",\"gflops\":" << r.gflops
        << ",\"valid\":" << (r.valid ? "true" : "false");
    const std::size_t at = r.config.find('@');
    const std::string tag = at == std::string::npos ? "fp32" : r.config.substr(at + 1);
    out << ",\"precision\":\"" << tag.substr(0, tag.find('_')) << "\",\"frac_of_peak\":"
        << r.frac_of_peak << ",\"algo_gbs\":" << r.algo_gbs << "}\n";
  }
  if (!out) throw IoError("save_db: write to " + path + " failed");
}

inline std::vector<TuningRecord> load_db(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("load_db: cannot open " + path);
  std::vector<TuningRecord> records;
  std::map<std::tuple<std::string, std::string, std::string>, std::size_t> where;
  std::string line;
  for (std::size_t lineno = 1; std::getline(in, line); ++lineno) {
    if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
    const std::string loc = path + ":" + std::to_string(lineno);
    const auto kv = detail::parse_flat_json(line, loc);
    auto need = [&](const char* k) -> const std::string& {
      const auto it = kv.find(k);
      if (it == kv.end())
        throw ParseError(loc + ": malformed tuning record: missing key \"" + std::string(k) + "\"");
      return it->second;
    };
    auto as_str = [&](const char* k) {
      const std::string& v = need(k);
      if (v.empty() || v[0] != '"')
        throw ParseError(loc + ": malformed tuning record: \"" + std::string(k) + "\" is not a string");
      return v.substr(1);
    };
    auto as_num = [&](const char* k) {
      const std::string& v = need(k);
      try {
        std::size_t used = 0;
        const double d = std::stod(v, &used);
        if (used != v.size()) throw std::invalid_argument(v);
        return d;
      } catch (const std::exception&) {
        throw ParseError(loc + ": malformed tuning record: \"" + std::string(k) + "\" is not a number");
      }
    };
    TuningRecord r;
    r.problem = as_str("problem");
    r.config = as_str("config");
    r.device = as_str("device");
    r.samples = static_cast<int>(as_num("samples"));
    r.median_ns = static_cast<std::int64_t>(as_num("median_ns"));
    r.min_ns = static_cast<std::int64_t>(as_num("min_ns"));
    r.mean_ns = static_cast<std::int64_t>(as_num("mean_ns"));
    r.gflops = as_num("gflops");
    const std::string& valid = need("valid");
    if (valid != "true" && valid != "false")
      throw ParseError(loc + ": malformed tuning record: \"valid\" is not a bool");
    r.valid = valid == "true";
    if (kv.count("frac_of_peak")) r.frac_of_peak = as_num("frac_of_peak");
    if (kv.count("algo_gbs")) r.algo_gbs = as_num("algo_gbs");
    const auto key = std::make_tuple(r.problem, r.config, r.device);
    const auto it = where.find(key);
    if (it != where.end()) {
      std::cerr << "load_db: " << loc << ": duplicate record for (" << r.problem << ", "
                << r.config << ", " << r.device << "); keeping the later one\n";
      records[it->second] = r;
    } else {
      where.emplace(key, records.size());
      records.push_back(r);
    }
  }
  return records;
}

inline std::optional<TuningRecord> lookup_best(const std::vector<TuningRecord>& records,
                                               const std::string& problem_key,
                                               const std::string& device_name) {
  std::vector<TuningRecord> match;
  for (const TuningRecord& r : records)
    if (r.problem == problem_key && r.device == device_name) match.push_back(r);
  return select_best(match);
}

// ---- B200 search space ----------------------------------------------------------------

namespace b200 {

// Tunes one problem over the B200 space: the reference's candidates in
// exact FP32 plus, for the tensor-core precisions in the space, the
// tensor-core paths (conv: im2col and Winograd; GEMM: the tcgen05 GEMM per
// N tile).  Device-timed; every record verified; same selection rule.
inline TuneResult tune(const Problem& problem, const ParamSpace& space, const DeviceSpec& dev,
                       const BenchOptions& base = {}) {
  std::vector<TuningRecord> records;
  for (Precision prec : space.precisions) {
    BenchOptions o = base;
    o.exec.precision = prec;
    if (prec == Precision::Fp32Exact) {
      if (problem.kind == Problem::Kind::Gemm) {
        for (const GemmConfig& c : enumerate_gemm_configs(space, dev, problem.gemm))
          records.push_back(benchmark_config(problem, c, dev, o));
      } else {
        for (const ConvAlgoParams& p : enumerate_conv_configs(space, problem.conv))
          records.push_back(benchmark_config(problem, p, dev, o));
      }
      continue;
    }
    for (int stages : space.tc_stages) {
      for (int cluster : space.tc_clusters) {
        o.exec.tc_stages = stages;
        o.exec.tc_cluster = cluster;
        if (problem.kind == Problem::Kind::Gemm) {
          for (int tile : space.tc_tiles) {
            o.exec.tc_tile_n = tile;
            records.push_back(benchmark_config(problem, GemmConfig{}, dev, o));
          }
          continue;
        }
        ParamSpace tc = space;
        tc.algos = {ConvAlgo::Im2col, ConvAlgo::Winograd};
        for (const ConvAlgoParams& p : enumerate_conv_configs(tc, problem.conv)) {
          if (p.algo == ConvAlgo::Winograd && prec != Precision::Tf32) continue;
          for (TcMode mode : space.tc_modes) {
            if (p.algo == ConvAlgo::Winograd && mode != TcMode::Auto) continue;
            o.exec.tc_mode = mode;
            // A knob combination the shape cannot run is a rejected
            // candidate, not a failed tune.
            try {
              records.push_back(benchmark_config(problem, p, dev, o));
            } catch (const CapabilityError&) {
            }
          }
          o.exec.tc_mode = TcMode::Auto;
        }
      }
    }
  }
  if (records.empty()) throw TuningError("tune: empty B200 search space");
  return tilekit::detail::finish(std::move(records));
}

}  // namespace b200
}  // namespace tilekit

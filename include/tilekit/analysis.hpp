// tilekit/analysis.hpp -- roofline model, GEMM sweep and report formats of
// the drop-in API (reference analysis.hpp:29-259).
//
// Operational intensity follows the reference's compulsory-traffic model
// (every operand read once, the result written once, C read again when
// beta != 0).  `sweep` times every (size, config) point through the B200
// tuner clock (`benchmark_config`, CUDA events on the device) and keeps
// failing points flagged instead of aborting.  Reports are the reference's
// two formats: CSV with the fixed header and `%.9g` numbers, or a JSON
// array laid out the way nlohmann::json::dump(2) lays it out (sorted keys,
// two-space indent, shortest round-trip numbers) -- no JSON library needed.
#pragma once

#include <algorithm>
#include <array>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <fstream>
#include <string>
#include <tuple>
#include <vector>

#include "tilekit/config.hpp"
#include "tilekit/conv.hpp"
#include "tilekit/device.hpp"
#include "tilekit/errors.hpp"
#include "tilekit/tuner.hpp"

namespace tilekit {

// ---- operational intensity (analysis.hpp:29-52) ---------------------------------------

// flops / compulsory bytes of a GEMM: A, B and C once, C twice with beta != 0.
inline double gemm_oi(const GemmShape& shape) {
  const double m = static_cast<double>(shape.m), n = static_cast<double>(shape.n),
               k = static_cast<double>(shape.k);
  const double c_traffic = (shape.beta != 0.0f ? 2.0 : 1.0) * m * n;
  return 2.0 * m * n * k / (4.0 * (m * k + k * n + c_traffic));
}

// conv_flops / compulsory bytes of a convolution: input, filter, output once.
inline double conv_oi(const ConvShape& shape) {
  const double n = static_cast<double>(shape.batch);
  const double elems =
      n * static_cast<double>(shape.in_rows) * static_cast<double>(shape.in_cols) *
          static_cast<double>(shape.channels) +
      static_cast<double>(shape.window_rows) * static_cast<double>(shape.window_cols) *
          static_cast<double>(shape.channels) * static_cast<double>(shape.features) +
      n * static_cast<double>(shape.out_rows()) * static_cast<double>(shape.out_cols()) *
          static_cast<double>(shape.features);
  return static_cast<double>(conv_flops(shape)) / (4.0 * elems);
}

// ---- sweep (analysis.hpp:58-118) ------------------------------------------------------

struct RooflinePoint {
  std::string problem;
  std::string config;
  double oi = 0.0;
  double gflops = 0.0;
  bool ok = true;     // false when this point's benchmark failed
  std::string error;  // why, when !ok
};

// {64, 128, 256, 512, 1024}^3 in (m, n, k) lexicographic order: 125 points.
inline std::vector<std::array<std::size_t, 3>> default_sweep_grid() {
  constexpr std::size_t kDims[] = {64, 128, 256, 512, 1024};
  std::vector<std::array<std::size_t, 3>> grid;
  grid.reserve(125);
  for (std::size_t m : kDims)
    for (std::size_t n : kDims)
      for (std::size_t k : kDims) grid.push_back({m, n, k});
  return grid;
}

// One point per (size, config), sizes outermost.  The template supplies
// alpha, beta and the ops; `opts.exec` selects the B200 precision the
// candidates run at (exact FP32 reproduces the reference's numbers).
inline std::vector<RooflinePoint> sweep(const GemmShape& tmpl,
                                        const std::vector<std::array<std::size_t, 3>>& sizes,
                                        const std::vector<GemmConfig>& configs,
                                        const DeviceSpec& dev, const BenchOptions& opts = {}) {
  if (sizes.empty()) throw ContractError("sweep: empty size list");
  std::vector<RooflinePoint> points;
  points.reserve(sizes.size() * configs.size());
  for (const auto& [m, n, k] : sizes) {
    GemmShape shape = tmpl;
    shape.m = m;
    shape.n = n;
    shape.k = k;
    for (const GemmConfig& cfg : configs) {
      RooflinePoint pt;
      pt.problem = shape.key();
      pt.config = cfg.name();
      pt.oi = gemm_oi(shape);
      try {
        const TuningRecord rec = benchmark_config(Problem::of(shape), cfg, dev, opts);
        pt.config = rec.config;  // carries the @precision suffix off the exact path
        pt.gflops = rec.gflops;
        if (!rec.valid) {
          pt.ok = false;
          pt.error = "oracle mismatch";
        }
      } catch (const std::exception& e) {
        pt.ok = false;
        pt.error = e.what();
      }
      points.push_back(std::move(pt));
    }
  }
  return points;
}

// ---- reports (analysis.hpp:124-259) ---------------------------------------------------

enum class ReportFormat { Csv, Json };

inline ReportFormat parse_report_format(const std::string& text) {
  if (text == "csv") return ReportFormat::Csv;
  if (text == "json") return ReportFormat::Json;
  throw ParseError("unknown report format \"" + text + "\" (csv or json)");
}

namespace detail {

inline constexpr const char* kReportHeader = "problem,config,oi_flops_per_byte,gflops";

inline std::string sig9(double v) {
  char buf[48];
  std::snprintf(buf, sizeof buf, "%.9g", v);
  return buf;
}

// A double the way nlohmann::json serialises it: shortest round-trip
// digits; plain notation for decimal exponents in (-4, 15] (".0" appended
// to integral values), otherwise d.ddde+XX; non-finite values as null.
inline std::string json_number(double v) {
  if (!std::isfinite(v)) return "null";
  if (v == 0.0) return std::signbit(v) ? "-0.0" : "0.0";
  char buf[64];
  const auto res = std::to_chars(buf, buf + sizeof buf, v, std::chars_format::scientific);
  std::string sci(buf, res.ptr);
  std::string sign;
  if (sci[0] == '-') {
    sign = "-";
    sci.erase(0, 1);
  }
  const std::size_t e = sci.find('e');
  std::string digits = sci.substr(0, e);
  digits.erase(std::remove(digits.begin(), digits.end(), '.'), digits.end());
  const int exp10 = std::stoi(sci.substr(e + 1));
  const int k = static_cast<int>(digits.size());
  const int n = exp10 + 1;  // value = 0.digits * 10^n
  std::string out;
  if (k <= n && n <= 15) {
    out = digits + std::string(static_cast<std::size_t>(n - k), '0') + ".0";
  } else if (0 < n && n <= 15) {
    out = digits.substr(0, static_cast<std::size_t>(n)) + "." + digits.substr(static_cast<std::size_t>(n));
  } else if (-4 < n && n <= 0) {
    out = "0." + std::string(static_cast<std::size_t>(-n), '0') + digits;
  } else {
    out = digits.substr(0, 1);
    if (k > 1) out += "." + digits.substr(1);
    const int x = n - 1;
    char eb[16];
    std::snprintf(eb, sizeof eb, "e%c%02d", x < 0 ? '-' : '+', x < 0 ? -x : x);
    out += eb;
  }
  return sign + out;
}

inline std::vector<RooflinePoint> report_rows(std::vector<RooflinePoint> points) {
  points.erase(std::remove_if(points.begin(), points.end(),
                              [](const RooflinePoint& p) { return !p.ok; }),
               points.end());
  std::stable_sort(points.begin(), points.end(), [](const RooflinePoint& a, const RooflinePoint& b) {
    return std::tie(a.problem, a.config) < std::tie(b.problem, b.config);
  });
  return points;
}

// Splits a JSON array of flat objects into the objects' source text.
inline std::vector<std::string> json_array_objects(const std::string& text) {
  auto bad = [](const std::string& why) { return ParseError("report JSON: " + why); };
  std::vector<std::string> objs;
  std::size_t i = 0;
  auto ws = [&] {
    while (i < text.size() && std::isspace(static_cast<unsigned char>(text[i]))) ++i;
  };
  ws();
  if (i >= text.size() || text[i] != '[') {
    if (i < text.size() && text[i] == '{') throw bad("expected an array");
    throw bad("syntax error: expected '['");
  }
  ++i;
  ws();
  if (i < text.size() && text[i] == ']') {
    ++i;
  } else {
    while (true) {
      ws();
      if (i >= text.size() || text[i] != '{') throw bad("syntax error: expected an object");
      const std::size_t b = i;
      bool in_str = false;
      for (; i < text.size(); ++i) {
        const char ch = text[i];
        if (in_str) {
          if (ch == '\\') ++i;
          else if (ch == '"') in_str = false;
        } else if (ch == '"') {
          in_str = true;
        } else if (ch == '{' && i != b) {
          throw bad("nested objects are not report points");
        } else if (ch == '}') {
          break;
        }
      }
      if (i >= text.size()) throw bad("syntax error: unterminated object");
      objs.push_back(text.substr(b, ++i - b));
      ws();
      if (i < text.size() && text[i] == ',') {
        ++i;
        continue;
      }
      if (i < text.size() && text[i] == ']') {
        ++i;
        break;
      }
      throw bad("syntax error: expected ',' or ']'");
    }
  }
  ws();
  if (i != text.size()) throw bad("syntax error: trailing characters");
  return objs;
}

}  // namespace detail

// Failed points dropped, rows sorted by (problem, config): byte-stable.
inline std::string render_report(const std::vector<RooflinePoint>& points, ReportFormat format) {
  const std::vector<RooflinePoint> rows = detail::report_rows(points);
  std::string out;
  if (format == ReportFormat::Csv) {
    out = std::string(detail::kReportHeader) + "\n";
    for (const RooflinePoint& p : rows)
      out += p.problem + "," + p.config + "," + detail::sig9(p.oi) + "," + detail::sig9(p.gflops) +
             "\n";
    return out;
  }
  if (rows.empty()) return "[]\n";
  out = "[\n";
  for (std::size_t i = 0; i < rows.size(); ++i) {
    const RooflinePoint& p = rows[i];
    out += "  {\n    \"config\": \"" + detail::json_escape(p.config) + "\",\n    \"gflops\": " +
           detail::json_number(p.gflops) + ",\n    \"oi_flops_per_byte\": " +
           detail::json_number(p.oi) + ",\n    \"problem\": \"" + detail::json_escape(p.problem) +
           "\"\n  }" + (i + 1 < rows.size() ? ",\n" : "\n");
  }
  return out + "]\n";
}

inline void emit_report(const std::vector<RooflinePoint>& points, ReportFormat format,
                        const std::string& path) {
  std::ofstream out(path, std::ios::trunc);
  if (!out) throw IoError("emit_report: cannot open " + path + " for writing");
  out << render_report(points, format);
  if (!out) throw IoError("emit_report: write to " + path + " failed");
}

// Inverse of render_report up to number formatting; every point is ok.
inline std::vector<RooflinePoint> parse_report(const std::string& text, ReportFormat format) {
  std::vector<RooflinePoint> points;
  auto number = [](const std::string& s, const std::string& where) {
    try {
      std::size_t used = 0;
      const double v = std::stod(s, &used);
      if (used != s.size()) throw std::invalid_argument(s);
      return v;
    } catch (const std::exception&) {
      throw ParseError(where + ": malformed number");
    }
  };
  if (format == ReportFormat::Csv) {
    std::size_t pos = 0, lineno = 0;
    while (pos < text.size()) {
      std::size_t eol = text.find('\n', pos);
      if (eol == std::string::npos) eol = text.size();
      const std::string line = text.substr(pos, eol - pos);
      pos = eol + 1;
      ++lineno;
      if (line.empty()) continue;
      const std::string where = "report line " + std::to_string(lineno);
      if (lineno == 1) {
        if (line != detail::kReportHeader)
          throw ParseError(where + ": unexpected CSV header \"" + line + "\"");
        continue;
      }
      std::vector<std::string> f;
      for (std::size_t b = 0;;) {
        const std::size_t c = line.find(',', b);
        f.push_back(line.substr(b, c == std::string::npos ? std::string::npos : c - b));
        if (c == std::string::npos) break;
        b = c + 1;
      }
      if (f.size() != 4) throw ParseError(where + ": expected 4 comma-separated fields");
      RooflinePoint p;
      p.problem = f[0];
      p.config = f[1];
      p.oi = number(f[2], where);
      p.gflops = number(f[3], where);
      points.push_back(std::move(p));
    }
    return points;
  }
  for (const std::string& obj : detail::json_array_objects(text)) {
    std::map<std::string, std::string> kv;
    try {
      kv = detail::parse_flat_json(obj, "report JSON");
    } catch (const ParseError& e) {
      throw ParseError(std::string("report JSON: ") + e.what());
    }
    auto need = [&](const char* key) -> const std::string& {
      const auto it = kv.find(key);
      if (it == kv.end()) throw ParseError(std::string("report JSON: key '") + key + "' not found");
      return it->second;
    };
    auto str = [&](const char* key) {
      const std::string& v = need(key);
      if (v.empty() || v[0] != '"')
        throw ParseError(std::string("report JSON: '") + key + "' is not a string");
      return v.substr(1);
    };
    RooflinePoint p;
    p.problem = str("problem");
    p.config = str("config");
    p.oi = number(need("oi_flops_per_byte"), "report JSON");
    p.gflops = number(need("gflops"), "report JSON");
    points.push_back(std::move(p));
  }
  return points;
}

}  // namespace tilekit

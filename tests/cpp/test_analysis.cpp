// test_analysis.cpp -- roofline model, sweep, reports and layer tables of the
// drop-in API.
//
//   test_analysis cpu <golden_dir> <data_dir>   model, reports, layer tables,
//                                               sweep through the tuner's
//                                               host-only seams
//   test_analysis gpu <golden_dir> <data_dir>   + a device-clock sweep
//
// Cases follow the reference's tests/test_analysis.cpp and
// tests/test_layers.cpp; report bytes and layer-table errors are compared
// with fixtures rendered by the unmodified reference
// (tests/golden/make_golden_formats.py).
#include <cmath>
#include <cstdio>
#include <fstream>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "tilekit/tilekit.hpp"

using namespace tilekit;

static int g_fail = 0;
#define CHECK(cond)                                               \
  do {                                                            \
    if (!(cond)) {                                                \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++g_fail;                                                   \
    }                                                             \
  } while (0)

template <typename E, typename F>
static bool throws_with(F&& f, const char* needle = nullptr) {
  try {
    f();
  } catch (const E& e) {
    return !needle || std::string(e.what()).find(needle) != std::string::npos;
  } catch (...) {
    return false;
  }
  return false;
}

static bool near(double a, double b, double eps) { return std::fabs(a - b) <= eps * std::fabs(b); }

static std::string slurp(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

static GemmShape cube(std::size_t d, float beta = 0.0f) {
  return GemmShape{d, d, d, 1.0f, beta, Op::Identity, Op::Identity};
}

static BenchOptions scripted() {
  BenchOptions o;
  o.warmup = 1;
  o.samples = 3;
  o.time_one = [](const std::function<void()>&) -> std::int64_t { return 1000; };
  o.verify_override = [] { return true; };
  o.run_override = [] {};
  return o;
}

// ---- minimal JSON string-array reader for the fixtures -----------------------------

static std::vector<std::string> json_strings_after(const std::string& text, const std::string& key,
                                                   std::vector<std::size_t>* at = nullptr) {
  std::vector<std::string> out;
  const std::string pat = "\"" + key + "\": \"";
  for (std::size_t p = text.find(pat); p != std::string::npos; p = text.find(pat, p + 1)) {
    std::string v;
    std::size_t i = p + pat.size();
    for (; text[i] != '"'; ++i) {
      if (text[i] == '\\') {
        ++i;
        v += text[i] == 'n' ? '\n' : text[i] == 't' ? '\t' : text[i];
      } else {
        v += text[i];
      }
    }
    out.push_back(v);
    if (at) at->push_back(p);
  }
  return out;
}

static void model_checks() {
  // analysis.hpp:29-52 / test_analysis.cpp:22-68
  CHECK(near(gemm_oi(cube(1024)), 2048.0 / 12.0, 1e-12));
  CHECK(gemm_oi(cube(1024, 1.0f)) == 128.0);
  for (std::size_t d : {64, 128, 256, 512, 1024}) CHECK(near(gemm_oi(cube(d, 1.0f)), d / 8.0, 1e-12));
  GemmShape s{384, 192, 96, 1.0f, 0.0f, Op::Identity, Op::Identity};
  const double base = gemm_oi(s);
  s.op_a = s.op_b = Op::Transpose;
  CHECK(gemm_oi(s) == base);
  s.beta = 1.0f;
  const double upd = gemm_oi(s);
  CHECK(upd < base);
  s.beta = -2.5f;
  CHECK(gemm_oi(s) == upd);

  const ConvShape pw{1, 56, 56, 64, 64, 1, 1, 1, Padding::Same};
  const double flops = 2.0 * 56 * 56 * 64 * 64;
  const double bytes = 4.0 * (56 * 56 * 64 + 64 * 64 + 56 * 56 * 64);
  CHECK(near(conv_oi(pw), flops / bytes, 1e-12));
  CHECK(near(conv_oi(pw), 15.8384, 1e-4));
  ConvShape sp = pw;
  sp.window_rows = sp.window_cols = 3;
  CHECK(conv_oi(sp) > 8.0 * conv_oi(pw) && conv_oi(sp) < 9.0 * conv_oi(pw));
  ConvShape b2 = pw;
  b2.batch = 2;
  CHECK(conv_oi(b2) > conv_oi(pw));

  const auto grid = default_sweep_grid();
  CHECK(grid.size() == 125);
  const std::set<std::array<std::size_t, 3>> uniq(grid.begin(), grid.end());
  CHECK(uniq.size() == 125);
  CHECK((grid.front() == std::array<std::size_t, 3>{64, 64, 64}));
  CHECK((grid[1] == std::array<std::size_t, 3>{64, 64, 128}));
}

static void sweep_checks_host() {
  const DeviceSpec dev = find_device("Intel Core i7-6700K GPU");
  const std::vector<std::array<std::size_t, 3>> sizes = {{16, 16, 16}, {16, 32, 16}};
  const std::vector<GemmConfig> cfgs = {parse_gemm_config("4x4_8x8_noloc"),
                                        parse_gemm_config("4x4_8x8_loc")};
  const auto pts = sweep(cube(0), sizes, cfgs, dev, scripted());
  CHECK(pts.size() == 4);
  for (const auto& p : pts) CHECK(p.ok && p.oi > 0.0 && p.gflops > 0.0);
  CHECK(pts[0].problem == "gemm_nn_m16_n16_k16" && pts[2].problem == "gemm_nn_m16_n32_k16");
  CHECK(pts[1].config == "4x4_8x8_loc");
  CHECK(pts[0].gflops == 2.0 * 16 * 16 * 16 / 1000.0);
  CHECK(throws_with<ContractError>([&] { sweep(cube(0), {}, cfgs, dev, scripted()); }));

  // A _loc config on a device without local memory: flagged, scan continues.
  const auto mali = sweep(cube(0), {{16, 16, 16}}, cfgs, find_device("mali"), scripted());
  CHECK(mali.size() == 2 && mali[0].ok && !mali[1].ok);
  CHECK(mali[1].error.find("local-memory budget") != std::string::npos);

  // A failing oracle check keeps the point, flagged.
  BenchOptions bad = scripted();
  bad.verify_override = [] { return false; };
  const auto wrong = sweep(cube(0), {{16, 16, 16}}, {cfgs[0]}, dev, bad);
  CHECK(!wrong[0].ok && wrong[0].error == "oracle mismatch");

  // Off the exact path the point's config names the precision.
  BenchOptions tf = scripted();
  tf.exec.precision = b200::Precision::Tf32;
  const auto tfp = sweep(cube(0), {{16, 16, 16}}, {cfgs[0]}, dev, tf);
  CHECK(tfp[0].ok && tfp[0].config == "gemm@tf32");
}

static void report_checks(const std::string& golden) {
  // Byte-identical to the reference's render_report on the same points.
  std::vector<RooflinePoint> pts;
  {
    // report_points.json: [[problem, config, oi, gflops, ok], ...]
    const std::string t = slurp(golden + "/report_points.json");
    std::size_t i = 0;
    while ((i = t.find('[', i + 1)) != std::string::npos) {
      const std::size_t e = t.find(']', i);
      std::string row = t.substr(i + 1, e - i - 1);
      std::vector<std::string> f;
      std::stringstream ss(row);
      for (std::string x; std::getline(ss, x, ',');) f.push_back(detail::strip(x));
      RooflinePoint p;
      p.problem = f[0].substr(1, f[0].size() - 2);
      p.config = f[1].substr(1, f[1].size() - 2);
      p.oi = std::stod(f[2]);
      p.gflops = std::stod(f[3]);
      p.ok = f[4] != "0";
      pts.push_back(p);
      i = e;
    }
  }
  CHECK(pts.size() == 12);
  const std::string csv = render_report(pts, ReportFormat::Csv);
  const std::string json = render_report(pts, ReportFormat::Json);
  CHECK(csv == slurp(golden + "/report.csv"));
  CHECK(json == slurp(golden + "/report.json"));
  if (json != slurp(golden + "/report.json")) std::printf("%s\n", json.c_str());

  // Round trips at 6+ significant digits, sorted (test_analysis.cpp:125-161).
  for (ReportFormat f : {ReportFormat::Csv, ReportFormat::Json}) {
    const auto back = parse_report(render_report(pts, f), f);
    CHECK(back.size() == 11);
    for (std::size_t i = 1; i < back.size(); ++i)
      CHECK(std::tie(back[i - 1].problem, back[i - 1].config) <
            std::tie(back[i].problem, back[i].config));
    for (const auto& b : back)
      for (const auto& p : pts)
        if (p.problem == b.problem && p.config == b.config) {
          CHECK(near(b.oi, p.oi, 1e-6) || (b.oi == 0 && p.oi == 0));
          CHECK(near(b.gflops, p.gflops, 1e-6));
        }
  }
  CHECK(render_report({}, ReportFormat::Csv) == "problem,config,oi_flops_per_byte,gflops\n");
  CHECK(render_report({}, ReportFormat::Json) == "[]\n");
  CHECK(csv.find("broken") == std::string::npos);

  CHECK(throws_with<ParseError>([] { parse_report("wrong,header\n", ReportFormat::Csv); }, "header"));
  CHECK(throws_with<ParseError>([] {
    parse_report("problem,config,oi_flops_per_byte,gflops\nonly,three,fields\n", ReportFormat::Csv);
  }));
  CHECK(throws_with<ParseError>([] {
    parse_report("problem,config,oi_flops_per_byte,gflops\na,b,not_a_number,1\n", ReportFormat::Csv);
  }));
  CHECK(throws_with<ParseError>([] { parse_report("{not json", ReportFormat::Json); }));
  CHECK(throws_with<ParseError>([] { parse_report("{\"a\": 1}", ReportFormat::Json); }, "array"));
  CHECK(throws_with<ParseError>([] { parse_report("[{\"problem\": \"p\"}]", ReportFormat::Json); }));
  CHECK(parse_report("[]", ReportFormat::Json).empty());

  const std::string path = "tilekit_test_report.csv";
  std::vector<RooflinePoint> one(1);
  one[0].problem = "gemm_nn_m8_n8_k8";
  one[0].config = "cfg";
  one[0].oi = 0.5;
  one[0].gflops = 1.5;
  emit_report(one, ReportFormat::Csv, path);
  CHECK(slurp(path).find("gemm_nn_m8_n8_k8") != std::string::npos);
  std::remove(path.c_str());
  CHECK(throws_with<IoError>([&] { emit_report(one, ReportFormat::Csv, "no_such_dir/r.csv"); }));
  CHECK(parse_report_format("csv") == ReportFormat::Csv);
  CHECK(parse_report_format("json") == ReportFormat::Json);
  CHECK(throws_with<ParseError>([] { parse_report_format("xml"); }));
}

static void layer_checks(const std::string& golden, const std::string& data) {
  // Every fixture table: same serialisation or the same error message as
  // the reference's load_layer_rows.
  const std::string t = slurp(golden + "/layers.json");
  std::vector<std::size_t> at_text;
  const auto texts = json_strings_after(t, "text", &at_text);
  CHECK(texts.size() == 17);
  for (std::size_t i = 0; i < texts.size(); ++i) {
    const std::size_t end = i + 1 < at_text.size() ? at_text[i + 1] : t.size();
    const std::string entry = t.substr(at_text[i], end - at_text[i]);
    const auto err = json_strings_after(entry, "error");
    const auto ser = json_strings_after(entry, "serialized");
    std::istringstream in(texts[i]);
    try {
      const auto rows = load_layer_rows(in, "test.csv");
      CHECK(ser.size() == 1 && serialize_layer_rows(rows) == ser[0]);
    } catch (const ParseError& e) {
      CHECK(err.size() == 1 && err[0] == e.what());
      if (err.empty() || err[0] != e.what()) std::printf("  got: %s\n", e.what());
    }
  }
  // test_layers.cpp:41-73
  LayerRow same{"same", 3, 1, {56, 56, 128}, {56, 56, 256}};
  CHECK(same.to_shape().padding == Padding::Same && same.to_shape().features == 256);
  LayerRow valid{"valid", 3, 1, {10, 10, 4}, {8, 8, 6}};
  CHECK(valid.to_shape().padding == Padding::Valid && valid.to_shape().out_rows() == 8);
  LayerRow stem{"stem", 7, 2, {224, 224, 3}, {112, 112, 64}};
  CHECK(stem.to_shape(8).batch == 8 && stem.to_shape().pad_top() == 2);

  // Bundled tables (test_layers.cpp:130-166)
  const auto vgg = load_layer_rows(data + "/vgg_layers.csv");
  CHECK(vgg.size() == 9 && vgg[0].layer == "vgg_conv1_1");
  for (const ConvShape& s : load_layers(data + "/vgg_layers.csv", 4))
    CHECK(s.batch == 4 && s.padding == Padding::Same && s.window_rows == 3 && s.stride == 1);
  const auto rn = load_layer_rows(data + "/resnet_layers.csv");
  CHECK(rn.size() == 21 && rn[0].layer == "resnet_conv1" && rn[0].window == 7);
  CHECK(rn[0].to_shape().out_rows() == 112 && rn[0].to_shape().pad_top() == 2);
  CHECK(throws_with<IoError>([] { load_layer_rows("no_such_layers.csv"); }));
}

static void gpu_checks(const std::string& data) {
  // Device-clock sweep over the VGG16 table's im2col GEMMs on exact FP32
  // and TF32 + the reference grid corner.
  const DeviceSpec b200 = b200_device();
  BenchOptions o;
  o.warmup = 2;
  o.samples = 5;
  const auto pts = sweep(cube(0), {{64, 64, 64}, {1024, 1024, 1024}},
                         {parse_gemm_config("8x8_16x16_loc_db"), parse_gemm_config("4x4_8x8_loc")},
                         b200, o);
  CHECK(pts.size() == 4);
  for (const auto& p : pts) {
    CHECK(p.ok && p.gflops > 0.0);
    if (!p.ok) std::printf("  %s %s: %s\n", p.problem.c_str(), p.config.c_str(), p.error.c_str());
  }
  o.exec.precision = b200::Precision::Tf32;
  const auto tf = sweep(cube(0), {{1024, 1024, 1024}}, {parse_gemm_config("4x4_8x8_loc")}, b200, o);
  CHECK(tf.size() == 1 && tf[0].ok && tf[0].config == "gemm@tf32");
  CHECK(tf[0].gflops > pts[2].gflops);  // tensor cores beat the exact SIMT path
  const auto back = parse_report(render_report(pts, ReportFormat::Json), ReportFormat::Json);
  CHECK(back.size() == 4);
  std::printf("%s", render_report(pts, ReportFormat::Csv).c_str());
  // Every VGG16 layer's conv roofline model evaluates (config 5 of SURVEY 8d).
  for (const ConvShape& s : load_layers(data + "/vgg_layers.csv", 32)) CHECK(conv_oi(s) > 10.0);
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  const std::string golden = argc > 2 ? argv[2] : "tests/golden";
  const std::string data = argc > 3 ? argv[3] : "data";
  model_checks();
  sweep_checks_host();
  report_checks(golden);
  layer_checks(golden, data);
  if (mode == "gpu") gpu_checks(data);
  std::printf("%s: %d failure(s)\n", mode.c_str(), g_fail);
  return g_fail;
}

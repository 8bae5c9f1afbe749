// test_tuner.cpp -- the tuner / tuning DB of the drop-in API.
//
//   test_tuner cpu   selection, enumeration, DB and benchmarking logic via the
//                    reference's test seams (scripted clock, verify override,
//                    plus the B200 run_override) -- no device needed
//   test_tuner gpu   device-clock tuning of a GEMM and a VGG16 layer over the
//                    B200 space (exact FP32 / TF32 / BF16), DB round trip
//
// Cases follow the reference's tests/test_tuner.cpp.
#include <cstdio>
#include <set>
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
static bool throws_with(F&& f, const char* needle) {
  try {
    f();
  } catch (const E& e) {
    return !needle || std::string(e.what()).find(needle) != std::string::npos;
  } catch (...) {
    return false;
  }
  return false;
}

struct ScriptedClock {
  std::vector<std::int64_t> times;
  std::size_t next = 0;
  std::int64_t operator()(const std::function<void()>&) { return times[next++ % times.size()]; }
};

static BenchOptions scripted(std::vector<std::int64_t> times) {
  BenchOptions o;
  o.warmup = 1;
  o.samples = static_cast<int>(times.size());
  o.time_one = ScriptedClock{std::move(times), 0};
  o.verify_override = [] { return true; };
  o.run_override = [] {};  // host-only: never touch the device
  return o;
}

static TuningRecord rec(const std::string& cfg, std::int64_t median,
                        const std::string& problem = "gemm_nn_m64_n64_k64",
                        const std::string& device = "dev") {
  TuningRecord r;
  r.problem = problem;
  r.config = cfg;
  r.device = device;
  r.samples = 5;
  r.median_ns = median;
  r.min_ns = median - 1;
  r.mean_ns = median;
  r.gflops = 1.0;
  return r;
}

static GemmShape g(std::size_t m, std::size_t n, std::size_t k) {
  GemmShape s;
  s.m = m;
  s.n = n;
  s.k = k;
  return s;
}

static void cpu_checks() {
  const DeviceSpec gpu = find_device("Intel Core i7-6700K GPU");
  for (const GemmConfig& c : stock_gemm_configs()) {
    CHECK(parse_gemm_config(c.name()).name() == c.name());
    CHECK(validate_config(c, gpu, {}).ok);
  }
  ParamSpace space;
  const auto cands = enumerate_gemm_configs(space, gpu, g(64, 64, 64));
  CHECK(!cands.empty());
  for (const GemmConfig& c : cands) CHECK(validate_config(c, gpu, {}).ok);
  for (std::size_t i = 1; i < cands.size(); ++i) CHECK(cands[i - 1].name() < cands[i].name());
  for (const GemmConfig& c : enumerate_gemm_configs(space, find_device("mali"), g(64, 64, 64)))
    CHECK(!c.use_local_memory);
  DeviceSpec small = gpu;
  small.local_memory_bytes = 4096;
  CHECK(enumerate_gemm_configs(space, small, g(64, 64, 64)).size() <= cands.size());

  DeviceSpec impossible = gpu;
  impossible.max_workgroup_size = 1;
  CHECK(throws_with<TuningError>(
      [&] { tune(Problem::of(g(64, 64, 64)), space, impossible, scripted({1, 1, 1})); },
      "binding constraint: work-group budget"));

  // conv applicability (test_tuner.cpp:150-189)
  ConvShape s2;
  s2.in_rows = s2.in_cols = 8;
  s2.channels = s2.features = 4;
  s2.window_rows = s2.window_cols = 3;
  s2.stride = 2;
  for (const ConvAlgoParams& p : enumerate_conv_configs(space, s2))
    CHECK(p.algo != ConvAlgo::Winograd);
  ConvShape s1 = s2;
  s1.stride = 1;
  int wino = 0;
  for (const ConvAlgoParams& p : enumerate_conv_configs(space, s1)) wino += p.algo == ConvAlgo::Winograd;
  CHECK(wino == 2);

  // scripted benchmark (test_tuner.cpp:191-240)
  const Problem p64 = Problem::of(g(64, 64, 64));
  const TuningRecord r = benchmark_config(p64, parse_gemm_config("4x4_8x8_loc"), gpu,
                                          scripted({500, 100, 300}));
  CHECK(r.median_ns == 300 && r.min_ns == 100 && r.mean_ns == 300 && r.samples == 3);
  CHECK(r.gflops == static_cast<double>(p64.flops()) / 300.0);
  BenchOptions bad = scripted({5, 5, 5});
  bad.verify_override = [] { return false; };
  CHECK(!benchmark_config(p64, parse_gemm_config("4x4_8x8_loc"), gpu, bad).valid);
  BenchOptions few = scripted({5, 5});
  CHECK(throws_with<ContractError>(
      [&] { benchmark_config(p64, parse_gemm_config("4x4_8x8_loc"), gpu, few); }, "samples"));

  // selection (test_tuner.cpp:259-317)
  std::vector<TuningRecord> rs = {rec("8x4_8x16_loc", 100), rec("4x4_8x8_loc", 100),
                                  rec("4x4_8x8_noloc", 100), rec("2x2_8x8_loc", 150)};
  CHECK(select_best(rs)->config == "4x4_8x8_noloc");  // fewer local memory at equal registers
  rs[2].valid = false;
  CHECK(select_best(rs)->config == "4x4_8x8_loc");
  rs.push_back(rec("8x8_16x16_loc@tf32", 50));
  CHECK(select_best(rs)->config == "8x8_16x16_loc@tf32");
  const TuneResult tr = tune(p64, stock_gemm_configs(), gpu, scripted({7, 7, 7}));
  CHECK(tr.records.size() == 7 && tr.best.config == "4x4_8x8_noloc");

  // DB (test_tuner.cpp:319-375)
  const std::string path = "tilekit_test_db.ndjson";
  save_db(tr.records, path);
  CHECK(load_db(path) == tr.records);
  {
    std::FILE* f = std::fopen(path.c_str(), "a");
    std::fprintf(f, "{\"problem\":\"%s\",\"config\":\"4x4_8x8_loc\",\"device\":\"%s\","
                    "\"samples\":3,\"median_ns\":1,\"min_ns\":1,\"mean_ns\":1,\"gflops\":9.5,"
                    "\"valid\":true}\n",
                 p64.key().c_str(), gpu.name.c_str());
    std::fclose(f);
  }
  const auto db = load_db(path);
  CHECK(db.size() == 7);
  CHECK(lookup_best(db, p64.key(), gpu.name)->config == "4x4_8x8_loc");
  CHECK(!lookup_best(db, p64.key(), "other").has_value());
  {
    std::FILE* f = std::fopen(path.c_str(), "a");
    std::fprintf(f, "\n{\"problem\": \"x\", \"config\": }\n");
    std::fclose(f);
  }
  CHECK(throws_with<ParseError>([&] { load_db(path); }, ":10:"));
  std::remove(path.c_str());
  CHECK(throws_with<IoError>([&] { load_db("/nonexistent/db.ndjson"); }, "cannot open"));

  // conv end to end with a scripted clock (test_tuner.cpp:377-398)
  ConvShape vc;
  vc.in_rows = vc.in_cols = 8;
  vc.channels = vc.features = 4;
  vc.window_rows = vc.window_cols = 3;
  ParamSpace narrow;
  narrow.tile_rows = {2};
  narrow.tile_cols = {2};
  narrow.channel_vectors = {4};
  narrow.feature_vectors = {4};
  const TuneResult ct = tune(Problem::of(vc), narrow, gpu, scripted({3, 3, 3}));
  CHECK(ct.records.size() == 4);  // im2col, naive, tiled_t2x2_v4x4, winograd_t2x2
  std::set<std::string> names;
  for (const auto& x : ct.records) names.insert(x.config);
  CHECK(names.count("winograd_t2x2") == 1);
}

static void gpu_checks() {
  const DeviceSpec b200 = b200_device();
  BenchOptions o;
  o.warmup = 2;
  o.samples = 5;
  // GEMM: the reference's stock candidates on the device clock
  const TuneResult gt = tune(Problem::of(g(512, 512, 512)), stock_gemm_configs(), b200, o);
  CHECK(gt.records.size() == 7);
  for (const auto& r : gt.records) CHECK(r.valid && r.median_ns > 0);
  // B200 space on a VGG16 layer (batch 1): exact, TF32, BF16 candidates
  ConvShape vs;
  vs.in_rows = vs.in_cols = 56;
  vs.channels = vs.features = 256;
  vs.window_rows = vs.window_cols = 3;
  ParamSpace sp;
  sp.tile_rows = {2, 4};
  sp.tile_cols = {2, 4};
  sp.channel_vectors = {4};
  sp.feature_vectors = {4};
  const TuneResult ct = b200::tune(Problem::of(vs), sp, b200, o);
  std::set<std::string> precs;
  for (const auto& r : ct.records) {
    CHECK(r.valid);
    const auto at = r.config.find('@');
    const std::string tag = at == std::string::npos ? "fp32" : r.config.substr(at + 1);
    precs.insert(tag.substr(0, tag.find('_')));
    CHECK(r.frac_of_peak > 0.0 && r.algo_gbs > 0.0);  // Winograd counts direct flops: may exceed 1
  }
  CHECK(precs.count("fp32") && precs.count("tf32") && precs.count("bf16"));
  CHECK(ct.best.config.find('@') != std::string::npos);  // tensor cores win on this layer

  // Pipeline depth, cluster shape and operand path as tuning axes: every
  // candidate runs, verifies, and is named by its knobs.
  ParamSpace kn;
  kn.precisions = {b200::Precision::Tf32};
  kn.tc_stages = {0, 4};
  kn.tc_clusters = {0, 1};
  kn.tc_modes = {b200::TcMode::Auto, b200::TcMode::PixN, b200::TcMode::PixM};
  ConvShape ks = vs;
  ks.batch = 2;
  const TuneResult kt = b200::tune(Problem::of(ks), kn, b200, o);
  std::set<std::string> names;
  for (const auto& r : kt.records) {
    CHECK(r.valid);
    names.insert(r.config);
  }
  const bool all = names.count("im2col@tf32") && names.count("im2col@tf32_s4") &&
                   names.count("im2col@tf32_c1_pixn") && names.count("im2col@tf32_s4_pixm");
  CHECK(all);
  if (!all)
    for (const auto& n : names) std::printf("  candidate %s\n", n.c_str());
  std::printf("knob tune best for %s: %s (%.1f GFLOP/s, %.0f%% of peak)\n",
              kt.best.problem.c_str(), kt.best.config.c_str(), kt.best.gflops,
              100.0 * kt.best.frac_of_peak);
  save_db(ct.records, "tilekit_test_gpu.ndjson");
  CHECK(load_db("tilekit_test_gpu.ndjson").size() == ct.records.size());
  std::remove("tilekit_test_gpu.ndjson");
  std::printf("best for %s: %s (%.1f GFLOP/s)\n", ct.best.problem.c_str(), ct.best.config.c_str(),
              ct.best.gflops);
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  cpu_checks();
  if (mode == "gpu") gpu_checks();
  std::printf("%s: %d failure(s)\n", mode.c_str(), g_fail);
  return g_fail;
}

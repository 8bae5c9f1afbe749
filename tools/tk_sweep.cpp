// tk_sweep -- the roofline sweep of SURVEY.md 8(d) config 4 on the B200:
// the reference grid {64..1024}^3 (analysis.hpp:58-81), the large squares
// 2048/4096/8192 and the im2col GEMMs of every VGG16 / ResNet-50 layer at
// batch 32 (data/*.csv), each at one precision, written as the reference's
// CSV report (`reference roofline` workflow, tilekit_cli.cpp:305-345).
//
//   tk_sweep fp32|tf32|bf16 <out.csv> [grid|squares|layers|all] [db.ndjson[,db2...]]
//
// With tuning DBs (tools/tune_gemm.py, tools/tune_ncu.py) loaded, every
// tensor-core point runs its per-shape tuned knobs (tk_tuning_db_load:
// lookup_best on the launch path) -- configs[3]'s "per-shape tuned tile
// parameters".
//
// Build: g++ -std=c++20 -O2 -I include tools/tk_sweep.cpp -o tools/tk_sweep
//        -L paper_1904_05347_b200 -ltilekit_b200 -Wl,-rpath,$PWD/paper_1904_05347_b200
#include <cstdio>
#include <string>
#include <vector>

#include "tilekit/tilekit.hpp"

using namespace tilekit;

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: tk_sweep fp32|tf32|bf16 out.csv [grid|squares|layers|all] [db.ndjson,...]\n");
    return 2;
  }
  const std::string prec = argv[1], out = argv[2], which = argc > 3 ? argv[3] : "all";
  if (argc > 4) {
    std::string dbs = argv[4];
    for (std::size_t p = 0; p <= dbs.size();) {
      const std::size_t e = std::min(dbs.find(',', p), dbs.size());
      const std::string path = dbs.substr(p, e - p);
      std::size_t n = 0;
      if (!path.empty() && tk_tuning_db_load(path.c_str(), nullptr, &n) != TK_OK) {
        std::fprintf(stderr, "tuning DB %s: %s\n", path.c_str(), tk_last_error());
        return 2;
      }
      std::printf("tuning DB %s: %zu records\n", path.c_str(), n);
      p = e + 1;
    }
  }
  const DeviceSpec dev = b200_device();
  BenchOptions opts;
  opts.warmup = 3;
  opts.samples = 10;
  opts.exec.precision = prec == "tf32"   ? b200::Precision::Tf32
                        : prec == "bf16" ? b200::Precision::Bf16
                                         : b200::Precision::Fp32Exact;
  // The exact path runs the library default tile plus the reference's best
  // stock config; tensor-core points ignore the SIMT config.
  std::vector<GemmConfig> cfgs = {parse_gemm_config("8x8_16x16_loc_db")};
  if (prec == "fp32") cfgs.push_back(parse_gemm_config("8x4_8x16_loc"));

  std::vector<std::array<std::size_t, 3>> sizes;
  if (which == "grid" || which == "all") sizes = default_sweep_grid();
  if (which == "squares" || which == "all")
    for (std::size_t d : {2048, 4096, 8192}) sizes.push_back({d, d, d});
  if (which == "layers" || which == "all") {
    for (const char* table : {"data/vgg_layers.csv", "data/resnet_layers.csv"})
      for (const ConvShape& s : load_layers(table, 32))
        sizes.push_back({s.batch * s.out_rows() * s.out_cols(), s.features,
                         s.window_rows * s.window_cols * s.channels});
  }
  GemmShape tmpl;
  tmpl.alpha = 1.0f;
  tmpl.beta = 0.0f;
  const auto points = sweep(tmpl, sizes, cfgs, dev, opts);
  std::size_t failed = 0;
  for (const RooflinePoint& p : points)
    if (!p.ok) {
      ++failed;
      std::fprintf(stderr, "%s %s: %s\n", p.problem.c_str(), p.config.c_str(), p.error.c_str());
    }
  emit_report(points, ReportFormat::Csv, out);
  std::printf("%zu points (%zu failed) -> %s\n", points.size(), failed, out.c_str());
  return failed ? 1 : 0;
}

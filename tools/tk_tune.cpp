// tk_tune -- tune every distinct conv layer of VGG-16 / ResNet-50 (the
// reference's layer tables, proj/data/*.csv) over the B200 search space and
// write the NDJSON tuning DB (the reference's `tilekit tune`/`layers`
// workflow, tilekit_cli.cpp:252-437, reduced to what the hot path needs).
//
//   tk_tune vgg16|resnet50 [batch] [db.ndjson]
#include <cstdio>
#include <string>
#include <vector>

#include "tilekit/tilekit.hpp"

using namespace tilekit;

struct Layer {
  const char* name;
  std::size_t r, stride, h, c, k;
};

static const std::vector<Layer> kVgg = {
    {"vgg_conv1_1", 3, 1, 224, 3, 64},   {"vgg_conv1_2", 3, 1, 224, 64, 64},
    {"vgg_conv2_1", 3, 1, 112, 64, 128}, {"vgg_conv2_2", 3, 1, 112, 128, 128},
    {"vgg_conv3_1", 3, 1, 56, 128, 256}, {"vgg_conv3_2", 3, 1, 56, 256, 256},
    {"vgg_conv4_1", 3, 1, 28, 256, 512}, {"vgg_conv4_2", 3, 1, 28, 512, 512},
    {"vgg_conv5", 3, 1, 14, 512, 512}};
static const std::vector<Layer> kResnet = {
    {"resnet_conv1", 7, 2, 224, 3, 64},          {"res2a_branch2a", 1, 1, 56, 64, 64},
    {"res2a_branch2b", 3, 1, 56, 64, 64},        {"res2a_branch2c", 1, 1, 56, 64, 256},
    {"res2b_branch2a", 1, 1, 56, 256, 64},       {"res3a_branch2a", 1, 2, 56, 256, 128},
    {"res3a_branch2b", 3, 1, 28, 128, 128},      {"res3a_branch2c", 1, 1, 28, 128, 512},
    {"res3a_branch1", 1, 2, 56, 256, 512},       {"res3b_branch2a", 1, 1, 28, 512, 128},
    {"res4a_branch2a", 1, 2, 28, 512, 256},      {"res4a_branch2b", 3, 1, 14, 256, 256},
    {"res4a_branch2c", 1, 1, 14, 256, 1024},     {"res4a_branch1", 1, 2, 28, 512, 1024},
    {"res4b_branch2a", 1, 1, 14, 1024, 256},     {"res5a_branch2a", 1, 2, 14, 1024, 512},
    {"res5a_branch2b", 3, 1, 7, 512, 512},       {"res5a_branch2c", 1, 1, 7, 512, 2048},
    {"res5a_branch1", 1, 2, 14, 1024, 2048},     {"res5b_branch2a", 1, 1, 7, 2048, 512}};

int main(int argc, char** argv) {
  const std::string which = argc > 1 ? argv[1] : "vgg16";
  const std::size_t batch = argc > 2 ? std::stoul(argv[2]) : 32;
  const std::string db = argc > 3 ? argv[3] : which + "_tune.ndjson";
  const auto& layers = which == "resnet50" ? kResnet : kVgg;
  const DeviceSpec dev = b200_device();
  ParamSpace space;  // exact FP32: one tiled point per algorithm family
  space.tile_rows = {2, 4};
  space.tile_cols = {2, 4};
  space.channel_vectors = {4};
  space.feature_vectors = {4};
  // tensor cores: pipeline depth x cluster shape x operand path
  space.tc_stages = {0, 4};
  space.tc_clusters = {0, 1};
  space.tc_modes = {b200::TcMode::Auto, b200::TcMode::Halo, b200::TcMode::PixN,
                    b200::TcMode::PixM, b200::TcMode::Pointwise, b200::TcMode::Im2col};
  BenchOptions opts;
  opts.warmup = 2;
  opts.samples = 5;
  std::vector<TuningRecord> all;
  std::printf("%-16s %-30s %12s %10s %7s\n", "layer", "best", "GFLOP/s", "median_us", "%peak");
  for (const Layer& L : layers) {
    ConvShape s;
    s.batch = batch;
    s.in_rows = s.in_cols = L.h;
    s.channels = L.c;
    s.features = L.k;
    s.window_rows = s.window_cols = L.r;
    s.stride = L.stride;
    s.padding = Padding::Same;
    const TuneResult t = b200::tune(Problem::of(s), space, dev, opts);
    all.insert(all.end(), t.records.begin(), t.records.end());
    std::printf("%-16s %-30s %12.1f %10.1f %6.1f%%\n", L.name, t.best.config.c_str(),
                t.best.gflops, t.best.median_ns / 1e3, 100.0 * t.best.frac_of_peak);
    std::fflush(stdout);
  }
  save_db(all, db);
  std::printf("%zu records -> %s\n", all.size(), db.c_str());
  return 0;
}

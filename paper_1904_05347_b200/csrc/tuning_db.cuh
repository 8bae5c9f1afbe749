// tuning_db.cuh -- the tuning DB the library consults (lookup_best, reference
// tuner.hpp:684-694, on the launch path).
//
// tk_tuning_db_load reads the tuner's NDJSON (the reference's nine keys;
// tools/tune_ncu.py and tilekit::b200::tune write it).  A call whose
// tk_exec_options leave every tensor-core knob automatic looks up its
// (problem key, algorithm, precision); the fastest valid record's knobs
// (N tile, stages, cluster, operand path, split-K) replace the hand-written
// rules for that call.  No record: the rules.  Knobs named by the caller
// always win.
#pragma once

#include <string>

#include "tc_gemm.cuh"

namespace tkb {

struct TunedKnobs {
  int tile_n = 0, stages = 0, cluster = 0, mode = 0, split = 0;
  long long median_ns = 0;
  std::string config;
};

// Load (merge) an NDJSON DB for `device` ("" = any); returns records kept.
size_t tuning_db_load(const std::string& path, const std::string& device);
void tuning_db_clear();
size_t tuning_db_size();
// The DB's knobs for (problem, algorithm family, precision), if any.
bool tuning_db_lookup(const std::string& problem, const std::string& family, int precision,
                      TunedKnobs* out);

}  // namespace tkb

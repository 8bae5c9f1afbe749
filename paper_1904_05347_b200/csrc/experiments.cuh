// experiments.cuh -- process-wide A/B experiment knobs (NOT product knobs).
//
// Per-call tuning goes through tk_exec_options (the tuner's axes).  The
// knobs below exist only for same-box A/B measurements; the product launch
// path never reads the environment: they are read ONCE, at first use, and
// only when TK_EXPERIMENTS=1 is set -- otherwise every field keeps its
// default and a stray TK_* variable changes nothing.
#pragma once

#include <string>

namespace tkb {

struct Experiments {
  bool enabled = false;
  bool pdl = true;              // TK_PDL=0: no programmatic dependent launch
  bool tail = true;             // TK_TAIL=0: no stream-K tail
  bool tail_force = false;      // TK_TAIL_FORCE=1: take the tail wherever it applies
  double red_gbs = 4000.0;      // TK_RED_GBS: reduction-pass rate the split/tail models assume
  int pipe_chunks = 0;          // TK_PIPE_CHUNKS: max batch chunks of the host-buffer pipeline
  int pipe_min_kb = 0;          // TK_PIPE_MIN_KB: smallest chunk copy (KiB)
  int tc_stages = 0;            // TK_TC_STAGES: operand ring depth cap
  int tc_epi = 0;               // TK_TC_EPI: staging buffers cap
  bool epi_ring = true;         // TK_EPI_RING=0: whole-tile epilogue staging
  int epi_ring_n = 0;           // TK_EPI_RING_N: chunks per staging slot
  int epi_slots = 0;            // TK_EPI_SLOTS: staging slots (2..8)
  int direct_store = 0;         // TK_DIRECT_STORE=1: register -> global epilogue (narrow halo)
  int epi_groups = 0;           // TK_EPI_GROUPS: 1 or 2 epilogue warpgroups
  int tc_acc = 0;               // TK_TC_ACC: TMEM accumulator slots (2/4/8)
  int raster = 8;               // TK_RASTER: M-blocks per raster group (0 = linear)
  bool trace = false;           // TK_TC_TRACE=1: in-kernel timeline probe
  bool a_mn = true;             // TK_A_MN=0: pack a column-major A instead
  std::string conv_mode;        // TK_CONV_MODE: force an operand path
  int pw_bn = 0;                // TK_PW_BN: pixels-on-M GEMM feature tile
  bool no_split = false;        // TK_NO_SPLIT=1: no split-K on pixN
  bool tf32_round = true;       // TK_TF32_ROUND=0: truncate the TF32 filter
  int gather_cg = 1;            // TK_GATHER_CG=2: gather on SM pairs
  int halo_bn = 0;              // TK_HALO_BN: 64 / 128
  int exact_stages = 0;         // TK_EXACT_STAGES
  int exact_tile[4] = {0, 0, 0, 0};  // TK_EXACT_TILE="h,w,r,c"
};

// The knobs of this process (defaults unless TK_EXPERIMENTS=1).
const Experiments& experiments();

}  // namespace tkb

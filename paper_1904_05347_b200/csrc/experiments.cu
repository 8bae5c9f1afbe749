// experiments.cu -- one-time read of the A/B experiment knobs (see
// experiments.cuh).  Nothing else in the library calls getenv.
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "experiments.cuh"

namespace tkb {

namespace {
int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
bool env_flag(const char* name, bool dflt) {
  const char* e = std::getenv(name);
  if (!e) return dflt;
  return e[0] != '0';
}
}  // namespace

const Experiments& experiments() {
  static Experiments x;
  static std::once_flag once;
  std::call_once(once, [] {
    const char* on = std::getenv("TK_EXPERIMENTS");
    if (!(on && on[0] == '1')) return;
    x.enabled = true;
    x.pdl = env_flag("TK_PDL", true);
    x.tail = env_flag("TK_TAIL", true);
    x.tail_force = env_flag("TK_TAIL_FORCE", false);
    x.red_gbs = env_int("TK_RED_GBS", 4000);
    x.pipe_chunks = env_int("TK_PIPE_CHUNKS", 0);
    x.pipe_min_kb = env_int("TK_PIPE_MIN_KB", 0);
    x.tc_stages = env_int("TK_TC_STAGES", 0);
    x.tc_epi = env_int("TK_TC_EPI", 0);
    x.epi_ring = env_flag("TK_EPI_RING", true);
    x.epi_ring_n = env_int("TK_EPI_RING_N", 0);
    x.epi_slots = env_int("TK_EPI_SLOTS", 0);
    x.direct_store = env_int("TK_DIRECT_STORE", 0);
    x.epi_groups = env_int("TK_EPI_GROUPS", 0);
    x.tc_acc = env_int("TK_TC_ACC", 0);
    x.raster = env_int("TK_RASTER", 8);
    x.trace = env_flag("TK_TC_TRACE", false);
    x.a_mn = env_flag("TK_A_MN", true);
    if (const char* m = std::getenv("TK_CONV_MODE")) x.conv_mode = m;
    x.pw_bn = env_int("TK_PW_BN", 0);
    x.no_split = env_flag("TK_NO_SPLIT", false);
    x.tf32_round = env_flag("TK_TF32_ROUND", true);
    x.gather_cg = env_int("TK_GATHER_CG", 1) == 2 ? 2 : 1;
    x.halo_bn = env_int("TK_HALO_BN", 0);
    x.exact_stages = env_int("TK_EXACT_STAGES", 0);
    if (const char* t = std::getenv("TK_EXACT_TILE"))
      std::sscanf(t, "%d,%d,%d,%d", &x.exact_tile[0], &x.exact_tile[1], &x.exact_tile[2],
                  &x.exact_tile[3]);
    std::fprintf(stderr, "tilekit_b200: TK_EXPERIMENTS=1 -- A/B experiment knobs active\n");
  });
  return x;
}

}  // namespace tkb

// exact_gemm.cu -- instantiation table + launcher for the exact SIMT family.
#include <string>

#include "exact_gemm.cuh"
#include "exact_gen.cuh"
#include "launch_cache.cuh"

namespace tkb {

namespace {

using LocFn = void (*)(ExactArgs, int, int, int);
using NolocFn = void (*)(ExactArgs, int, int);

template <int H, int W>
LocFn pick_loc(int al, int bl, bool conv) {
  if (conv) return exact_gemm_loc_kernel<H, W, kK, kMN, true>;
  if (al == kMN && bl == kMN) return exact_gemm_loc_kernel<H, W, kMN, kMN, false>;
  if (al == kMN && bl == kK) return exact_gemm_loc_kernel<H, W, kMN, kK, false>;
  if (al == kK && bl == kMN) return exact_gemm_loc_kernel<H, W, kK, kMN, false>;
  return exact_gemm_loc_kernel<H, W, kK, kK, false>;
}

template <int H>
LocFn pick_loc_w(int w, int al, int bl, bool conv) {
  switch (w) {
    case 1: return pick_loc<H, 1>(al, bl, conv);
    case 2: return pick_loc<H, 2>(al, bl, conv);
    case 4: return pick_loc<H, 4>(al, bl, conv);
    case 8: return pick_loc<H, 8>(al, bl, conv);
  }
  return nullptr;
}

LocFn pick_loc_hw(int h, int w, int al, int bl, bool conv) {
  switch (h) {
    case 1: return pick_loc_w<1>(w, al, bl, conv);
    case 2: return pick_loc_w<2>(w, al, bl, conv);
    case 4: return pick_loc_w<4>(w, al, bl, conv);
    case 8: return pick_loc_w<8>(w, al, bl, conv);
  }
  return nullptr;
}

template <int H>
NolocFn pick_noloc_w(int w, bool conv) {
  switch (w) {
    case 1: return conv ? exact_gemm_noloc_kernel<H, 1, true> : exact_gemm_noloc_kernel<H, 1, false>;
    case 2: return conv ? exact_gemm_noloc_kernel<H, 2, true> : exact_gemm_noloc_kernel<H, 2, false>;
    case 4: return conv ? exact_gemm_noloc_kernel<H, 4, true> : exact_gemm_noloc_kernel<H, 4, false>;
    case 8: return conv ? exact_gemm_noloc_kernel<H, 8, true> : exact_gemm_noloc_kernel<H, 8, false>;
  }
  return nullptr;
}

NolocFn pick_noloc(int h, int w, bool conv) {
  switch (h) {
    case 1: return pick_noloc_w<1>(w, conv);
    case 2: return pick_noloc_w<2>(w, conv);
    case 4: return pick_noloc_w<4>(w, conv);
    case 8: return pick_noloc_w<8>(w, conv);
  }
  return nullptr;
}

// Resource check: a configuration the SM cannot host is rejected loudly
// (the paper's register/local-memory budget, measured on the real kernel).
void check_fits(const void* fn, int threads, size_t smem, const ExactLaunch& L) {
  const cudaFuncAttributes& attr = func_attrs(fn);
  const std::string name = std::to_string(L.h) + "x" + std::to_string(L.w) + "_" +
                           std::to_string(L.r) + "x" + std::to_string(L.c);
  if (threads > attr.maxThreadsPerBlock) {
    fail(TK_ERR_CONFIG, "gemm_tiled: config \"" + name + "\" rejected: register budget: kernel uses " +
                            std::to_string(attr.numRegs) + " registers/thread, " +
                            std::to_string(threads) + " threads exceed the SM register file (max " +
                            std::to_string(attr.maxThreadsPerBlock) + " threads)");
  }
  if (smem > 232448) {
    fail(TK_ERR_CONFIG, "gemm_tiled: config \"" + name + "\" rejected: local-memory budget: " +
                            std::to_string(smem) + " bytes exceeds 232448 bytes of shared memory");
  }
}

}  // namespace

// conv2d_tiled's CTA block: the pr x pc grid of tile_rows x tile_cols
// patches (pr * pc = r threads along M) that pads the output plane least.
struct PatchGrid {
  int pr = 1, pc = 1, blk_r = 1, blk_c = 1;
};
PatchGrid patch_grid(int OH, int OW, int tile_rows, int tile_cols, int r) {
  PatchGrid best_g;
  double best = 1e30;
  for (int pr = 1; pr <= r; ++pr) {
    if (r % pr) continue;
    const int pc = r / pr;
    const long long BR = (long long)tile_rows * pr, BC = (long long)tile_cols * pc;
    const long long br = (OH + BR - 1) / BR, bc = (OW + BC - 1) / BC;
    const double waste = (double)(br * BR) * (bc * BC) / ((double)OH * OW);
    if (waste < best - 1e-9) {
      best = waste;
      best_g = PatchGrid{pr, pc, (int)br, (int)bc};
    }
  }
  return best_g;
}

void launch_exact(const ExactArgs& p0, const ExactLaunch& L, bool conv, int batch,
                  cudaStream_t stream) {
  if (p0.M <= 0 || p0.N <= 0) return;
  ExactArgs p = p0;
  auto pow2 = [](int v) { return v == 1 || v == 2 || v == 4 || v == 8; };
  // 2-D patches on the tuned kernels need whole 8-thread staging groups.
  const bool patch = conv && L.tile_rows > 0 && L.loc && ((L.r * L.c) & 7) == 0;
  if (L.gen || !pow2(L.h) || !pow2(L.w) || (conv && L.tile_rows > 0 && !patch)) {
    GenLaunch G;
    G.h = L.h;
    G.w = L.w;
    G.r = L.r;
    G.c = L.c;
    G.stages = L.loc ? L.stages : 2;  // "noloc" runtime tiles are staged too (same bits)
    G.tile_rows = L.tile_rows;
    G.tile_cols = L.tile_cols;
    G.cvec = L.cvec;
    G.shrink_ok = L.shrink_ok;
    launch_exact_gen(p, G, conv, batch, stream);
    return;
  }
  const int threads = L.r * L.c;
  if (threads <= 0 || threads > 1024)
    fail(TK_ERR_CAPABILITY, "gemm_tiled: work-group of " + std::to_string(threads) +
                                " threads exceeds the B200 limit of 1024");
  const size_t BM = (size_t)L.h * L.r, BN = (size_t)L.w * L.c;
  dim3 grid((unsigned)ceil_div(p.M, BM), (unsigned)ceil_div(p.N, BN), (unsigned)batch);
  if (patch) {
    const PatchGrid g = patch_grid(p.OH, p.OW, L.tile_rows, L.tile_cols, L.r);
    p.t2_rows = L.tile_rows;
    p.t2_cols = L.tile_cols;
    p.t2_pr = g.pr;
    p.t2_pc = g.pc;
    p.t2_blk_r = g.blk_r;
    p.t2_blk_c = g.blk_c;
    grid.x = (unsigned)((long long)(p.M / ((long long)p.OH * p.OW)) * g.blk_r * g.blk_c);
  }
  if (grid.y > 65535 || grid.z > 65535)
    fail(TK_ERR_CAPABILITY, "gemm_tiled: grid too large for the chosen block shape");
  const int al = conv ? kK : (p.a_sm == 1 ? kMN : kK);
  const int bl = conv ? kMN : (p.b_sn == 1 ? kMN : kK);
  if (L.loc) {
    LocFn fn = pick_loc_hw(L.h, L.w, al, bl, conv);
    if (!fn) fail(TK_ERR_CAPABILITY, "gemm_tiled: register tile must be h,w in {1,2,4,8}");
    const int stages = L.stages < 1 ? 1 : (L.stages > 3 ? 3 : L.stages);
    const size_t words = (size_t)(al == kMN ? kExactBK * (BM + 4) : BM * (kExactBK + 4)) +
                         (size_t)(bl == kMN ? kExactBK * (BN + 4) : BN * (kExactBK + 4));
    const size_t smem =
        words * 4 * stages + (conv ? BM * (sizeof(PixRow) + sizeof(long long)) : 0);  // + pixel tables
    check_fits((const void*)fn, threads, smem, L);
    if (smem > 48 * 1024) func_smem((const void*)fn, smem);
    fn<<<grid, threads, smem, stream>>>(p, L.r, L.c, stages);
  } else {
    NolocFn fn = pick_noloc(L.h, L.w, conv);
    if (!fn) fail(TK_ERR_CAPABILITY, "gemm_tiled: register tile must be h,w in {1,2,4,8}");
    check_fits((const void*)fn, threads, 0, L);
    fn<<<grid, threads, 0, stream>>>(p, L.r, L.c);
  }
  note_launch();
  TKB_CUDA(cudaGetLastError());
}

}  // namespace tkb

// ---------------------------------------------------------------------------
// Runtime register tile (exact_gen.cuh).
// ---------------------------------------------------------------------------

namespace tkb {

namespace {

using GenFn = void (*)(ExactArgs, GenGeom, int, int, int);

template <int HM, int WM, bool SMALL>
GenFn pick_gen_s(int al, int bl, bool conv) {
  if (conv) return exact_gemm_gen_kernel<HM, WM, kK, kMN, true, SMALL>;
  if (al == kMN && bl == kMN) return exact_gemm_gen_kernel<HM, WM, kMN, kMN, false, SMALL>;
  if (al == kMN && bl == kK) return exact_gemm_gen_kernel<HM, WM, kMN, kK, false, SMALL>;
  if (al == kK && bl == kMN) return exact_gemm_gen_kernel<HM, WM, kK, kMN, false, SMALL>;
  return exact_gemm_gen_kernel<HM, WM, kK, kK, false, SMALL>;
}

// The small-work-group build (two CTAs per SM) whenever the work-group fits.
thread_local bool g_gen_small = true;
template <int HM, int WM>
GenFn pick_gen(int al, int bl, bool conv) {
  return g_gen_small ? pick_gen_s<HM, WM, true>(al, bl, conv) : pick_gen_s<HM, WM, false>(al, bl, conv);
}

// Compile-time bounds of the accumulator block (64 outputs each); wider or
// taller logical tiles are split over several GPU threads by the launcher.
constexpr int kGenVariants[4][2] = {{8, 8}, {16, 4}, {4, 16}, {32, 2}};

GenFn gen_variant(int v, int al, int bl, bool conv) {
  switch (v) {
    case 0: return pick_gen<8, 8>(al, bl, conv);
    case 1: return pick_gen<16, 4>(al, bl, conv);
    case 2: return pick_gen<4, 16>(al, bl, conv);
    default: return pick_gen<32, 2>(al, bl, conv);
  }
}

int fit_variant(int h, int w) {
  for (int v = 0; v < 4; ++v)
    if (h <= kGenVariants[v][0] && w <= kGenVariants[v][1]) return v;
  return -1;
}

}  // namespace

void launch_exact_gen(const ExactArgs& p, const GenLaunch& L0, bool conv, int batch,
                      cudaStream_t stream) {
  if (p.M <= 0 || p.N <= 0) return;
  GenLaunch L = L0;
  if (L.h < 1 || L.w < 1 || L.r < 1 || L.c < 1)
    fail(TK_ERR_CONFIG, "gemm_tiled: register tile and work-group must be >= 1");
  // A logical thread whose tile fits no variant runs as several GPU threads
  // (same CTA tile h*r x w*c, same per-output sums).
  if (L.tile_rows > 0 && L.h > 32) L.tile_rows = L.tile_cols = 0;
  while (fit_variant(L.h, L.w) < 0) {
    if (L.h >= L.w) {
      L.h = (L.h + 1) / 2;
      L.r *= 2;
    } else {
      L.w = (L.w + 1) / 2;
      L.c *= 2;
    }
    L.tile_rows = L.tile_cols = 0;  // the patch no longer matches one thread
  }
  const int al = conv ? kK : (p.a_sm == 1 ? kMN : kK);
  const int bl = conv ? kMN : (p.b_sn == 1 ? kMN : kK);
  if (L.shrink_ok && L.r * L.c > 256) L.r = std::max(1, 256 / L.c);
  g_gen_small = L.r * L.c <= 256;
  const GenFn fn = gen_variant(fit_variant(L.h, L.w), al, bl, conv);
  const cudaFuncAttributes& attr = func_attrs((const void*)fn);
  if (L.shrink_ok && L.r * L.c > attr.maxThreadsPerBlock)
    L.r = std::max(1, attr.maxThreadsPerBlock / L.c);  // (the patch grid follows r below)
  const int threads = L.r * L.c;
  if (threads > 1024)
    fail(TK_ERR_CAPABILITY, "gemm_tiled: work-group of " + std::to_string(threads) +
                                " GPU threads exceeds the B200 limit of 1024");
  GenGeom q{};
  q.h = L.h;
  q.w = L.w;
  q.cvec = L.cvec == 1 || L.cvec == 2 ? L.cvec : 4;
  const size_t BM = (size_t)L.h * L.r, BN = (size_t)L.w * L.c;
  unsigned gx = (unsigned)ceil_div(p.M, BM);
  if (conv && L.tile_rows > 0) {
    const PatchGrid g = patch_grid(p.OH, p.OW, L.tile_rows, L.tile_cols, L.r);
    q.tile_rows = L.tile_rows;
    q.tile_cols = L.tile_cols;
    q.pr = g.pr;
    q.pc = g.pc;
    q.blk_r = g.blk_r;
    q.blk_c = g.blk_c;
    gx = (unsigned)((long long)(p.M / ((long long)p.OH * p.OW)) * g.blk_r * g.blk_c);
  }
  dim3 grid(gx, (unsigned)ceil_div(p.N, BN), (unsigned)batch);
  if (grid.y > 65535 || grid.z > 65535)
    fail(TK_ERR_CAPABILITY, "gemm_tiled: grid too large for the chosen block shape");
  int stages = L.stages < 1 ? 1 : (L.stages > 3 ? 3 : L.stages);
  const size_t words = (size_t)(al == kMN ? kExactBK * (BM + 4) : BM * (kExactBK + 4)) +
                       (size_t)(bl == kMN ? kExactBK * (BN + 4) : BN * (kExactBK + 4));
  const size_t table = conv ? BM * sizeof(GenRow) : 0;
  while (stages > 1 && words * 4 * stages + table > 232448) --stages;  // shallower ring first
  const size_t smem = words * 4 * stages + table;
  if (smem > 232448)
    fail(TK_ERR_CONFIG, "gemm_tiled: config rejected: local-memory budget: " + std::to_string(smem) +
                            " bytes exceeds 232448 bytes of shared memory");
  if (threads > attr.maxThreadsPerBlock)
    fail(TK_ERR_CONFIG, "gemm_tiled: config rejected: register budget: kernel uses " +
                            std::to_string(attr.numRegs) + " registers/thread, " +
                            std::to_string(threads) + " threads exceed the SM register file");
  if (smem > 48 * 1024) func_smem((const void*)fn, smem);
  fn<<<grid, threads, smem, stream>>>(p, q, L.r, L.c, stages);
  note_launch();
  TKB_CUDA(cudaGetLastError());
}

}  // namespace tkb

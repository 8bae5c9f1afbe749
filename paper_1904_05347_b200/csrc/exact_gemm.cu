// exact_gemm.cu -- instantiation table + launcher for the exact SIMT family.
#include <string>

#include "exact_gemm.cuh"
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

void launch_exact(const ExactArgs& p, const ExactLaunch& L, bool conv, int batch,
                  cudaStream_t stream) {
  if (p.M <= 0 || p.N <= 0) return;
  const int threads = L.r * L.c;
  if (threads <= 0 || threads > 1024)
    fail(TK_ERR_CAPABILITY, "gemm_tiled: work-group of " + std::to_string(threads) +
                                " threads exceeds the B200 limit of 1024");
  const size_t BM = (size_t)L.h * L.r, BN = (size_t)L.w * L.c;
  dim3 grid((unsigned)ceil_div(p.M, BM), (unsigned)ceil_div(p.N, BN), (unsigned)batch);
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
    const size_t smem = words * 4 * stages + (conv ? BM * 16 : 0);  // + pixel table
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

// tc_gemm.cuh -- tensor-core (tcgen05 / TMEM / TMA) GEMM and implicit-GEMM
// convolution launchers.
#pragma once

#include <cuda_runtime.h>

#include "layout.cuh"

namespace tkb {

// What a tensor-core GEMM call runs (tk_gemm_plan_info): filled instead of
// launching when TcGemm::plan / the colmajor launcher's plan is non-null.
struct TcGemmPlan {
  int precision = 0;       // the MMA kind (TF32 for 3xTF32's tripled contraction)
  int cta_group = 1, tile_m = 0, tile_n = 0, splits = 1, tail_pieces = 0;
  int a_in_place = 0, b_in_place = 0;  // operands read where they lie (no pack)
  int k_depth = 0;         // contraction depth the MMAs run (3 kp for 3xTF32)
};

// Row-major batched GEMM on tensor cores:
//   D(m, n) = alpha * sum_k A[m][k] * B[n][k] (+ beta * C(m, n))
// A is [M][K], B is [N][K] (both K contiguous, K % 4 == 0), D(m, n) lives at
// d[z*d_batch + m*d_sm + n*d_sn] (C likewise).  d_sm == 1 gives coalesced
// stores.
struct TcGemm {
  int M = 0, N = 0, K = 0, batch = 1;
  const float* a = nullptr;
  long long a_batch = 0;
  const float* b = nullptr;
  long long b_batch = 0;
  float* d = nullptr;
  const float* c = nullptr;
  long long d_sm = 1, d_sn = 0, d_batch = 0;
  float alpha = 1.0f, beta = 0.0f;
  int precision = 1;
  int tile_n = 0;  // 0 = auto
  // TF32, batch 1: A given MN-major instead -- column-major [K][lda] with M
  // contiguous (M % 32 == 0), read by the tensor core as is (no transpose).
  bool a_mn = false;
  long long lda = 0;
  // MN-major A: its true K extent (K may be padded for B); the TMA zero-fills
  // past it instead of reading beyond the end of A.  0 = K.
  long long a_k = 0;
  TcGemmPlan* plan = nullptr;  // dry run: fill the plan, launch nothing
};

void launch_tc_gemm(const TcGemm& g, cudaStream_t st);

// 3xTF32 operand expansion: rows x [kp] K-major fp32 -> rows x [3 kp];
// pattern 0 = (x, x, x_lo) (the A side), 1 = (x_hi, x_lo, x_hi) (the B side):
// one TF32 contraction of depth 3 kp then sums a_hi b_hi + a_hi b_lo + a_lo b_hi.
void launch_split3_rows(const float* src, long long rows, long long kp, float* dst, int pattern,
                        cudaStream_t st);

// Per-call tensor-core knobs (tk_exec_options.tc_stages / tc_cluster /
// tc_mode / tc_split), set by the C ABI for the duration of one call on the
// calling thread; zero = automatic.
struct TcKnobs {
  int stages = 0, cluster = 0, mode = 0, split = 0;
  int io = 0;  // TK_IO_* (bf16 activations in HBM; BF16 tensor-core convs only)
};
TcKnobs& tc_knobs();

// Column-major C = alpha*OPa(A)*OPb(B) + beta*C (the reference GemmShape
// convention) on tensor cores; transposes operands into K-major scratch
// where needed.
void launch_tc_colmajor_gemm(size_t m, size_t n, size_t k, float alpha, float beta, bool ta,
                             bool tb, const float* a, const float* b, const float* c, float* d,
                             int precision, int tile_n, cudaStream_t st,
                             TcGemmPlan* plan = nullptr);

// Batched column-major C_g = A_g B_g (C zeroed: beta 0), g < batch, operand
// strides in elements (the reference gemm_batched_strided, gemm.hpp:451-479)
// on tensor cores: A_g packed K-major for all g, B_g read in place when it
// already is (TF32, k % 4 == 0), one batched launch; 3xTF32 per member.
void launch_tc_batched_colmajor(size_t m, size_t n, size_t k, size_t batch, const float* a,
                                long long sa, const float* b, long long sb, float* d, long long sc,
                                int precision, cudaStream_t st);

// Implicit-GEMM convolution on tensor cores (NHWC in, HWCK filter, NHWC
// out).  Workspace: packed filter (+ patch matrix on the fallback path).
size_t tc_conv_workspace(const ConvGeom& g, int precision);
// phase: kConvPrepare packs the filter into the workspace (depends only on
// the filter), kConvRun runs the convolution from a prepared workspace.
constexpr int kConvPrepare = 1, kConvRun = 2, kConvAll = 3;
// What launch_tc_conv will run for this geometry and precision request
// (tk_conv2d_plan_info): operand path, the precision the tensor cores
// actually compute in, tile and work split.
struct TcConvInfo {
  int mode = 0;        // enum tk_tc_mode of the operand path
  bool narrow = false; // halo over 16-byte padded pixels (TK_KERNEL_TC_HALO_NARROW)
  int precision = 0;   // effective enum tk_precision
  int cta_group = 1, tile_m = 0, tile_n = 0, splits = 1, tail_pieces = 0;
  int imgs = 1, flat = 0, box_w = 0, box_h = 0, halo_resident = 0;
};
TcConvInfo tc_conv_info(const ConvGeom& g, int precision);
void launch_tc_conv(const ConvGeom& g, const float* in, const float* filt, float* out,
                    int precision, void* ws, cudaStream_t st, int phase = kConvAll);

}  // namespace tkb

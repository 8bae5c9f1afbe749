// tilekit/winograd.hpp -- fast convolution and the conv2d selector.
//
// Reference: winograd.hpp (WinogradPlan :21-32, winograd_plan :50-119,
// WinogradStats :152-155, conv2d_winograd :169-301, conv2d :304-314).
// The transforms run as coalesced HBM-bound kernels and the transform-domain
// products as one batched GEMM on the B200; in FP32 the result is
// bit-identical to the reference (same transform arithmetic, ascending-
// channel sums).
#pragma once

#include <cstddef>
#include <cstdint>
#include <initializer_list>
#include <string>

#include "tilekit/b200.hpp"
#include "tilekit/config.hpp"
#include "tilekit/conv.hpp"
#include "tilekit/errors.hpp"
#include "tilekit/tensor.hpp"

namespace tilekit {

// Cook-Toom matrices for an M x N output tile under an R x S window:
// input_transform = B^T, filter_transform = G, output_transform = A^T.
struct WinogradPlan {
  std::size_t out_tile_rows = 0;
  std::size_t out_tile_cols = 0;
  std::size_t window_rows = 0;
  std::size_t window_cols = 0;
  Matrix input_transform;   // (M+R-1) x (M+R-1)
  Matrix filter_transform;  // (M+R-1) x R
  Matrix output_transform;  // M x (M+R-1)

  std::size_t input_tile_rows() const { return out_tile_rows + window_rows - 1; }
  std::size_t input_tile_cols() const { return out_tile_cols + window_cols - 1; }
};

namespace detail {

// Row-major initializer -> column-major Matrix.
inline Matrix rows_to_matrix(std::size_t rows, std::size_t cols,
                             std::initializer_list<float> values) {
  Matrix m(rows, cols);
  std::size_t idx = 0;
  for (float v : values) {
    m(idx / cols, idx % cols) = v;
    ++idx;
  }
  return m;
}

}  // namespace detail

// F(2x2,3x3) and F(4x4,3x3); anything else is a CapabilityError.
inline WinogradPlan winograd_plan(std::size_t out_tile_rows, std::size_t out_tile_cols,
                                  std::size_t window_rows, std::size_t window_cols) {
  WinogradPlan plan;
  plan.out_tile_rows = out_tile_rows;
  plan.out_tile_cols = out_tile_cols;
  plan.window_rows = window_rows;
  plan.window_cols = window_cols;
  const bool w3 = window_rows == 3 && window_cols == 3;
  if (w3 && out_tile_rows == 2 && out_tile_cols == 2) {
    plan.input_transform = detail::rows_to_matrix(4, 4, {1, 0, -1, 0,  //
                                                         0, 1, 1, 0,   //
                                                         0, -1, 1, 0,  //
                                                         0, 1, 0, -1});
    plan.filter_transform = detail::rows_to_matrix(4, 3, {1, 0, 0,           //
                                                          0.5f, 0.5f, 0.5f,  //
                                                          0.5f, -0.5f, 0.5f, //
                                                          0, 0, 1});
    plan.output_transform = detail::rows_to_matrix(2, 4, {1, 1, 1, 0,  //
                                                          0, 1, -1, -1});
    return plan;
  }
  if (w3 && out_tile_rows == 4 && out_tile_cols == 4) {
    plan.input_transform = detail::rows_to_matrix(6, 6, {4, 0, -5, 0, 1, 0,    //
                                                         0, -4, -4, 1, 1, 0,   //
                                                         0, 4, -4, -1, 1, 0,   //
                                                         0, -2, -1, 2, 1, 0,   //
                                                         0, 2, -1, -2, 1, 0,   //
                                                         0, 4, 0, -5, 0, 1});
    const float q = 1.0f / 4, s6 = 1.0f / 6, s12 = 1.0f / 12, s24 = 1.0f / 24;
    plan.filter_transform = detail::rows_to_matrix(6, 3, {q, 0, 0,          //
                                                          -s6, -s6, -s6,    //
                                                          -s6, s6, -s6,     //
                                                          s24, s12, s6,     //
                                                          s24, -s12, s6,    //
                                                          0, 0, 1});
    plan.output_transform = detail::rows_to_matrix(4, 6, {1, 1, 1, 1, 1, 0,    //
                                                          0, 1, -1, 2, -2, 0,  //
                                                          0, 1, 1, 4, 4, 0,    //
                                                          0, 1, -1, 8, -8, 1});
    return plan;
  }
  throw CapabilityError("winograd_plan: no transform set for a " + std::to_string(out_tile_rows) +
                        "x" + std::to_string(out_tile_cols) + " output tile under a " +
                        std::to_string(window_rows) + "x" + std::to_string(window_cols) +
                        " window (supported: 2x2 and 4x4 under 3x3)");
}

struct WinogradStats {
  std::uint64_t batched_multiplies = 0;  // scalar multiplies of the GEMM stage
  std::size_t tiles = 0;                 // output tiles over the batch
};

// Stride-1 fast convolution: input transform -> filter transform ->
// batched GEMM over the (M+R-1)(N+S-1) transform spots -> output
// transform.  Within 1e-3 of conv2d_naive under max_scaled_error.
inline Tensor4 conv2d_winograd(const Tensor4& input, const Tensor4& filter,
                               const ConvShape& shape, const ConvAlgoParams& params,
                               WinogradStats* stats = nullptr) {
  detail::check_conv_operands(input, filter, shape);
  Tensor4 out = detail::conv_output(shape);
  const tk_conv_shape s = detail::to_c(shape);
  const tk_conv_params p = detail::to_c(params);
  std::uint64_t mults = 0;
  std::size_t tiles = 0;
  detail::check_status(tk_conv2d_winograd(&s, &p, input.data.data(), filter.data.data(),
                                          out.data.data(), &mults, &tiles));
  if (stats) {
    stats->batched_multiplies = mults;
    stats->tiles = tiles;
  }
  return out;
}

// Algorithm dispatch by parameter set.
inline Tensor4 conv2d(const Tensor4& input, const Tensor4& filter, const ConvShape& shape,
                      const ConvAlgoParams& params) {
  switch (params.algo) {
    case ConvAlgo::Naive: return conv2d_naive(input, filter, shape);
    case ConvAlgo::Tiled: return conv2d_tiled(input, filter, shape, params);
    case ConvAlgo::Im2col: return conv2d_im2col(input, filter, shape);
    case ConvAlgo::Winograd: return conv2d_winograd(input, filter, shape, params);
  }
  throw ContractError("conv2d: unknown algorithm");
}

namespace b200 {

// conv2d with B200 execution options (precision etc.) on host tensors.
inline Tensor4 conv2d(const Tensor4& input, const Tensor4& filter, const ConvShape& shape,
                      const ConvAlgoParams& params, const ExecOptions& opts) {
  tilekit::detail::check_conv_operands(input, filter, shape);
  Tensor4 out = tilekit::detail::conv_output(shape);
  const tk_conv_shape s = tilekit::detail::to_c(shape);
  const tk_conv_params p = tilekit::detail::to_c(params);
  const tk_exec_options o = opts.c();
  tilekit::detail::check_status(
      tk_conv2d_ex(&s, &p, &o, input.data.data(), filter.data.data(), out.data.data()));
  return out;
}

}  // namespace b200
}  // namespace tilekit

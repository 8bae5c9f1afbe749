// tilekit/conv.hpp -- convolution entry points of the drop-in API.
//
// Reference: conv.hpp (conv_flops :19-23, operand checks :27-66,
// conv2d_naive :74-113, tiled_input_footprint :116-128, conv2d_tiled
// :136-248, im2col :255-300, filter_matrix :304-317, conv2d_im2col
// :320-362).  All arithmetic runs on the B200; the FP32 paths are
// bit-identical to conv2d_naive.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

#include "tilekit/b200.hpp"
#include "tilekit/config.hpp"
#include "tilekit/device.hpp"
#include "tilekit/errors.hpp"
#include "tilekit/gemm.hpp"
#include "tilekit/tensor.hpp"

namespace tilekit {

// Direct-convolution multiply-add count (2 flops each); the work figure
// every algorithm's GFLOP/s is quoted against, Winograd included.
inline std::uint64_t conv_flops(const ConvShape& s) {
  return std::uint64_t{2} * s.batch * s.out_rows() * s.out_cols() * s.features * s.window_rows *
         s.window_cols * s.channels;
}

namespace detail {

inline std::string dims4(std::size_t a, std::size_t b, std::size_t c, std::size_t d) {
  return std::to_string(a) + "x" + std::to_string(b) + "x" + std::to_string(c) + "x" +
         std::to_string(d);
}

inline void check_conv_operands(const Tensor4& input, const Tensor4& filter,
                                const ConvShape& s) {
  if (input.layout != Tensor4Layout::InputNhwc)
    throw ShapeError("conv2d: input tensor must use the NHWC layout");
  if (filter.layout != Tensor4Layout::FilterHwck)
    throw ShapeError("conv2d: filter tensor must use the HWCK layout");
  if (input.dim0 != s.batch || input.dim1 != s.in_rows || input.dim2 != s.in_cols ||
      input.dim3 != s.channels)
    throw ShapeError("conv2d: input is " + dims4(input.dim0, input.dim1, input.dim2, input.dim3) +
                     ", expected " + dims4(s.batch, s.in_rows, s.in_cols, s.channels));
  if (filter.dim0 != s.window_rows || filter.dim1 != s.window_cols || filter.dim2 != s.channels ||
      filter.dim3 != s.features)
    throw ShapeError("conv2d: filter is " +
                     dims4(filter.dim0, filter.dim1, filter.dim2, filter.dim3) + ", expected " +
                     dims4(s.window_rows, s.window_cols, s.channels, s.features));
  if (s.stride == 0) throw ShapeError("conv2d: stride must be >= 1");
  if (s.out_rows() == 0 || s.out_cols() == 0)
    throw ShapeError("conv2d: window " + std::to_string(s.window_rows) + "x" +
                     std::to_string(s.window_cols) + " does not fit the " +
                     std::to_string(s.in_rows) + "x" + std::to_string(s.in_cols) + " input");
}

inline Tensor4 conv_output(const ConvShape& s) {
  return Tensor4(Tensor4Layout::InputNhwc, s.batch, s.out_rows(), s.out_cols(), s.features);
}

}  // namespace detail

// Seven-loop reference semantics: ascending (x, y, c) per output element,
// out-of-range taps contribute nothing.
inline Tensor4 conv2d_naive(const Tensor4& input, const Tensor4& filter, const ConvShape& shape) {
  detail::check_conv_operands(input, filter, shape);
  Tensor4 out = detail::conv_output(shape);
  const tk_conv_shape s = detail::to_c(shape);
  detail::check_status(
      tk_conv2d_naive(&s, input.data.data(), filter.data.data(), out.data.data()));
  return out;
}

// Input rows x cols read by one tile_rows x tile_cols output tile.
struct TileFootprint {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::size_t elems(std::size_t channels) const { return rows * cols * channels; }
};

inline TileFootprint tiled_input_footprint(const ConvAlgoParams& p, const ConvShape& s) {
  return TileFootprint{(p.tile_rows - 1) * s.stride + s.window_rows,
                       (p.tile_cols - 1) * s.stride + s.window_cols};
}

// Register-tiled direct convolution: each thread owns tile_rows x
// tile_cols output positions x feature_vector features.  Stride 1 or 2.
inline Tensor4 conv2d_tiled(const Tensor4& input, const Tensor4& filter, const ConvShape& shape,
                            const ConvAlgoParams& params) {
  detail::check_conv_operands(input, filter, shape);
  Tensor4 out = detail::conv_output(shape);
  const tk_conv_shape s = detail::to_c(shape);
  const tk_conv_params p = detail::to_c(params);
  detail::check_status(
      tk_conv2d_tiled(&s, &p, input.data.data(), filter.data.data(), out.data.data()));
  return out;
}

// Column-major patch matrix (N*OH*OW) x (R*S*C), zero outside the input.
inline Matrix im2col(const Tensor4& input, const ConvShape& shape) {
  if (input.layout != Tensor4Layout::InputNhwc)
    throw ShapeError("im2col: input tensor must use the NHWC layout");
  if (input.dim0 != shape.batch || input.dim1 != shape.in_rows || input.dim2 != shape.in_cols ||
      input.dim3 != shape.channels)
    throw ShapeError("im2col: input does not match the stated shape");
  Matrix patches(shape.out_rows() * shape.out_cols() * shape.batch,
                 shape.window_rows * shape.window_cols * shape.channels);
  const tk_conv_shape s = detail::to_c(shape);
  detail::check_status(tk_im2col(&s, input.data.data(), patches.data.data()));
  return patches;
}

// HWCK filter as the column-major (R*S*C) x K GEMM operand.
inline Matrix filter_matrix(const Tensor4& filter) {
  if (filter.layout != Tensor4Layout::FilterHwck)
    throw ShapeError("filter_matrix: filter tensor must use the HWCK layout");
  Matrix f(filter.dim0 * filter.dim1 * filter.dim2, filter.dim3);
  detail::check_status(tk_filter_matrix(filter.dim0, filter.dim1, filter.dim2, filter.dim3,
                                        filter.data.data(), f.data.data()));
  return f;
}

// Convolution as one GEMM over the patch matrix, with an explicit GEMM
// config and device budget (validated like gemm_tiled).  The B200 path
// gathers patches implicitly instead of materialising them.
inline Tensor4 conv2d_im2col(const Tensor4& input, const Tensor4& filter, const ConvShape& shape,
                             const GemmConfig& cfg, const DeviceSpec& dev) {
  detail::check_conv_operands(input, filter, shape);
  Tensor4 out = detail::conv_output(shape);
  const tk_conv_shape s = detail::to_c(shape);
  const tk_gemm_config g = detail::to_c(cfg);
  const tk_device_spec d = detail::to_c(dev);
  detail::check_status(
      tk_conv2d_im2col(&s, &g, &d, input.data.data(), filter.data.data(), out.data.data()));
  return out;
}

// Default overload: the reference's 4x4_8x8_noloc on a generic 64-byte-line
// device without local memory (conv.hpp:353-362).
inline Tensor4 conv2d_im2col(const Tensor4& input, const Tensor4& filter, const ConvShape& shape) {
  DeviceSpec generic;
  generic.name = "generic";
  generic.cache_line_bytes = 64;
  generic.local_memory_bytes = 0;
  generic.compute_units = 1;
  return conv2d_im2col(input, filter, shape, parse_gemm_config("4x4_8x8_noloc"), generic);
}

}  // namespace tilekit

// tilekit/b200.hpp -- the B200 extension of the drop-in API.
//
// The reference structs stay exactly as they are; everything that only
// makes sense on the GPU (precision, tensor-core tile, pipeline depth,
// device-resident buffers) is here.  Also holds the struct conversions to
// the C ABI (tk_b200.h) used by the other headers.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

#include "tilekit/config.hpp"
#include "tilekit/device.hpp"
#include "tilekit/errors.hpp"
#include "tk_b200.h"

namespace tilekit {
namespace b200 {

enum class Precision {
  Fp32Exact = TK_PREC_FP32_EXACT,  // bit-identical to the reference
  Tf32 = TK_PREC_TF32,             // tcgen05 kind::tf32
  Bf16 = TK_PREC_BF16,             // tcgen05 kind::f16 with bf16 operands
  Tf32x3 = TK_PREC_3XTF32,         // split-precision TF32
};

// Tensor-core convolution operand path (tk_tc_mode).
enum class TcMode {
  Auto = TK_TC_AUTO,
  Halo = TK_TC_HALO,
  PixN = TK_TC_PIXN,
  PixM = TK_TC_PIXM,
  Gather = TK_TC_GATHER,
  Pointwise = TK_TC_POINTWISE,
  Im2col = TK_TC_IM2COL,
};

struct ExecOptions {
  Precision precision = Precision::Fp32Exact;
  int tc_tile_n = 0;   // GEMM N tile, 0 = auto
  int tc_stages = 0;   // shared-memory ring depth, 0 = auto
  int tc_cluster = 0;  // 1 = one SM, 2 = CTA pair, 0 = auto
  TcMode tc_mode = TcMode::Auto;
  int tc_split = 0;    // 0 = cost model, 1 = never split K, n > 1 = n splits
  int io = TK_IO_FP32; // TK_IO_IN_BF16 | TK_IO_OUT_BF16: bf16 activations in HBM
                       // (BF16 im2col convs on device buffers; see tk_b200.h)

  tk_exec_options c() const {
    tk_exec_options o{};
    o.precision = static_cast<int>(precision);
    o.tc_tile_n = tc_tile_n;
    o.tc_stages = tc_stages;
    o.tc_cluster = tc_cluster;
    o.tc_mode = static_cast<int>(tc_mode);
    o.tc_split = tc_split;
    o.io = io;
    return o;
  }

  // Config-name suffix of the non-default knobs, e.g. "_n128_s4_c1_halo".
  std::string suffix() const {
    static const char* modes[] = {"", "_halo", "_pixn", "_pixm", "_gather", "_pointwise", "_im2col"};
    std::string s;
    if (tc_tile_n) s += "_n" + std::to_string(tc_tile_n);
    if (tc_stages) s += "_s" + std::to_string(tc_stages);
    if (tc_cluster) s += "_c" + std::to_string(tc_cluster);
    s += modes[static_cast<int>(tc_mode)];
    if (tc_split == 1) s += "_nosplit";
    else if (tc_split > 1) s += "_k" + std::to_string(tc_split);
    return s;
  }
};

inline std::string precision_name(Precision p) {
  switch (p) {
    case Precision::Fp32Exact: return "fp32";
    case Precision::Tf32: return "tf32";
    case Precision::Bf16: return "bf16";
    case Precision::Tf32x3: return "3xtf32";
  }
  return "unknown";
}

// Number of usable B200 (sm_100) devices.
inline int device_count() { return tk_device_count(); }

}  // namespace b200

namespace detail {

inline tk_gemm_shape to_c(const GemmShape& s) {
  tk_gemm_shape o{};
  o.m = s.m;
  o.n = s.n;
  o.k = s.k;
  o.alpha = s.alpha;
  o.beta = s.beta;
  o.op_a = s.op_a == Op::Transpose;
  o.op_b = s.op_b == Op::Transpose;
  return o;
}

inline tk_gemm_config to_c(const GemmConfig& c) {
  tk_gemm_config o{};
  o.reg_rows = c.reg_rows;
  o.reg_cols = c.reg_cols;
  o.wg_rows = c.wg_rows;
  o.wg_cols = c.wg_cols;
  o.use_local_memory = c.use_local_memory;
  o.double_buffer = c.double_buffer;
  o.k_step = c.k_step;
  return o;
}

// The returned struct borrows d.name; keep d alive while it is used.
inline tk_device_spec to_c(const DeviceSpec& d) {
  tk_device_spec o{};
  o.name = d.name.c_str();
  o.cache_line_bytes = d.cache_line_bytes;
  o.local_memory_bytes = d.local_memory_bytes;
  o.compute_units = d.compute_units;
  o.register_budget = d.register_budget;
  o.max_workgroup_size = d.max_workgroup_size;
  return o;
}

inline tk_conv_shape to_c(const ConvShape& s) {
  tk_conv_shape o{};
  o.batch = s.batch;
  o.in_rows = s.in_rows;
  o.in_cols = s.in_cols;
  o.channels = s.channels;
  o.features = s.features;
  o.window_rows = s.window_rows;
  o.window_cols = s.window_cols;
  o.stride = s.stride;
  o.padding = s.padding == Padding::Same ? 1 : 0;
  return o;
}

inline tk_conv_params to_c(const ConvAlgoParams& p) {
  tk_conv_params o{};
  o.algo = static_cast<int>(p.algo);
  o.tile_rows = p.tile_rows;
  o.tile_cols = p.tile_cols;
  o.channel_vector = p.channel_vector;
  o.feature_vector = p.feature_vector;
  return o;
}

}  // namespace detail
}  // namespace tilekit

// tilekit/gemm.hpp -- GEMM entry points of the drop-in API.
//
// Signatures and validation semantics follow the reference gemm.hpp
// (reuse model :22-62, local_mem_elems :71-80, validate_config :103-146,
// gemm_naive :194-213, gemm_tiled :308-445, gemm_batched_strided :451-479).
// The arithmetic runs on the B200 through tk_b200.h; the FP32 path is
// bit-identical to the reference (ascending-k FMUL+FADD).
// Host logic (operand checks, budget verdicts) stays here, inline, and is
// also what the C ABI itself uses, so both boundaries reject the same
// inputs with the same messages.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "tilekit/b200.hpp"
#include "tilekit/config.hpp"
#include "tilekit/device.hpp"
#include "tilekit/errors.hpp"
#include "tilekit/tensor.hpp"

namespace tilekit {

// ---- reuse / traffic model (Eq. 3 of the paper) -----------------------

struct ReuseReport {
  double reuse = 0.0;
  std::uint64_t flops = 0;
  std::uint64_t elements_loaded = 0;
};

// 2 m'n'k' flops over m'k' + k'n' loads: reuse 2m'n'/(m'+n'), k'-free.
inline ReuseReport data_reuse(std::size_t block_rows, std::size_t block_cols, std::size_t depth) {
  if (block_rows == 0 || block_cols == 0 || depth == 0)
    throw ContractError("data_reuse: block dimensions must be >= 1");
  ReuseReport r;
  r.flops = std::uint64_t{2} * block_rows * block_cols * depth;
  r.elements_loaded = std::uint64_t{depth} * (block_rows + block_cols);
  r.reuse = static_cast<double>(r.flops) / static_cast<double>(r.elements_loaded);
  return r;
}

struct BlockTraffic {
  std::uint64_t flops = 0;
  std::uint64_t elements = 0;
};

// One m' x n' output block over the whole depth K.
inline BlockTraffic block_traffic(const GemmShape& shape, std::size_t block_rows,
                                  std::size_t block_cols) {
  BlockTraffic t;
  t.flops = std::uint64_t{2} * shape.k * block_rows * block_cols;
  t.elements = std::uint64_t{block_rows} * block_cols +
               std::uint64_t{shape.k} * (block_rows + block_cols);
  return t;
}

// ---- budgets -------------------------------------------------------------

// Staged elements: an (h*r) x X slab of A plus an X x (w*c) slab of B,
// doubled with double buffering; X = elements per cache line.
inline std::size_t local_mem_elems(const GemmConfig& cfg, const DeviceSpec& dev) {
  if (!cfg.use_local_memory)
    throw ContractError("local_mem_elems: config \"" + cfg.name() +
                        "\" does not use local memory");
  const std::size_t x = dev.elems_per_cache_line();
  const std::size_t one = x * (cfg.block_rows() + cfg.block_cols());
  return cfg.double_buffer ? 2 * one : one;
}

struct ConfigVerdict {
  bool ok = true;
  std::vector<std::string> violations;

  std::string summary() const {
    if (ok) return "valid";
    std::string joined;
    for (std::size_t i = 0; i < violations.size(); ++i)
      joined += (i ? "; " : "") + violations[i];
    return joined;
  }
};

// Every violated budget is reported, not only the first.
inline ConfigVerdict validate_config(const GemmConfig& cfg, const DeviceSpec& dev,
                                     [[maybe_unused]] const GemmShape& shape) {
  ConfigVerdict v;
  auto reject = [&v](std::string why) {
    v.ok = false;
    v.violations.push_back(std::move(why));
  };
  const std::size_t threads = cfg.workgroup_size();
  if (threads > dev.max_workgroup_size)
    reject("work-group budget: " + std::to_string(cfg.wg_rows) + "x" +
           std::to_string(cfg.wg_cols) + " = " + std::to_string(threads) +
           " threads exceeds max_workgroup_size " + std::to_string(dev.max_workgroup_size));

  const std::size_t x = dev.elems_per_cache_line();
  const std::size_t regs = cfg.register_tile() + 2 * x;
  if (regs > dev.register_budget)
    reject("register budget: " + std::to_string(cfg.register_tile()) + " + 2*" +
           std::to_string(x) + " = " + std::to_string(regs) +
           " registers exceeds register_budget " + std::to_string(dev.register_budget));

  if (cfg.double_buffer && !cfg.use_local_memory)
    reject("config invariant: double_buffer requires use_local_memory");

  if (cfg.use_local_memory) {
    if (dev.local_memory_bytes == 0) {
      reject("local-memory budget: device \"" + dev.name + "\" has no local memory");
    } else {
      const std::size_t bytes = 4 * local_mem_elems(cfg, dev);
      if (bytes > dev.local_memory_bytes)
        reject("local-memory budget: " + std::to_string(bytes) +
               " bytes exceeds local_memory_bytes " + std::to_string(dev.local_memory_bytes));
    }
  }
  return v;
}

namespace detail {

inline void check_gemm_operands(const Matrix& a, const Matrix& b, const Matrix& c,
                                const GemmShape& shape) {
  auto expect = [](const char* which, const Matrix& mat, std::size_t r, std::size_t cc) {
    if (mat.rows != r || mat.cols != cc)
      throw ShapeError(std::string("gemm: operand ") + which + " is " + std::to_string(mat.rows) +
                       "x" + std::to_string(mat.cols) + ", expected " + std::to_string(r) + "x" +
                       std::to_string(cc));
  };
  const bool ta = shape.op_a == Op::Transpose, tb = shape.op_b == Op::Transpose;
  expect("A", a, ta ? shape.k : shape.m, ta ? shape.m : shape.k);
  expect("B", b, tb ? shape.n : shape.k, tb ? shape.k : shape.n);
  expect("C", c, shape.m, shape.n);
}

}  // namespace detail

// ---- kernels ---------------------------------------------------------------

// The oracle's arithmetic, on the GPU: one ascending-k dot product per
// element, then alpha*r (+ beta*C when beta != 0; C is not read otherwise).
inline Matrix gemm_naive(const Matrix& a, const Matrix& b, const Matrix& c,
                         const GemmShape& shape) {
  detail::check_gemm_operands(a, b, c, shape);
  Matrix out(shape.m, shape.n);
  const tk_gemm_shape s = detail::to_c(shape);
  detail::check_status(tk_gemm_naive(&s, a.data.data(), b.data.data(), c.data.data(),
                                     out.data.data()));
  return out;
}

// Blocked GEMM with the GemmConfig's register tile, work-group, staging
// and double buffering mapped onto a B200 CTA.  Rejected
// configs raise ConfigError exactly as in the reference.
inline Matrix gemm_tiled(const Matrix& a, const Matrix& b, const Matrix& c,
                         const GemmShape& shape, const GemmConfig& cfg, const DeviceSpec& dev) {
  detail::check_gemm_operands(a, b, c, shape);
  Matrix out(shape.m, shape.n);
  const tk_gemm_shape s = detail::to_c(shape);
  const tk_gemm_config g = detail::to_c(cfg);
  const tk_device_spec d = detail::to_c(dev);
  detail::check_status(tk_gemm_tiled(&s, &g, &d, a.data.data(), b.data.data(), c.data.data(),
                                     out.data.data()));
  return out;
}

// C_g = A_g * B_g over packed column-major host matrices (C zeroed first);
// returns the scalar multiply count.
inline std::uint64_t gemm_batched_strided(const float* a, std::size_t stride_a, const float* b,
                                          std::size_t stride_b, float* c, std::size_t stride_c,
                                          std::size_t batch, std::size_t m, std::size_t n,
                                          std::size_t k) {
  std::uint64_t count = 0;
  detail::check_status(
      tk_gemm_batched_strided(a, stride_a, b, stride_b, c, stride_c, batch, m, n, k, &count));
  return count;
}

namespace b200 {

// gemm with B200 execution options (precision, tensor-core tile) on host
// matrices; same operand conventions and checks as gemm_naive.
inline Matrix gemm(const Matrix& a, const Matrix& b, const Matrix& c, const GemmShape& shape,
                   const ExecOptions& opts) {
  tilekit::detail::check_gemm_operands(a, b, c, shape);
  Matrix out(shape.m, shape.n);
  const tk_gemm_shape s = tilekit::detail::to_c(shape);
  const tk_exec_options o = opts.c();
  tilekit::detail::check_status(
      tk_gemm_ex(&s, &o, a.data.data(), b.data.data(), c.data.data(), out.data.data()));
  return out;
}

}  // namespace b200
}  // namespace tilekit

// ref_shim.cpp -- C-ABI wrapper over the UNMODIFIED reference headers.
//
// TEST INFRASTRUCTURE ONLY (see oracle/tk_oracle.c).  Compiled by
// oracle/Makefile straight from /root/reference/proj/include (never copied)
// into oracle/_ref/libtkref.so.  The reference namespace is renamed to
// tilekit_ref so this object can never collide with the product's own
// tilekit:: symbols (hard part 7).
//
// Uses: pinning oracle/tk_oracle.c (tests/golden/make_golden.py) and the
// CPU baseline / --impl reference arm of bench.py (the reference's own
// gemm_tiled / conv2d timed on the host cores).
#define tilekit tilekit_ref
#include "tilekit/analysis.hpp"
#include "tilekit/config.hpp"
#include "tilekit/conv.hpp"
#include "tilekit/device.hpp"
#include "tilekit/gemm.hpp"
#include "tilekit/layers.hpp"
#include "tilekit/numeric.hpp"
#include "tilekit/tuner.hpp"
#include "tilekit/winograd.hpp"
#undef tilekit

#include <chrono>
#include <cstring>
#include <sstream>
#include <string>

namespace tk = tilekit_ref;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
  g_err = e.what();
  if (dynamic_cast<const tk::ShapeError*>(&e)) return 1;
  if (dynamic_cast<const tk::ConfigError*>(&e)) return 2;
  if (dynamic_cast<const tk::ParseError*>(&e)) return 3;
  if (dynamic_cast<const tk::CapabilityError*>(&e)) return 4;
  if (dynamic_cast<const tk::ContractError*>(&e)) return 5;
  if (dynamic_cast<const tk::IoError*>(&e)) return 6;
  if (dynamic_cast<const tk::TuningError*>(&e)) return 7;
  return 99;
}

struct ShapeC {
  size_t batch, in_rows, in_cols, channels, features;
  size_t window_rows, window_cols, stride;
  int same;
};

tk::ConvShape to_shape(const ShapeC* s) {
  tk::ConvShape c;
  c.batch = s->batch;
  c.in_rows = s->in_rows;
  c.in_cols = s->in_cols;
  c.channels = s->channels;
  c.features = s->features;
  c.window_rows = s->window_rows;
  c.window_cols = s->window_cols;
  c.stride = s->stride;
  c.padding = s->same ? tk::Padding::Same : tk::Padding::Valid;
  return c;
}

tk::GemmShape gshape(size_t m, size_t n, size_t k, float alpha, float beta,
                     int ta, int tb) {
  tk::GemmShape g;
  g.m = m;
  g.n = n;
  g.k = k;
  g.alpha = alpha;
  g.beta = beta;
  g.op_a = ta ? tk::Op::Transpose : tk::Op::Identity;
  g.op_b = tb ? tk::Op::Transpose : tk::Op::Identity;
  return g;
}

tk::Matrix mat(size_t r, size_t c, const float* p) {
  return tk::Matrix(r, c, std::vector<float>(p, p + r * c));
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void ref_fill_random(float* data, size_t n, uint64_t seed) {
  std::vector<float> v(n);
  tk::detail::fill_random(v, seed);
  std::memcpy(data, v.data(), n * sizeof(float));
}

uint64_t ref_fnv1a(const char* s) { return tk::detail::fnv1a(s); }

int ref_gemm_naive(size_t m, size_t n, size_t k, float alpha, float beta,
                   int ta, int tb, const float* a, const float* b,
                   const float* c, float* out) {
  try {
    tk::GemmShape g = gshape(m, n, k, alpha, beta, ta, tb);
    tk::Matrix A = mat(ta ? k : m, ta ? m : k, a);
    tk::Matrix B = mat(tb ? n : k, tb ? k : n, b);
    tk::Matrix C = mat(m, n, c);
    tk::Matrix O = tk::gemm_naive(A, B, C, g);
    std::memcpy(out, O.data.data(), m * n * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// dev_name: a find_device() name, or "" for host_device().
int ref_gemm_tiled(size_t m, size_t n, size_t k, float alpha, float beta,
                   int ta, int tb, const float* a, const float* b,
                   const float* c, float* out, const char* cfg_name,
                   const char* dev_name) {
  try {
    tk::GemmShape g = gshape(m, n, k, alpha, beta, ta, tb);
    tk::Matrix A = mat(ta ? k : m, ta ? m : k, a);
    tk::Matrix B = mat(tb ? n : k, tb ? k : n, b);
    tk::Matrix C = mat(m, n, c);
    tk::DeviceSpec dev =
        (dev_name && *dev_name) ? tk::find_device(dev_name) : tk::host_device();
    tk::Matrix O = tk::gemm_tiled(A, B, C, g, tk::parse_gemm_config(cfg_name), dev);
    std::memcpy(out, O.data.data(), m * n * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

uint64_t ref_gemm_batched_strided(const float* a, size_t sa, const float* b,
                                  size_t sb, float* c, size_t sc, size_t batch,
                                  size_t m, size_t n, size_t k) {
  return tk::gemm_batched_strided(a, sa, b, sb, c, sc, batch, m, n, k);
}

// params: the conv grammar ("naive", "im2col", "tiled_t4x5_v4x2",
// "winograd_t2x2"), dispatched through the reference conv2d selector.
int ref_conv2d(const ShapeC* s, const char* params, const float* in,
               const float* filt, float* out) {
  try {
    tk::ConvShape cs = to_shape(s);
    tk::Tensor4 I(tk::Tensor4Layout::InputNhwc, cs.batch, cs.in_rows,
                  cs.in_cols, cs.channels,
                  std::vector<float>(in, in + cs.batch * cs.in_rows *
                                                  cs.in_cols * cs.channels));
    tk::Tensor4 F(tk::Tensor4Layout::FilterHwck, cs.window_rows,
                  cs.window_cols, cs.channels, cs.features,
                  std::vector<float>(filt, filt + cs.window_rows *
                                                      cs.window_cols *
                                                      cs.channels * cs.features));
    tk::Tensor4 O = tk::conv2d(I, F, cs, tk::parse_conv_params(params));
    std::memcpy(out, O.data.data(), O.data.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_conv2d_winograd(const ShapeC* s, size_t m, const float* in,
                        const float* filt, float* out, uint64_t* mults,
                        size_t* tiles) {
  try {
    tk::ConvShape cs = to_shape(s);
    tk::Tensor4 I(tk::Tensor4Layout::InputNhwc, cs.batch, cs.in_rows,
                  cs.in_cols, cs.channels,
                  std::vector<float>(in, in + cs.batch * cs.in_rows *
                                                  cs.in_cols * cs.channels));
    tk::Tensor4 F(tk::Tensor4Layout::FilterHwck, cs.window_rows,
                  cs.window_cols, cs.channels, cs.features,
                  std::vector<float>(filt, filt + cs.window_rows *
                                                      cs.window_cols *
                                                      cs.channels * cs.features));
    tk::ConvAlgoParams p;
    p.algo = tk::ConvAlgo::Winograd;
    p.tile_rows = m;
    p.tile_cols = m;
    tk::WinogradStats st;
    tk::Tensor4 O = tk::conv2d_winograd(I, F, cs, p, &st);
    std::memcpy(out, O.data.data(), O.data.size() * sizeof(float));
    if (mults) *mults = st.batched_multiplies;
    if (tiles) *tiles = st.tiles;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

int ref_im2col(const ShapeC* s, const float* in, float* patches) {
  try {
    tk::ConvShape cs = to_shape(s);
    tk::Tensor4 I(tk::Tensor4Layout::InputNhwc, cs.batch, cs.in_rows,
                  cs.in_cols, cs.channels,
                  std::vector<float>(in, in + cs.batch * cs.in_rows *
                                                  cs.in_cols * cs.channels));
    tk::Matrix P = tk::im2col(I, cs);
    std::memcpy(patches, P.data.data(), P.data.size() * sizeof(float));
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The reference's own GEMM selection (tuner.hpp:560-578) over the stock
// configs on host_device(); returns the best median ns and writes the
// winning config name.  This is the CPU baseline for SGEMM.
int ref_tune_gemm_stock(size_t m, size_t n, size_t k, int warmup, int samples,
                        int64_t* best_median_ns, char* best_cfg, size_t cap) {
  try {
    tk::GemmShape g = gshape(m, n, k, 1.0f, 0.0f, 0, 0);
    tk::BenchOptions o;
    o.warmup = warmup;
    o.samples = samples;
    tk::TuningRecord best = tk::tune(tk::Problem::of(g), tk::stock_gemm_configs(),
                                     tk::host_device(), o).best;
    *best_median_ns = best.median_ns;
    std::snprintf(best_cfg, cap, "%s", best.config.c_str());
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// The reference's benchmark_config for one conv algorithm (tuner.hpp:411).
int ref_benchmark_conv(const ShapeC* s, const char* params, int warmup,
                       int samples, int64_t* median_ns, int* valid) {
  try {
    tk::BenchOptions o;
    o.warmup = warmup;
    o.samples = samples;
    tk::TuningRecord r = tk::benchmark_config(tk::Problem::of(to_shape(s)),
                                              tk::parse_conv_params(params),
                                              tk::host_device(), o);
    *median_ns = r.median_ns;
    *valid = r.valid ? 1 : 0;
    return 0;
  } catch (const std::exception& e) {
    return fail(e);
  }
}

// Wall time of one reference conv2d call on caller-provided data.
int64_t ref_time_conv2d(const ShapeC* s, const char* params, const float* in,
                        const float* filt, float* out) {
  auto t0 = std::chrono::steady_clock::now();
  int rc = ref_conv2d(s, params, in, filt, out);
  auto t1 = std::chrono::steady_clock::now();
  if (rc != 0) return -rc;
  return std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
}

// Copies text into a caller buffer; returns the full length (truncates).
static size_t put_text(const std::string& t, char* out, size_t cap) {
  if (cap) {
    const size_t n = t.size() < cap - 1 ? t.size() : cap - 1;
    std::memcpy(out, t.data(), n);
    out[n] = 0;
  }
  return t.size();
}

// The reference's render_report over n points (analysis.hpp:157-181).
// Returns the text length, or -1 with the message in ref_last_error.
long long ref_render_report(int n, const char** problems, const char** configs,
                            const double* oi, const double* gflops, const int* ok, int json,
                            char* out, size_t cap) {
  try {
    std::vector<tk::RooflinePoint> pts(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      pts[i].problem = problems[i];
      pts[i].config = configs[i];
      pts[i].oi = oi[i];
      pts[i].gflops = gflops[i];
      pts[i].ok = ok[i] != 0;
    }
    return (long long)put_text(
        tk::render_report(pts, json ? tk::ReportFormat::Json : tk::ReportFormat::Csv), out, cap);
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

// The reference's load_layer_rows on in-memory text, re-serialised
// (layers.hpp:90-185): returns the serialised table, or on a parse error
// -1 with the exception message in ref_last_error.
long long ref_layer_table(const char* text, const char* origin, char* out, size_t cap) {
  try {
    std::istringstream in(text);
    return (long long)put_text(tk::serialize_layer_rows(tk::load_layer_rows(in, origin)), out,
                               cap);
  } catch (const std::exception& e) {
    fail(e);
    return -1;
  }
}

}  // extern "C"

// test_dropin.cpp -- the reference's C++ API, recompiled against the B200
// headers (include/tilekit/*.hpp) and linked to libtilekit_b200.so.
//
//   test_dropin cpu   host-only checks (grammars, budgets, geometry, errors)
//   test_dropin gpu   compute checks on the B200 (known answers from the
//                     reference's own unit tests + bit-identity)
//
// Written like the reference's acceptance suite (plain main, no framework):
// every CHECK prints on failure and the exit code is the failure count.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "tilekit/tilekit.hpp"

using namespace tilekit;

static int g_fail = 0;
#define CHECK(cond)                                                   \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
      ++g_fail;                                                       \
    }                                                                 \
  } while (0)

template <typename E, typename F>
static bool throws_with(F&& f, const char* needle) {
  try {
    f();
  } catch (const E& e) {
    return needle == nullptr || std::string(e.what()).find(needle) != std::string::npos;
  } catch (...) {
    return false;
  }
  return false;
}

// Same generator as the reference tests (helpers.hpp: mt19937_64 + U[-1,1)).
static void fill(std::vector<float>& v, std::uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<float> d(-1.0f, 1.0f);
  for (float& x : v) x = d(rng);
}

static bool bits_equal(const std::vector<float>& a, const std::vector<float>& b) {
  return a.size() == b.size() && std::memcmp(a.data(), b.data(), a.size() * 4) == 0;
}

static GemmShape gshape(std::size_t m, std::size_t n, std::size_t k, float al = 1, float be = 0,
                        Op oa = Op::Identity, Op ob = Op::Identity) {
  GemmShape s;
  s.m = m;
  s.n = n;
  s.k = k;
  s.alpha = al;
  s.beta = be;
  s.op_a = oa;
  s.op_b = ob;
  return s;
}

static ConvShape cshape(std::size_t h, std::size_t w, std::size_t c, std::size_t k, std::size_t r,
                        std::size_t stride, Padding pad, std::size_t batch = 1) {
  ConvShape s;
  s.batch = batch;
  s.in_rows = h;
  s.in_cols = w;
  s.channels = c;
  s.features = k;
  s.window_rows = r;
  s.window_cols = r;
  s.stride = stride;
  s.padding = pad;
  return s;
}

static void cpu_checks() {
  // grammars (test_config.cpp)
  for (const char* n : {"4x4_8x8_loc", "8x4_8x16_loc_db", "8x2_4x16_noloc"})
    CHECK(parse_gemm_config(n).name() == n);
  CHECK(throws_with<ParseError>([] { parse_gemm_config("4x4_8x8_noloc_db"); }, "trailing"));
  CHECK(throws_with<ParseError>([] { parse_gemm_config("0x4_8x8_loc"); }, "positive"));
  for (const char* n : {"naive", "im2col", "tiled_t4x5_v4x2", "winograd_t2x2"})
    CHECK(parse_conv_params(n).name() == n);
  CHECK(throws_with<ParseError>([] { parse_conv_params("tiled_t4x5_v3x2"); }, "vector widths"));
  CHECK(parse_conv_algo("winograd") == ConvAlgo::Winograd);

  // budgets (test_gemm.cpp:160-195, acceptance 9)
  const DeviceSpec gpu = find_device("Intel Core i7-6700K GPU");
  CHECK(validate_config(parse_gemm_config("4x4_8x8_loc"), gpu, {}).ok);
  DeviceSpec tiny = gpu;
  tiny.register_budget = 20;
  tiny.max_workgroup_size = 16;
  tiny.local_memory_bytes = 1024;
  const ConfigVerdict v = validate_config(parse_gemm_config("8x4_16x16_loc"), tiny, {});
  CHECK(!v.ok && v.violations.size() == 3);
  CHECK(!validate_config(parse_gemm_config("4x4_8x8_loc"), find_device("mali"), {}).ok);
  CHECK(local_mem_elems(parse_gemm_config("4x4_8x8_loc_db"), gpu) == 2 * 16 * (32 + 32));
  CHECK(builtin_devices().size() == 7);
  CHECK(throws_with<ParseError>([] { find_device("intel"); }, "ambiguous"));

  // reuse model (Eq. 3)
  CHECK(std::fabs(data_reuse(8, 4, 16).reuse - 2.0 * 8 * 4 / 12.0) < 1e-12);

  // geometry (config.hpp:137-195): TF-style Same padding for the stem
  const ConvShape stem = cshape(224, 224, 3, 64, 7, 2, Padding::Same);
  CHECK(stem.out_rows() == 112 && stem.pad_top() == 2 && stem.pad_left() == 2);
  CHECK(cshape(4, 4, 1, 1, 3, 1, Padding::Valid).out_rows() == 2);

  // Winograd plans (test_winograd.cpp:55-71)
  CHECK(winograd_plan(2, 2, 3, 3).input_transform.rows == 4);
  CHECK(winograd_plan(4, 4, 3, 3).output_transform.cols == 6);
  CHECK(throws_with<CapabilityError>([] { winograd_plan(3, 3, 3, 3); }, "supported"));

  // B200 device record (kept out of builtin_devices)
  const DeviceSpec b200 = b200_device();
  CHECK(b200.cache_line_bytes == 128 && b200.max_workgroup_size == 1024);
  CHECK(validate_config(parse_gemm_config("8x8_16x16_loc_db"), b200, {}).ok);

  // operand checks happen before any device work (test_gemm.cpp:235-249)
  Matrix a(2, 3), b(3, 2), c(2, 2), bad_b(4, 2);
  CHECK(throws_with<ShapeError>([&] { gemm_naive(a, bad_b, c, gshape(2, 2, 3)); }, "B"));
  CHECK(throws_with<ConfigError>(
      [&] { gemm_tiled(a, b, c, gshape(2, 2, 3), parse_gemm_config("4x4_8x8_loc"),
                       find_device("mali")); },
      "local-memory budget"));
}

static void gpu_checks() {
  const DeviceSpec gpu = find_device("Intel Core i7-6700K GPU");
  // gemm_naive known answers (test_gemm.cpp:199-233)
  {
    Matrix a(2, 2, {1, 3, 2, 4}), b(2, 2, {5, 7, 6, 8}), c(2, 2);
    const Matrix out = gemm_naive(a, b, c, gshape(2, 2, 2));
    CHECK(out(0, 0) == 19 && out(0, 1) == 22 && out(1, 0) == 43 && out(1, 1) == 50);
    Matrix one_a(1, 1, {2}), one_b(1, 1, {3}), nan_c(1, 1, {std::nanf("")});
    CHECK(gemm_naive(one_a, one_b, nan_c, gshape(1, 1, 1))(0, 0) == 6.0f);
  }
  // gemm_tiled == gemm_naive bit for bit, every op combo and stock config
  for (Op oa : {Op::Identity, Op::Transpose})
    for (Op ob : {Op::Identity, Op::Transpose}) {
      const GemmShape s = gshape(33, 29, 21, 1.5f, -0.5f, oa, ob);
      Matrix a(oa == Op::Identity ? 33 : 21, oa == Op::Identity ? 21 : 33);
      Matrix b(ob == Op::Identity ? 21 : 29, ob == Op::Identity ? 29 : 21);
      Matrix c(33, 29);
      fill(a.data, 17);
      fill(b.data, 23);
      fill(c.data, 31);
      const Matrix want = gemm_naive(a, b, c, s);
      for (const char* name : {"4x4_8x8_loc", "8x4_4x8_noloc", "8x4_8x16_loc_db"}) {
        const Matrix got = gemm_tiled(a, b, c, s, parse_gemm_config(name), gpu);
        CHECK(bits_equal(got.data, want.data));
        CHECK(max_rel_error(got.data, want.data) == 0.0);
      }
    }
  // conv known answers (test_conv.cpp:39-89)
  {
    Tensor4 in(Tensor4Layout::InputNhwc, 1, 3, 3, 1), f(Tensor4Layout::FilterHwck, 3, 3, 1, 1);
    std::fill(in.data.begin(), in.data.end(), 1.0f);
    std::fill(f.data.begin(), f.data.end(), 1.0f);
    const Tensor4 out = conv2d_naive(in, f, cshape(3, 3, 1, 1, 3, 1, Padding::Same));
    const float expect[9] = {4, 6, 4, 6, 9, 6, 4, 6, 4};
    for (int i = 0; i < 9; ++i) CHECK(out.data[i] == expect[i]);
  }
  // every algorithm vs conv2d_naive (tiled/im2col bit-identical, Winograd
  // FP32 bit-identical to the reference Winograd and <= 1e-3 scaled of naive)
  for (std::size_t stride : {1, 2})
    for (Padding pad : {Padding::Valid, Padding::Same}) {
      const ConvShape s = cshape(12, 10, 6, 8, 3, stride, pad, 2);
      Tensor4 in(Tensor4Layout::InputNhwc, 2, 12, 10, 6), f(Tensor4Layout::FilterHwck, 3, 3, 6, 8);
      fill(in.data, 81 + stride);
      fill(f.data, 82);
      const Tensor4 want = conv2d_naive(in, f, s);
      CHECK(bits_equal(conv2d(in, f, s, parse_conv_params("im2col")).data, want.data));
      CHECK(bits_equal(conv2d(in, f, s, parse_conv_params("tiled_t4x5_v4x2")).data, want.data));
      if (stride == 1) {
        WinogradStats st;
        const Tensor4 w = conv2d_winograd(in, f, s, parse_conv_params("winograd_t4x4"), &st);
        CHECK(max_scaled_error(w.data, want.data) <= 1e-3);
        CHECK(st.tiles > 0 && st.batched_multiplies == 36ull * st.tiles * 8 * 6);
        // tensor-core extension: TF32 implicit GEMM within the stated tolerance
        b200::ExecOptions o;
        o.precision = b200::Precision::Tf32;
        const Tensor4 tc = b200::conv2d(in, f, s, parse_conv_params("im2col"), o);
        CHECK(max_scaled_error(tc.data, want.data) <= 1e-3);
      } else {
        CHECK(throws_with<CapabilityError>(
            [&] { conv2d_winograd(in, f, s, parse_conv_params("winograd_t2x2")); }, "stride"));
      }
    }
  // Winograd multiply counts on 8x8x1 (acceptance criterion 5)
  {
    Tensor4 in(Tensor4Layout::InputNhwc, 1, 8, 8, 1), f(Tensor4Layout::FilterHwck, 3, 3, 1, 1);
    fill(in.data, 1);
    fill(f.data, 2);
    WinogradStats s2, s4;
    conv2d_winograd(in, f, cshape(8, 8, 1, 1, 3, 1, Padding::Same),
                    parse_conv_params("winograd_t2x2"), &s2);
    conv2d_winograd(in, f, cshape(8, 8, 1, 1, 3, 1, Padding::Same),
                    parse_conv_params("winograd_t4x4"), &s4);
    CHECK(s2.batched_multiplies == 256 && s2.tiles == 16);
    CHECK(s4.batched_multiplies == 144 && s4.tiles == 4);
  }
  // gemm_batched_strided count
  {
    std::vector<float> a(4 * 5 * 3), b(4 * 3 * 2), c(4 * 5 * 2);
    fill(a, 1);
    fill(b, 2);
    CHECK(gemm_batched_strided(a.data(), 15, b.data(), 6, c.data(), 10, 4, 5, 2, 3) == 120);
  }
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  cpu_checks();
  if (mode == "gpu") gpu_checks();
  std::printf("%s: %d failure(s)\n", mode.c_str(), g_fail);
  return g_fail;
}

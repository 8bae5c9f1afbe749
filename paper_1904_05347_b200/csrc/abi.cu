// abi.cu -- the C ABI of libtilekit_b200.so (declared in include/tk_b200.h).
//
// Host-side validation reuses the drop-in headers (include/tilekit/*.hpp),
// so the C ABI and the C++ API reject the same inputs with the same
// messages as the reference (gemm.hpp:103-146, 308-317; conv.hpp:57-66,
// 140-150; winograd.hpp:114-118, 174-177).  Everything numeric runs on the
// GPU: there is no CPU fallback, and without an sm_100 device every compute
// entry point fails with TK_ERR_CUDA.
#include <atomic>
#include <map>
#include <memory>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <cstdlib>
#include <string>

#include "common.cuh"
#include "exact_gemm.cuh"
#include "experiments.cuh"
#include "launch_cache.cuh"
#include "tuning_db.cuh"
#include "layout.cuh"
#include "tc_gemm.cuh"
#include "tilekit/gemm.hpp"
#include "winograd.cuh"

namespace tkb {

namespace {

std::atomic<uint64_t> g_launches{0};
thread_local std::string g_error;

int usable_devices() {
  static int count = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
      cudaGetLastError();
      count = 0;
      return;
    }
    int usable = 0;
    for (int i = 0; i < n; ++i) {
      cudaDeviceProp prop{};
      if (cudaGetDeviceProperties(&prop, i) == cudaSuccess && prop.major == 10) ++usable;
    }
    count = usable;
  });
  return count;
}

void require_gpu() {
  if (usable_devices() == 0)
    fail(TK_ERR_CUDA, "no sm_100 (B200) GPU available: the tilekit B200 kernels have no CPU "
                      "fallback");
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return TK_OK;
  } catch (const Failure& f) {
    g_error = f.msg;
    return f.code;
  } catch (const tilekit::ShapeError& e) {
    g_error = e.what();
    return TK_ERR_SHAPE;
  } catch (const tilekit::ConfigError& e) {
    g_error = e.what();
    return TK_ERR_CONFIG;
  } catch (const tilekit::ParseError& e) {
    g_error = e.what();
    return TK_ERR_PARSE;
  } catch (const tilekit::CapabilityError& e) {
    g_error = e.what();
    return TK_ERR_CAPABILITY;
  } catch (const tilekit::ContractError& e) {
    g_error = e.what();
    return TK_ERR_CONTRACT;
  } catch (const std::exception& e) {
    g_error = e.what();
    return TK_ERR_CUDA;
  }
}

// Stream-ordered scratch allocation (pool-backed, so repeated calls reuse
// memory without device-wide synchronisation).
struct DevBuf {
  void* p = nullptr;
  cudaStream_t st = nullptr;
  DevBuf(size_t bytes, cudaStream_t s) : st(s) {
    if (bytes) TKB_CUDA(cudaMallocAsync(&p, bytes, st));
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  float* f() const { return static_cast<float*>(p); }
};

void keep_pool_memory() {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t threshold = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold);
    }
  });
}

cudaStream_t host_stream() {
  require_gpu();
  keep_pool_memory();
  return cudaStreamPerThread;
}

void h2d(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes) TKB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
}
void d2h(void* dst, const void* src, size_t bytes, cudaStream_t st) {
  if (bytes) TKB_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
}
void finish(cudaStream_t st) { TKB_CUDA(cudaStreamSynchronize(st)); }

// ---- struct conversions ----------------------------------------------------

tilekit::GemmShape gemm_shape(const tk_gemm_shape* s) {
  if (!s) fail(TK_ERR_CONTRACT, "gemm: shape must not be NULL");
  tilekit::GemmShape g;
  g.m = s->m;
  g.n = s->n;
  g.k = s->k;
  g.alpha = s->alpha;
  g.beta = s->beta;
  g.op_a = s->op_a ? tilekit::Op::Transpose : tilekit::Op::Identity;
  g.op_b = s->op_b ? tilekit::Op::Transpose : tilekit::Op::Identity;
  if (g.m == 0 || g.n == 0 || g.k == 0)
    fail(TK_ERR_SHAPE, "gemm: dimensions must be positive, got m=" + std::to_string(g.m) +
                           " n=" + std::to_string(g.n) + " k=" + std::to_string(g.k));
  return g;
}

tilekit::GemmConfig gemm_config(const tk_gemm_config* c) {
  tilekit::GemmConfig g;
  g.reg_rows = c->reg_rows;
  g.reg_cols = c->reg_cols;
  g.wg_rows = c->wg_rows;
  g.wg_cols = c->wg_cols;
  g.use_local_memory = c->use_local_memory != 0;
  g.double_buffer = c->double_buffer != 0;
  g.k_step = c->k_step;
  return g;
}

tilekit::DeviceSpec device_spec(const tk_device_spec* d) {
  tilekit::DeviceSpec s;
  s.name = d->name ? d->name : "";
  s.cache_line_bytes = d->cache_line_bytes;
  s.local_memory_bytes = d->local_memory_bytes;
  s.compute_units = d->compute_units;
  s.register_budget = d->register_budget;
  s.max_workgroup_size = d->max_workgroup_size;
  return s;
}

tilekit::ConvShape conv_shape(const tk_conv_shape* s) {
  if (!s) fail(TK_ERR_CONTRACT, "conv2d: shape must not be NULL");
  tilekit::ConvShape c;
  c.batch = s->batch;
  c.in_rows = s->in_rows;
  c.in_cols = s->in_cols;
  c.channels = s->channels;
  c.features = s->features;
  c.window_rows = s->window_rows;
  c.window_cols = s->window_cols;
  c.stride = s->stride;
  c.padding = s->padding ? tilekit::Padding::Same : tilekit::Padding::Valid;
  return c;
}

// The shape-only part of check_conv_operands (conv.hpp:57-66).
ConvGeom conv_geom(const tilekit::ConvShape& s) {
  if (s.batch == 0 || s.in_rows == 0 || s.in_cols == 0 || s.channels == 0 || s.features == 0 ||
      s.window_rows == 0 || s.window_cols == 0)
    fail(TK_ERR_SHAPE, "conv2d: dimensions must be positive");
  if (s.stride == 0) fail(TK_ERR_SHAPE, "conv2d: stride must be >= 1");
  if (s.out_rows() == 0 || s.out_cols() == 0)
    fail(TK_ERR_SHAPE, "conv2d: window " + std::to_string(s.window_rows) + "x" +
                           std::to_string(s.window_cols) + " does not fit the " +
                           std::to_string(s.in_rows) + "x" + std::to_string(s.in_cols) +
                           " input");
  const double pix = (double)s.batch * s.out_rows() * s.out_cols();
  if (pix > 2.0e9 || (double)s.window_rows * s.window_cols * s.channels > 2.0e9)
    fail(TK_ERR_CAPABILITY, "conv2d: problem exceeds 32-bit index range");
  ConvGeom g;
  g.N = (int)s.batch;
  g.H = (int)s.in_rows;
  g.W = (int)s.in_cols;
  g.C = (int)s.channels;
  g.K = (int)s.features;
  g.R = (int)s.window_rows;
  g.S = (int)s.window_cols;
  g.stride = (int)s.stride;
  g.OH = (int)s.out_rows();
  g.OW = (int)s.out_cols();
  g.pad_t = (int)s.pad_top();
  g.pad_l = (int)s.pad_left();
  return g;
}

size_t in_elems(const ConvGeom& g) { return (size_t)g.N * g.H * g.W * g.C; }
size_t filt_elems(const ConvGeom& g) { return (size_t)g.R * g.S * g.C * g.K; }
size_t out_elems(const ConvGeom& g) { return (size_t)g.N * g.OH * g.OW * g.K; }

int precision_of(const tk_exec_options* o) { return o ? o->precision : TK_PREC_FP32_EXACT; }

// Tensor-core knobs of one C-ABI call (restored on return).
struct KnobScope {
  TcKnobs saved;
  explicit KnobScope(const tk_exec_options* o) : saved(tc_knobs()) {
    TcKnobs k;
    if (o) {
      k.stages = o->tc_stages;
      k.cluster = o->tc_cluster;
      k.mode = o->tc_mode;
      k.split = o->tc_split;
      k.io = o->io;
    }
    tc_knobs() = k;
  }
  ~KnobScope() { tc_knobs() = saved; }
  KnobScope(const KnobScope&) = delete;
  KnobScope& operator=(const KnobScope&) = delete;
};

// Tuning DB on the launch path: a call whose tensor-core knobs are all
// automatic takes the DB's fastest valid record for its problem (tuning_db.cuh).
bool all_auto(const tk_exec_options* o) {
  return !o || (o->tc_tile_n == 0 && o->tc_stages == 0 && o->tc_cluster == 0 && o->tc_mode == 0 &&
                o->tc_split == 0);
}

bool apply_tuned_conv(const tilekit::ConvShape& s, const tk_conv_params* p,
                      const tk_exec_options* o) {
  const int prec = o ? o->precision : TK_PREC_FP32_EXACT;
  if (!p || p->algo != 2 || prec == TK_PREC_FP32_EXACT || !all_auto(o)) return false;
  TunedKnobs k;
  // bf16 activations in HBM (io flags) are tuned separately ("im2col_io").
  if (!tuning_db_lookup(s.key(), o->io ? "im2col_io" : "im2col", prec, &k)) return false;
  if (!k.stages && !k.cluster && !k.mode && !k.split) return false;  // the DB keeps the rules
  TcKnobs& t = tc_knobs();
  t.stages = k.stages;
  t.cluster = k.cluster;
  t.mode = k.mode;
  t.split = k.split;
  return true;
}

// GEMM: the N tile travels as an argument, the rest through tc_knobs.
int tuned_gemm_tile(const tilekit::GemmShape& g, const tk_exec_options* o, bool* hit = nullptr) {
  const int prec = o ? o->precision : TK_PREC_FP32_EXACT;
  if (hit) *hit = false;
  if (prec == TK_PREC_FP32_EXACT) return 0;
  if (!all_auto(o)) return o->tc_tile_n;
  TunedKnobs k;
  if (!tuning_db_lookup(g.key(), "gemm", prec, &k)) return 0;
  if (!k.tile_n && !k.stages && !k.cluster && !k.split) return 0;  // the DB keeps the rules
  if (hit) *hit = true;
  TcKnobs& t = tc_knobs();
  t.stages = k.stages;
  t.cluster = k.cluster;
  t.split = k.split;
  return k.tile_n;
}

// ---- exact GEMM plumbing ---------------------------------------------------

// Library default for the exact path: 8x8 register tile, 16x16 threads
// (128x128 CTA tile), three-stage cp.async ring.
constexpr ExactLaunch kExactDefault{8, 8, 16, 16, true, 3};

// Library tile for the exact path when the caller names no GemmConfig,
// from the output extent (measured on B200, profiles/r01_sweep_fp32.csv and
// the VGG16 layers): 128x128 CTAs (two per SM) while they fill four waves;
// <= 64 output columns would idle half of that tile, so 256x64; smaller
// problems drop to 64x128 / 64x64 CTAs to fill the 148 SMs.  Two stages:
// a third costs the second resident CTA for no gain.
// TK_EXACT_STAGES / TK_EXACT_TILE="h,w,r,c" override (tuning experiments).
ExactLaunch exact_auto(long long M, long long N) {
  auto tiles = [&](long long bm, long long bn) { return ((M + bm - 1) / bm) * ((N + bn - 1) / bn); };
  ExactLaunch L = kExactDefault;
  L.stages = 2;
  if (N <= 64) {
    L.r = 32;
    L.c = 8;
  } else if (tiles(128, 128) < 4 * 148) {
    L.r = 8;  // 64 x 128
    if (tiles(64, 128) < 2 * 148) L.w = 4;  // 64 x 64
  }
  const Experiments& xp = experiments();
  if (xp.exact_stages > 0) L.stages = xp.exact_stages;
  if (xp.exact_tile[0] > 0) {
    L.h = xp.exact_tile[0];
    L.w = xp.exact_tile[1];
    L.r = xp.exact_tile[2];
    L.c = xp.exact_tile[3];
  }
  return L;
}

ExactLaunch exact_conv_default(const ConvGeom& g) {
  return exact_auto((long long)g.N * g.OH * g.OW, g.K);
}

ExactLaunch exact_launch_of(const tilekit::GemmConfig& c) {
  ExactLaunch L;
  L.h = (int)c.reg_rows;
  L.w = (int)c.reg_cols;
  L.r = (int)c.wg_rows;
  L.c = (int)c.wg_cols;
  L.loc = c.use_local_memory;
  L.stages = c.double_buffer ? 3 : 1;
  // h, w outside {1, 2, 4, 8}: the runtime-tile kernel (microkernel_generic,
  // gemm.hpp:247-292), bit-identical like every exact path.
  auto pow2 = [](int v) { return v == 1 || v == 2 || v == 4 || v == 8; };
  L.gen = !pow2(L.h) || !pow2(L.w);
  return L;
}

ExactArgs gemm_args(const tilekit::GemmShape& g, const float* a, const float* b, const float* c,
                    float* d) {
  ExactArgs p{};
  if (g.m > 2147483647ull || g.n > 2147483647ull || g.k > 2147483647ull)
    fail(TK_ERR_CAPABILITY, "gemm: dimensions exceed the 32-bit index range");
  p.M = (int)g.m;
  p.N = (int)g.n;
  p.K = (int)g.k;
  p.a = a;
  const bool ta = g.op_a == tilekit::Op::Transpose, tb = g.op_b == tilekit::Op::Transpose;
  p.a_sm = ta ? (long long)g.k : 1;
  p.a_sk = ta ? 1 : (long long)g.m;
  p.b = b;
  p.b_sk = tb ? (long long)g.n : 1;
  p.b_sn = tb ? 1 : (long long)g.k;
  p.c = c;
  p.d = d;
  p.d_sm = 1;
  p.d_sn = (long long)g.m;
  p.alpha = g.alpha;
  p.beta = g.beta;
  p.read_c = g.beta != 0.0f;  // beta == 0 (either sign): C is never read
  p.tx_on_m = 1;
  return p;
}

ExactArgs conv_args(const ConvGeom& g, const float* in, const float* filt, float* out) {
  ExactArgs p{};
  p.M = g.N * g.OH * g.OW;
  p.N = g.K;
  p.K = g.R * g.S * g.C;
  p.a = in;
  p.b = filt;
  p.b_sk = g.K;
  p.b_sn = 1;
  p.d = out;
  p.d_sm = g.K;
  p.d_sn = 1;
  p.alpha = 1.0f;
  p.beta = 0.0f;
  p.read_c = 0;
  p.tx_on_m = 0;
  p.H = g.H;
  p.W = g.W;
  p.C = g.C;
  p.OH = g.OH;
  p.OW = g.OW;
  p.R = g.R;
  p.S = g.S;
  p.stride = g.stride;
  p.pad_t = g.pad_t;
  p.pad_l = g.pad_l;
  return p;
}

// conv2d_tiled parameters (conv.hpp:136-248) -> the CTA of the runtime-
// tile kernel: each thread owns a tile_rows x tile_cols patch of output
// pixels (h = tile_rows * tile_cols register rows) for feature_vector
// features (w), the CTA's threads tile the output plane with such patches
// (r along pixels, c along features: 256 threads), the input is staged
// channel_vector channels per copy.  Same per-output sums: bit-identical.
ExactLaunch tiled_launch(const tk_conv_params* p, const ConvGeom& g) {
  ExactLaunch L{};
  L.h = (int)(p->tile_rows * p->tile_cols);
  auto pow2 = [](int v) { return v == 1 || v == 2 || v == 4 || v == 8; };
  // Patches of 1/2/4/8 pixels x 1/2/4/8 features run on the tuned kernels
  // (2-D patch rows through their pixel table); other tiles on the
  // runtime-tile kernel.
  L.gen = !(pow2(L.h) && pow2((int)p->feature_vector));
  L.w = (int)p->feature_vector;
  L.tile_rows = (int)p->tile_rows;
  L.tile_cols = (int)p->tile_cols;
  L.cvec = (int)std::min<size_t>(4, p->channel_vector);
  int c = 1;  // feature threads: enough to cover K, at most 16
  while (c < 16 && (size_t)c * p->feature_vector < (size_t)g.K) c *= 2;
  L.c = c;
  // 256 threads, at most ~320 pixel rows per CTA (the staged slab of the
  // patch matrix: 320 x 36 words, 46 KiB a stage).
  L.r = std::max(1, std::min(256 / c, 320 / std::max(1, L.h)));
  L.loc = true;
  L.stages = 2;
  L.shrink_ok = true;
  return L;
}

void check_tiled_params(const tilekit::ConvShape& s, const tk_conv_params* p) {
  if (p->tile_rows == 0 || p->tile_cols == 0)
    fail(TK_ERR_CONFIG, "conv2d_tiled: tile dimensions must be >= 1");
  if (!tilekit::valid_vector_width(p->channel_vector) ||
      !tilekit::valid_vector_width(p->feature_vector))
    fail(TK_ERR_CONFIG, "conv2d_tiled: vector widths must be one of 1, 2, 4, 8");
  if (s.stride != 1 && s.stride != 2)
    fail(TK_ERR_CAPABILITY, "conv2d_tiled: stride " + std::to_string(s.stride) + " not supported");
}

WinoGeom wino_geom(const ConvGeom& g, int m) {
  WinoGeom w{};
  w.m = m;
  w.t = m + 2;
  w.N = g.N;
  w.H = g.H;
  w.W = g.W;
  w.C = g.C;
  w.K = g.K;
  w.OH = g.OH;
  w.OW = g.OW;
  w.tiles_r = (g.OH + m - 1) / m;
  w.tiles_c = (g.OW + m - 1) / m;
  w.tiles = g.N * w.tiles_r * w.tiles_c;
  w.pad_t = g.pad_t;
  w.pad_l = g.pad_l;
  return w;
}

int check_winograd(const tilekit::ConvShape& s, const tk_conv_params* p) {
  if (s.stride != 1)
    fail(TK_ERR_CAPABILITY, "conv2d_winograd: stride " + std::to_string(s.stride) +
                                " not supported");
  const bool ok = s.window_rows == 3 && s.window_cols == 3 && p->tile_rows == p->tile_cols &&
                  (p->tile_rows == 2 || p->tile_rows == 4);
  if (!ok)
    fail(TK_ERR_CAPABILITY,
         "winograd_plan: no transform set for a " + std::to_string(p->tile_rows) + "x" +
             std::to_string(p->tile_cols) + " output tile under a " +
             std::to_string(s.window_rows) + "x" + std::to_string(s.window_cols) +
             " window (supported: 2x2 and 4x4 under 3x3)");
  return (int)p->tile_rows;
}

struct WinoSizes {
  size_t v, u, p;
  bool split3 = false;  // 3xTF32: + the tripled V and U operands
  size_t bytes() const { return 4 * (v + u + p) + 3 * 256 + (split3 ? 12 * (v + u) + 2 * 256 : 0); }
};
WinoSizes wino_sizes(const WinoGeom& w, int precision = TK_PREC_FP32_EXACT) {
  const size_t spots = (size_t)w.t * w.t;
  WinoSizes z{spots * w.tiles * w.C, spots * (size_t)w.C * w.K, spots * w.tiles * w.K};
  z.split3 = precision == TK_PREC_3XTF32 && w.C % 4 == 0;
  return z;
}

float* carve(char*& cursor, size_t elems) {
  float* p = reinterpret_cast<float*>(cursor);
  cursor += (elems * 4 + 255) / 256 * 256;
  return p;
}

// Device-side Winograd: transforms + batched GEMM on caller buffers.
void winograd_dev(const ConvGeom& g, int m, int precision, const float* in, const float* filt,
                  float* out, void* ws, cudaStream_t st, int phase = kConvAll) {
  const WinoGeom w = wino_geom(g, m);
  const WinoSizes sz = wino_sizes(w, precision);
  char* cur = static_cast<char*>(ws);
  float* v = carve(cur, sz.v);
  float* u = carve(cur, sz.u);
  float* prod = carve(cur, sz.p);
  float* v3 = sz.split3 ? carve(cur, 3 * sz.v) : nullptr;
  float* u3 = sz.split3 ? carve(cur, 3 * sz.u) : nullptr;
  // TMA needs 16-byte row strides; odd channel counts keep the exact GEMM.
  const bool tc = precision != TK_PREC_FP32_EXACT && w.C % 4 == 0;
  const int spots = w.t * w.t;
  // The filter transform depends only on the filter: the prepare phase
  // (3xTF32: also its (hi, lo, hi) expansion along C).
  if (phase & kConvPrepare) {
    wino_filter_transform(w, filt, u, /*k_major=*/tc, st);
    if (sz.split3) launch_split3_rows(u, (long long)spots * w.K, w.C, u3, 1, st);
  }
  if (!(phase & kConvRun)) return;
  wino_input_transform(w, in, v, st);
  if (sz.split3) launch_split3_rows(v, (long long)spots * w.tiles, w.C, v3, 0, st);
  if (!tc) {
    ExactArgs p{};
    p.M = w.tiles;
    p.N = w.K;
    p.K = w.C;
    p.a = v;
    p.a_sm = w.C;
    p.a_sk = 1;
    p.a_batch = (long long)w.tiles * w.C;
    p.b = u;
    p.b_sk = w.K;
    p.b_sn = 1;
    p.b_batch = (long long)w.C * w.K;
    p.d = prod;
    p.d_sm = w.K;
    p.d_sn = 1;
    p.d_batch = (long long)w.tiles * w.K;
    p.alpha = 1.0f;
    p.read_c = 0;
    p.tx_on_m = 0;
    launch_exact(p, exact_auto((long long)w.tiles * spots, w.K), false, spots, st);
  } else {
    // P[tile][k] = sum_c V[tile][c] * Ut[k][c]: tiles on the MMA M side,
    // features on N, so P's rows (k contiguous) leave through the TMA-store
    // epilogue (features on M stored column by column from registers: the
    // F(4x4) batched GEMM of VGG conv4_2 ran 109 us that way).
    // 3xTF32: the same GEMM over 3C ([v | v | v_lo] . [u_hi | u_lo | u_hi]),
    // ~fp32-accurate products, so F(4x4) meets the reference's 1e-3.
    const int kx = sz.split3 ? 3 : 1;
    TcGemm t{};
    t.M = w.tiles;
    t.N = w.K;
    t.K = kx * w.C;
    t.batch = spots;
    t.a = sz.split3 ? v3 : v;
    t.a_batch = (long long)w.tiles * w.C * kx;
    t.b = sz.split3 ? u3 : u;
    t.b_batch = (long long)w.C * w.K * kx;
    t.d = prod;
    t.d_sm = w.K;
    t.d_sn = 1;
    t.d_batch = (long long)w.tiles * w.K;
    // The transform-domain operands are fp32 scratch: the batched GEMM runs
    // kind::tf32 for every tensor-core precision request.
    t.precision = TK_PREC_TF32;
    launch_tc_gemm(t, st);
  }
  wino_output_transform(w, prod, out, st);
}

// tk_exec_options.io (bf16 activations in HBM): BF16 tensor-core convs only.
void check_io(const tk_conv_params* p, int precision) {
  const int io = tc_knobs().io;
  if (io == 0) return;
  if ((io & ~(TK_IO_IN_BF16 | TK_IO_OUT_BF16)) != 0)
    fail(TK_ERR_CONTRACT, "conv2d: unknown io flags " + std::to_string(io));
  if (precision != TK_PREC_BF16 || p->algo != 2)
    fail(TK_ERR_CAPABILITY, "conv2d: bf16 activations (io flags) need BF16 precision and the "
                            "im2col algorithm");
}

size_t conv_workspace(const ConvGeom& g, const tk_conv_params* p, int precision) {
  check_io(p, precision);
  if (p->algo == 3) return wino_sizes(wino_geom(g, (int)p->tile_rows), precision).bytes();
  if (precision != TK_PREC_FP32_EXACT) return tc_conv_workspace(g, precision);
  return 0;
}

// Dispatch of the conv2d selector on device buffers.
void conv_dev(const tilekit::ConvShape& s, const tk_conv_params* p, int precision,
              const float* in, const float* filt, float* out, void* ws, cudaStream_t st,
              int phase = kConvAll) {
  const ConvGeom g = conv_geom(s);
  check_io(p, precision);
  // Exact FP32 paths read the filter directly: nothing to prepare.
  const bool exact_run = (phase & kConvRun) != 0;
  switch (p->algo) {
    case 0:  // Naive: the oracle's arithmetic
      if (precision == TK_PREC_FP32_EXACT) {
        if (exact_run) launch_exact(conv_args(g, in, filt, out), exact_conv_default(g), true, 1, st);
        return;
      }
      break;
    case 1:  // Tiled
      check_tiled_params(s, p);
      if (precision == TK_PREC_FP32_EXACT) {
        if (exact_run) launch_exact(conv_args(g, in, filt, out), tiled_launch(p, g), true, 1, st);
        return;
      }
      break;
    case 2:  // Im2col: implicit GEMM (tensor cores when a TC precision is set)
      if (precision == TK_PREC_FP32_EXACT) {
        if (exact_run) launch_exact(conv_args(g, in, filt, out), exact_conv_default(g), true, 1, st);
      } else {
        launch_tc_conv(g, in, filt, out, precision, ws, st, phase);
      }
      return;
    case 3: {
      const int m = check_winograd(s, p);
      winograd_dev(g, m, precision, in, filt, out, ws, st, phase);
      return;
    }
    default:
      fail(TK_ERR_CONTRACT, "conv2d: unknown algorithm");
  }
  fail(TK_ERR_CAPABILITY, "conv2d: algorithm \"" + std::string(p->algo == 0 ? "naive" : "tiled") +
                              "\" is FP32-exact only; use im2col or winograd for tensor cores");
}

// Host-buffer conv: copy in, run, copy out -- pipelined over batch chunks
// so the host->device copy of chunk i+1, the convolution of chunk i and the
// device->host copy of chunk i-1 overlap (separate copy engines for the two
// directions; concurrency needs page-locked host buffers, pageable ones
// still work, serialised by the driver).  Chunks are equal slices of the
// batch (NHWC: a contiguous range of images), so one prepared workspace
// serves every chunk.
struct HostPipe {
  cudaStream_t compute = nullptr, copy_in = nullptr, copy_out = nullptr;
  static constexpr int kMaxChunks = 32;
  cudaEvent_t ready = nullptr, in_done[kMaxChunks] = {}, run_done[kMaxChunks] = {},
              out_done = nullptr;
  HostPipe() {
    TKB_CUDA(cudaStreamCreateWithFlags(&compute, cudaStreamNonBlocking));
    TKB_CUDA(cudaStreamCreateWithFlags(&copy_in, cudaStreamNonBlocking));
    TKB_CUDA(cudaStreamCreateWithFlags(&copy_out, cudaStreamNonBlocking));
    TKB_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    TKB_CUDA(cudaEventCreateWithFlags(&out_done, cudaEventDisableTiming));
    for (int i = 0; i < kMaxChunks; ++i) {
      TKB_CUDA(cudaEventCreateWithFlags(&in_done[i], cudaEventDisableTiming));
      TKB_CUDA(cudaEventCreateWithFlags(&run_done[i], cudaEventDisableTiming));
    }
  }
};

// One set of streams/events per (host thread, device): streams belong to
// the device current when they were created.
HostPipe& host_pipe() {
  host_stream();  // device + pool checks
  int dev = 0;
  TKB_CUDA(cudaGetDevice(&dev));
  thread_local std::map<int, std::unique_ptr<HostPipe>> pipes;
  std::unique_ptr<HostPipe>& p = pipes[dev];
  if (!p) p = std::make_unique<HostPipe>();
  return *p;
}

// Number of equal batch chunks: the largest divisor of the batch <= 8 that
// keeps every chunk's copies >= 2 MiB (a copy's fixed cost is ~10 us).
int pipeline_chunks(const ConvGeom& g) {
  const Experiments& xp = experiments();
  const int max_chunks = xp.pipe_chunks > 0 ? std::min(xp.pipe_chunks, HostPipe::kMaxChunks) : 8;
  const size_t min_bytes = xp.pipe_min_kb > 0 ? (size_t)xp.pipe_min_kb << 10 : (2u << 20);
  const size_t per_image = 4 * ((size_t)g.H * g.W * g.C + (size_t)g.OH * g.OW * g.K);
  for (int n = max_chunks; n > 1; --n)
    if (g.N % n == 0 && per_image * (size_t)(g.N / n) >= min_bytes) return n;
  return 1;
}

void conv_host(const tilekit::ConvShape& s, const tk_conv_params* p, int precision,
               const float* in, const float* filt, float* out) {
  const ConvGeom g = conv_geom(s);
  if (tc_knobs().io != 0)
    fail(TK_ERR_CAPABILITY, "conv2d: bf16 activations (io flags) apply to the device-buffer calls; "
                            "the host-buffer calls take the reference's fp32 tensors");
  if (p->algo == 1) check_tiled_params(s, p);
  if (p->algo == 3) check_winograd(s, p);
  HostPipe& hp = host_pipe();
  const int chunks = pipeline_chunks(g);
  tilekit::ConvShape cs = s;
  cs.batch = s.batch / (size_t)chunks;
  const ConvGeom cg = conv_geom(cs);
  const size_t in_chunk = in_elems(cg), out_chunk = out_elems(cg);
  cudaStream_t st = hp.compute;
  {
    DevBuf din(4 * in_elems(g), st), dfl(4 * filt_elems(g), st), dout(4 * out_elems(g), st);
    DevBuf ws(conv_workspace(cg, p, precision), st);
    try {
      h2d(dfl.p, filt, 4 * filt_elems(g), st);
      conv_dev(cs, p, precision, nullptr, dfl.f(), nullptr, ws.p, st, kConvPrepare);
      TKB_CUDA(cudaEventRecord(hp.ready, st));  // allocations exist from here on
      TKB_CUDA(cudaStreamWaitEvent(hp.copy_in, hp.ready, 0));
      for (int i = 0; i < chunks; ++i) {
        h2d(din.f() + i * in_chunk, in + i * in_chunk, 4 * in_chunk, hp.copy_in);
        TKB_CUDA(cudaEventRecord(hp.in_done[i], hp.copy_in));
        TKB_CUDA(cudaStreamWaitEvent(st, hp.in_done[i], 0));
        conv_dev(cs, p, precision, din.f() + i * in_chunk, dfl.f(), dout.f() + i * out_chunk,
                 ws.p, st, kConvRun);
        TKB_CUDA(cudaEventRecord(hp.run_done[i], st));
        TKB_CUDA(cudaStreamWaitEvent(hp.copy_out, hp.run_done[i], 0));
        d2h(out + i * out_chunk, dout.f() + i * out_chunk, 4 * out_chunk, hp.copy_out);
      }
      TKB_CUDA(cudaEventRecord(hp.out_done, hp.copy_out));
      TKB_CUDA(cudaStreamWaitEvent(st, hp.out_done, 0));  // frees are ordered after the copies
    } catch (...) {
      // No queued copy may touch the caller's host buffers (or the device
      // buffers freed below) after the error is reported.
      cudaStreamSynchronize(hp.copy_in);
      cudaStreamSynchronize(st);
      cudaStreamSynchronize(hp.copy_out);
      throw;
    }
  }
  finish(st);
}

}  // namespace

void note_launch(int n) { g_launches += (uint64_t)n; }

}  // namespace tkb


namespace tkb {
namespace {

struct EventTimer {
  cudaEvent_t a = nullptr, b = nullptr;
  EventTimer() {
    TKB_CUDA(cudaEventCreate(&a));
    TKB_CUDA(cudaEventCreate(&b));
  }
  ~EventTimer() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

template <typename Run>
void time_samples(Run&& run, int warmup, int samples, int64_t* ns, cudaStream_t st) {
  if (samples < 1 || !ns) fail(TK_ERR_CONTRACT, "bench: samples must be >= 1 with an output array");
  for (int i = 0; i < warmup; ++i) run();
  TKB_CUDA(cudaStreamSynchronize(st));
  EventTimer t;
  for (int i = 0; i < samples; ++i) {
    TKB_CUDA(cudaEventRecord(t.a, st));
    run();
    TKB_CUDA(cudaEventRecord(t.b, st));
    TKB_CUDA(cudaEventSynchronize(t.b));
    float ms = 0.0f;
    TKB_CUDA(cudaEventElapsedTime(&ms, t.a, t.b));
    ns[i] = (int64_t)((double)ms * 1.0e6);
  }
}

}  // namespace
}  // namespace tkb

using namespace tkb;

extern "C" {

const char* tk_last_error(void) { return g_error.c_str(); }
int tk_abi_version(void) { return TK_ABI_VERSION; }
int tk_device_count(void) { return usable_devices(); }
uint64_t tk_launch_count(void) { return g_launches.load(); }

int tk_synchronize(void) {
  return guarded([&] {
    require_gpu();
    TKB_CUDA(cudaDeviceSynchronize());
  });
}

int tk_b200_device_spec(tk_device_spec* out) {
  return guarded([&] {
    if (!out) fail(TK_ERR_CONTRACT, "tk_b200_device_spec: out must not be NULL");
    static char name[256] = "NVIDIA B200 (nominal)";
    tk_device_spec s{name, 128, 232448, 148, 255, 1024};
    if (usable_devices() > 0) {
      int dev = 0;
      TKB_CUDA(cudaGetDevice(&dev));
      cudaDeviceProp prop{};
      TKB_CUDA(cudaGetDeviceProperties(&prop, dev));
      std::snprintf(name, sizeof name, "%s", prop.name);
      s.local_memory_bytes = prop.sharedMemPerBlockOptin;
      s.compute_units = (size_t)prop.multiProcessorCount;
      s.max_workgroup_size = (size_t)prop.maxThreadsPerBlock;
    }
    *out = s;
  });
}

int tk_validate_gemm_config(const tk_gemm_config* cfg, const tk_device_spec* dev, int* ok,
                            char* msg, size_t cap) {
  return guarded([&] {
    if (!cfg || !dev || !ok) fail(TK_ERR_CONTRACT, "tk_validate_gemm_config: NULL argument");
    const auto v = tilekit::validate_config(gemm_config(cfg), device_spec(dev), {});
    *ok = v.ok ? 1 : 0;
    if (msg && cap) std::snprintf(msg, cap, "%s", v.summary().c_str());
  });
}

int tk_local_mem_elems(const tk_gemm_config* cfg, const tk_device_spec* dev, size_t* elems) {
  return guarded([&] {
    if (!cfg || !dev || !elems) fail(TK_ERR_CONTRACT, "tk_local_mem_elems: NULL argument");
    *elems = tilekit::local_mem_elems(gemm_config(cfg), device_spec(dev));
  });
}

int tk_gemm_tiled(const tk_gemm_shape* shape, const tk_gemm_config* cfg, const tk_device_spec* dev,
                  const float* a, const float* b, const float* c, float* out) {
  return guarded([&] {
    const tilekit::GemmShape g = gemm_shape(shape);
    if (!cfg || !dev) fail(TK_ERR_CONTRACT, "gemm_tiled: config and device must not be NULL");
    const tilekit::GemmConfig gc = gemm_config(cfg);
    const auto verdict = tilekit::validate_config(gc, device_spec(dev), g);
    if (!verdict.ok)
      fail(TK_ERR_CONFIG, "gemm_tiled: config \"" + gc.name() + "\" rejected: " + verdict.summary());
    if (gc.k_step == 0) fail(TK_ERR_CONFIG, "gemm_tiled: k_step must be positive");
    const ExactLaunch L = exact_launch_of(gc);
    cudaStream_t st = host_stream();
    const size_t na = g.m * g.k, nb = g.k * g.n, nc = g.m * g.n;
    const bool read_c = g.beta != 0.0f;
    DevBuf da(4 * na, st), db(4 * nb, st), dc(read_c ? 4 * nc : 0, st), dd(4 * nc, st);
    h2d(da.p, a, 4 * na, st);
    h2d(db.p, b, 4 * nb, st);
    if (read_c) h2d(dc.p, c, 4 * nc, st);
    launch_exact(gemm_args(g, da.f(), db.f(), dc.f(), dd.f()), L, false, 1, st);
    d2h(out, dd.p, 4 * nc, st);
    finish(st);
  });
}

int tk_gemm_naive(const tk_gemm_shape* shape, const float* a, const float* b, const float* c,
                  float* out) {
  return guarded([&] {
    const tilekit::GemmShape g = gemm_shape(shape);
    cudaStream_t st = host_stream();
    const size_t na = g.m * g.k, nb = g.k * g.n, nc = g.m * g.n;
    const bool read_c = g.beta != 0.0f;
    DevBuf da(4 * na, st), db(4 * nb, st), dc(read_c ? 4 * nc : 0, st), dd(4 * nc, st);
    h2d(da.p, a, 4 * na, st);
    h2d(db.p, b, 4 * nb, st);
    if (read_c) h2d(dc.p, c, 4 * nc, st);
    launch_exact(gemm_args(g, da.f(), db.f(), dc.f(), dd.f()), exact_auto((long long)g.m, (long long)g.n), false, 1,
                 st);
    d2h(out, dd.p, 4 * nc, st);
    finish(st);
  });
}

int tk_gemm_plan_info(const tk_gemm_shape* shape, const tk_gemm_config* cfg,
                      const tk_exec_options* opts, tk_gemm_plan* out) {
  return guarded([&] {
    if (!out) fail(TK_ERR_CONTRACT, "gemm_plan_info: out must not be NULL");
    KnobScope knobs(opts);
    const tilekit::GemmShape g = gemm_shape(shape);
    const int prec = precision_of(opts);
    std::memset(out, 0, sizeof(*out));
    out->requested_precision = prec;
    out->splits = 1;
    out->cta_group = 1;
    if (prec == TK_PREC_FP32_EXACT) {
      const ExactLaunch L = cfg ? exact_launch_of(gemm_config(cfg)) : exact_auto((long long)g.m, (long long)g.n);
      out->kernel = TK_KERNEL_EXACT;
      out->precision = TK_PREC_FP32_EXACT;
      out->tile_m = L.h * L.r;
      out->tile_n = L.w * L.c;
      out->a_in_place = out->b_in_place = 1;
      out->k_depth = (int)g.k;
      return;
    }
    bool hit = false;
    const int tile = tuned_gemm_tile(g, opts, &hit);
    TcGemmPlan pl;
    launch_tc_colmajor_gemm(g.m, g.n, g.k, g.alpha, g.beta, g.op_a == tilekit::Op::Transpose,
                            g.op_b == tilekit::Op::Transpose, nullptr, nullptr,
                            g.beta != 0.0f ? reinterpret_cast<const float*>(16) : nullptr, nullptr,
                            prec, tile, nullptr, &pl);
    out->kernel = TK_KERNEL_TC_PLAIN;
    out->precision = prec;
    out->cta_group = pl.cta_group;
    out->tile_m = pl.tile_m;
    out->tile_n = pl.tile_n;
    out->splits = pl.splits;
    out->tail_pieces = pl.tail_pieces;
    out->a_in_place = pl.a_in_place;
    out->b_in_place = pl.b_in_place;
    out->k_depth = pl.k_depth;
    out->tuned = hit ? 1 : 0;
  });
}

int tk_gemm_dev(const tk_gemm_shape* shape, const tk_gemm_config* cfg, const tk_exec_options* opts,
                const float* d_a, const float* d_b, const float* d_c, float* d_out, void* stream) {
  return guarded([&] {
    KnobScope knobs(opts);
    require_gpu();
    const tilekit::GemmShape g = gemm_shape(shape);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int prec = precision_of(opts);
    if (tc_knobs().io != 0 && (tc_knobs().io != TK_IO_IN_BF16 || prec != TK_PREC_BF16))
      fail(TK_ERR_CAPABILITY, "gemm: io flags: bf16 operands (TK_IO_IN_BF16) with BF16 precision "
                              "only; C and the output stay fp32");
    if (prec == TK_PREC_FP32_EXACT) {
      const ExactLaunch L = cfg ? exact_launch_of(gemm_config(cfg)) : exact_auto((long long)g.m, (long long)g.n);
      launch_exact(gemm_args(g, d_a, d_b, d_c, d_out), L, false, 1, st);
    } else {
      const int tile = tuned_gemm_tile(g, opts);
      launch_tc_colmajor_gemm(g.m, g.n, g.k, g.alpha, g.beta, g.op_a == tilekit::Op::Transpose,
                              g.op_b == tilekit::Op::Transpose, d_a, d_b, d_c, d_out, prec, tile,
                              st);
    }
  });
}

int tk_gemm_ex(const tk_gemm_shape* shape, const tk_exec_options* opts, const float* a,
               const float* b, const float* c, float* out) {
  return guarded([&] {
    KnobScope knobs(opts);
    if (tc_knobs().io != 0)
      fail(TK_ERR_CAPABILITY, "gemm: io flags apply to the device-buffer call (tk_gemm_dev)");
    const tilekit::GemmShape g = gemm_shape(shape);
    cudaStream_t st = host_stream();
    const size_t na = g.m * g.k, nb = g.k * g.n, nc = g.m * g.n;
    const bool read_c = g.beta != 0.0f;
    DevBuf da(4 * na, st), db(4 * nb, st), dc(read_c ? 4 * nc : 0, st), dd(4 * nc, st);
    h2d(da.p, a, 4 * na, st);
    h2d(db.p, b, 4 * nb, st);
    if (read_c) h2d(dc.p, c, 4 * nc, st);
    const int prec = precision_of(opts);
    if (prec == TK_PREC_FP32_EXACT)
      launch_exact(gemm_args(g, da.f(), db.f(), dc.f(), dd.f()), exact_auto((long long)g.m, (long long)g.n), false, 1,
                 st);
    else
      launch_tc_colmajor_gemm(g.m, g.n, g.k, g.alpha, g.beta, g.op_a == tilekit::Op::Transpose,
                              g.op_b == tilekit::Op::Transpose, da.f(), db.f(), dc.f(), dd.f(),
                              prec, tuned_gemm_tile(g, opts), st);
    d2h(out, dd.p, 4 * nc, st);
    finish(st);
  });
}

int tk_gemm_batched_strided(const float* a, size_t sa, const float* b, size_t sb, float* c,
                            size_t sc, size_t batch, size_t m, size_t n, size_t k,
                            uint64_t* multiplies) {
  return guarded([&] {
    if (multiplies) *multiplies = (uint64_t)batch * m * n * k;
    if (batch == 0 || m == 0 || n == 0) return;
    if (m > 2147483647ull || n > 2147483647ull || k > 2147483647ull || batch > 65535ull)
      fail(TK_ERR_CAPABILITY, "gemm_batched_strided: dimensions exceed the 32-bit index range");
    cudaStream_t st = host_stream();
    // Span of each operand: the last batch member's end.
    const size_t ea = (batch - 1) * sa + m * k, eb = (batch - 1) * sb + k * n,
                 ec = (batch - 1) * sc + m * n;
    DevBuf da(4 * ea, st), db(4 * eb, st), dc(4 * ec, st);
    h2d(da.p, a, 4 * ea, st);
    h2d(db.p, b, 4 * eb, st);
    if (ec > batch * m * n) h2d(dc.p, c, 4 * ec, st);  // keep gaps between members intact
    if (k == 0) {
      for (size_t g = 0; g < batch; ++g)
        TKB_CUDA(cudaMemsetAsync(dc.f() + g * sc, 0, 4 * m * n, st));
    } else {
      ExactArgs p{};
      p.M = (int)m;
      p.N = (int)n;
      p.K = (int)k;
      p.a = da.f();
      p.a_sm = 1;
      p.a_sk = (long long)m;
      p.a_batch = (long long)sa;
      p.b = db.f();
      p.b_sk = 1;
      p.b_sn = (long long)k;
      p.b_batch = (long long)sb;
      p.d = dc.f();
      p.d_sm = 1;
      p.d_sn = (long long)m;
      p.d_batch = (long long)sc;
      p.alpha = 1.0f;
      p.tx_on_m = 1;
      launch_exact(p, exact_auto((long long)(m * batch), (long long)n), false, (int)batch, st);
    }
    d2h(c, dc.p, 4 * ec, st);
    finish(st);
  });
}

int tk_gemm_batched_strided_dev(const float* d_a, size_t sa, const float* d_b, size_t sb,
                                float* d_c, size_t sc, size_t batch, size_t m, size_t n, size_t k,
                                const tk_exec_options* opts, void* stream) {
  return guarded([&] {
    KnobScope knobs(opts);
    require_gpu();
    if (batch == 0 || m == 0 || n == 0) return;  // nothing to write (reference: 0 multiplies)
    if (precision_of(opts) != TK_PREC_FP32_EXACT) {  // tensor cores (TF32 / BF16 / 3xTF32)
      if (tc_knobs().io != 0) fail(TK_ERR_CAPABILITY, "gemm_batched_strided: io flags not supported");
      if (k == 0) {  // C_g = 0
        for (size_t g = 0; g < batch; ++g)
          TKB_CUDA(cudaMemsetAsync(d_c + g * sc, 0, m * n * 4, static_cast<cudaStream_t>(stream)));
        return;
      }
      launch_tc_batched_colmajor(m, n, k, batch, d_a, (long long)sa, d_b, (long long)sb, d_c,
                                 (long long)sc, precision_of(opts), static_cast<cudaStream_t>(stream));
      return;
    }
    if (m > 2147483647ull || n > 2147483647ull || k > 2147483647ull || batch > 65535ull)
      fail(TK_ERR_CAPABILITY, "gemm_batched_strided: dimensions exceed the 32-bit index range");
    ExactArgs p{};
    p.M = (int)m;
    p.N = (int)n;
    p.K = (int)k;
    p.a = d_a;
    p.a_sm = 1;
    p.a_sk = (long long)m;
    p.a_batch = (long long)sa;
    p.b = d_b;
    p.b_sk = 1;
    p.b_sn = (long long)k;
    p.b_batch = (long long)sb;
    p.d = d_c;
    p.d_sm = 1;
    p.d_sn = (long long)m;
    p.d_batch = (long long)sc;
    p.alpha = 1.0f;
    p.tx_on_m = 1;
    launch_exact(p, exact_auto((long long)(m * batch), (long long)n), false, (int)batch,
                 static_cast<cudaStream_t>(stream));
  });
}

int tk_conv2d(const tk_conv_shape* shape, const tk_conv_params* params, const float* in,
              const float* filt, float* out) {
  return guarded([&] {
    if (!params) fail(TK_ERR_CONTRACT, "conv2d: params must not be NULL");
    // Selector semantics.  The default conv2d_im2col overload names
    // 4x4_8x8_noloc on a generic 64-byte-line device (conv.hpp:353-362),
    // a config that always validates; its bits do not depend on the tile,
    // so the library's own exact tile runs it (exact_conv_default).  A
    // caller that names a config goes through tk_conv2d_im2col.
    conv_host(conv_shape(shape), params, TK_PREC_FP32_EXACT, in, filt, out);
  });
}

int tk_conv2d_ex(const tk_conv_shape* shape, const tk_conv_params* params,
                 const tk_exec_options* opts, const float* in, const float* filt, float* out) {
  return guarded([&] {
    KnobScope knobs(opts);
    if (!params) fail(TK_ERR_CONTRACT, "conv2d: params must not be NULL");
    apply_tuned_conv(conv_shape(shape), params, opts);
    conv_host(conv_shape(shape), params, precision_of(opts), in, filt, out);
  });
}

int tk_conv2d_naive(const tk_conv_shape* shape, const float* in, const float* filt, float* out) {
  tk_conv_params p{0, 1, 1, 1, 1};
  return tk_conv2d_ex(shape, &p, nullptr, in, filt, out);
}

int tk_conv2d_tiled(const tk_conv_shape* shape, const tk_conv_params* params, const float* in,
                    const float* filt, float* out) {
  return guarded([&] {
    if (!params) fail(TK_ERR_CONTRACT, "conv2d_tiled: params must not be NULL");
    tk_conv_params p = *params;
    p.algo = 1;
    conv_host(conv_shape(shape), &p, TK_PREC_FP32_EXACT, in, filt, out);
  });
}

int tk_conv2d_im2col(const tk_conv_shape* shape, const tk_gemm_config* cfg,
                     const tk_device_spec* dev, const float* in, const float* filt, float* out) {
  return guarded([&] {
    const tilekit::ConvShape s = conv_shape(shape);
    const ConvGeom g = conv_geom(s);
    if (!cfg || !dev) fail(TK_ERR_CONTRACT, "conv2d_im2col: config and device must not be NULL");
    // The reference validates the patch-matrix GEMM through gemm_tiled.
    const tilekit::GemmConfig gc = gemm_config(cfg);
    tilekit::GemmShape gs;
    gs.m = (size_t)g.N * g.OH * g.OW;
    gs.n = (size_t)g.K;
    gs.k = (size_t)g.R * g.S * g.C;
    const auto verdict = tilekit::validate_config(gc, device_spec(dev), gs);
    if (!verdict.ok)
      fail(TK_ERR_CONFIG, "gemm_tiled: config \"" + gc.name() + "\" rejected: " + verdict.summary());
    if (gc.k_step == 0) fail(TK_ERR_CONFIG, "gemm_tiled: k_step must be positive");
    const ExactLaunch L = exact_launch_of(gc);
    cudaStream_t st = host_stream();
    DevBuf din(4 * in_elems(g), st), dfl(4 * filt_elems(g), st), dout(4 * out_elems(g), st);
    h2d(din.p, in, 4 * in_elems(g), st);
    h2d(dfl.p, filt, 4 * filt_elems(g), st);
    launch_exact(conv_args(g, din.f(), dfl.f(), dout.f()), L, true, 1, st);
    d2h(out, dout.p, 4 * out_elems(g), st);
    finish(st);
  });
}

int tk_conv2d_winograd(const tk_conv_shape* shape, const tk_conv_params* params, const float* in,
                       const float* filt, float* out, uint64_t* mults, size_t* tiles) {
  return guarded([&] {
    if (!params) fail(TK_ERR_CONTRACT, "conv2d_winograd: params must not be NULL");
    const tilekit::ConvShape s = conv_shape(shape);
    const ConvGeom g = conv_geom(s);
    tk_conv_params p = *params;
    p.algo = 3;
    const int m = check_winograd(s, &p);
    conv_host(s, &p, TK_PREC_FP32_EXACT, in, filt, out);
    const WinoGeom w = wino_geom(g, m);
    if (mults) *mults = (uint64_t)w.t * w.t * w.tiles * w.K * w.C;
    if (tiles) *tiles = (size_t)w.tiles;
  });
}

int tk_im2col(const tk_conv_shape* shape, const float* in, float* patches) {
  return guarded([&] {
    const ConvGeom g = conv_geom(conv_shape(shape));
    cudaStream_t st = host_stream();
    const size_t np = (size_t)g.N * g.OH * g.OW * g.R * g.S * g.C;
    DevBuf din(4 * in_elems(g), st), dp(4 * np, st);
    h2d(din.p, in, 4 * in_elems(g), st);
    launch_im2col(g, din.f(), dp.f(), st);
    d2h(patches, dp.p, 4 * np, st);
    finish(st);
  });
}

int tk_im2col_dev(const tk_conv_shape* shape, const float* d_in, float* d_patches, void* stream) {
  return guarded([&] {
    require_gpu();
    launch_im2col(conv_geom(conv_shape(shape)), d_in, d_patches, static_cast<cudaStream_t>(stream));
  });
}

int tk_filter_matrix(size_t r, size_t s, size_t c, size_t k, const float* filt, float* mat) {
  return guarded([&] {
    if (!r || !s || !c || !k) fail(TK_ERR_SHAPE, "filter_matrix: dimensions must be positive");
    cudaStream_t st = host_stream();
    const size_t rows = r * s * c, n = rows * k;
    DevBuf df(4 * n, st), dm(4 * n, st);
    h2d(df.p, filt, 4 * n, st);
    launch_transpose(df.f(), dm.f(), (long long)rows, (long long)k, st);  // [rows][k] -> col-major
    d2h(mat, dm.p, 4 * n, st);
    finish(st);
  });
}

int tk_conv2d_workspace_size(const tk_conv_shape* shape, const tk_conv_params* params,
                             const tk_exec_options* opts, size_t* bytes) {
  return guarded([&] {
    KnobScope knobs(opts);
    if (!params || !bytes) fail(TK_ERR_CONTRACT, "conv2d_workspace_size: NULL argument");
    const tilekit::ConvShape s = conv_shape(shape);
    if (params->algo == 3) check_winograd(s, params);
    apply_tuned_conv(s, params, opts);
    *bytes = conv_workspace(conv_geom(s), params, precision_of(opts));
  });
}

int tk_conv2d_dev(const tk_conv_shape* shape, const tk_conv_params* params,
                  const tk_exec_options* opts, const float* d_in, const float* d_filt,
                  float* d_out, void* d_ws, size_t ws_bytes, void* stream) {
  return guarded([&] {
    KnobScope knobs(opts);
    require_gpu();
    if (!params) fail(TK_ERR_CONTRACT, "conv2d: params must not be NULL");
    const tilekit::ConvShape s = conv_shape(shape);
    const int prec = precision_of(opts);
    if (params->algo == 3) check_winograd(s, params);
    apply_tuned_conv(s, params, opts);
    const size_t need = conv_workspace(conv_geom(s), params, prec);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (need && (!d_ws || ws_bytes < need)) {
      keep_pool_memory();
      Scratch tmp(st, kScratchConvWs, need);
      conv_dev(s, params, prec, d_in, d_filt, d_out, tmp.get(), st);
    } else {
      conv_dev(s, params, prec, d_in, d_filt, d_out, d_ws, st);
    }
  });
}

// Two-phase device convolution: prepare (filter-side work into the
// workspace) then run.  The phases may go to different streams as long as
// run is ordered after prepare on the same workspace.
static int conv_phase_dev(const tk_conv_shape* shape, const tk_conv_params* params,
                          const tk_exec_options* opts, const float* d_in, const float* d_filt,
                          float* d_out, void* d_ws, size_t ws_bytes, void* stream, int phase) {
  return guarded([&] {
    KnobScope knobs(opts);
    require_gpu();
    if (!params) fail(TK_ERR_CONTRACT, "conv2d: params must not be NULL");
    const tilekit::ConvShape s = conv_shape(shape);
    const int prec = precision_of(opts);
    if (params->algo == 3) check_winograd(s, params);
    if (params->algo == 1) check_tiled_params(s, params);
    apply_tuned_conv(s, params, opts);
    const size_t need = conv_workspace(conv_geom(s), params, prec);
    if (need && (!d_ws || ws_bytes < need))
      fail(TK_ERR_CONTRACT, "conv2d prepare/run: a workspace of " + std::to_string(need) +
                                " bytes is required (tk_conv2d_workspace_size)");
    conv_dev(s, params, prec, d_in, d_filt, d_out, d_ws, static_cast<cudaStream_t>(stream), phase);
  });
}

int tk_conv2d_prepare_dev(const tk_conv_shape* shape, const tk_conv_params* params,
                          const tk_exec_options* opts, const float* d_filt, void* d_ws,
                          size_t ws_bytes, void* stream) {
  return conv_phase_dev(shape, params, opts, nullptr, d_filt, nullptr, d_ws, ws_bytes, stream,
                        kConvPrepare);
}

int tk_conv2d_run_dev(const tk_conv_shape* shape, const tk_conv_params* params,
                      const tk_exec_options* opts, const float* d_in, const float* d_filt,
                      float* d_out, void* d_ws, size_t ws_bytes, void* stream) {
  return conv_phase_dev(shape, params, opts, d_in, d_filt, d_out, d_ws, ws_bytes, stream,
                        kConvRun);
}

int tk_conv2d_plan_info(const tk_conv_shape* shape, const tk_conv_params* params,
                        const tk_exec_options* opts, tk_conv_plan_info* out) {
  return guarded([&] {
    KnobScope knobs(opts);
    if (!params || !out) fail(TK_ERR_CONTRACT, "conv2d_plan_info: NULL argument");
    const tilekit::ConvShape s = conv_shape(shape);
    const ConvGeom g = conv_geom(s);
    const int prec = precision_of(opts);
    check_io(params, prec);
    tk_conv_plan_info r{};
    r.requested_precision = prec;
    r.tuned = apply_tuned_conv(s, params, opts) ? 1 : 0;
    r.cta_group = 1;
    r.splits = 1;
    r.imgs = 1;
    auto exact = [&](const ExactLaunch& L) {
      r.kernel = TK_KERNEL_EXACT;
      r.precision = TK_PREC_FP32_EXACT;
      r.tile_m = L.h * L.r;
      r.tile_n = L.w * L.c;
    };
    switch (params->algo) {
      case 0:
      case 2:
        if (prec == TK_PREC_FP32_EXACT) {
          exact(exact_conv_default(g));
          break;
        }
        if (params->algo == 0)
          fail(TK_ERR_CAPABILITY, "conv2d: algorithm \"naive\" is FP32-exact only; use im2col or "
                                  "winograd for tensor cores");
        {
          const TcConvInfo t = tc_conv_info(g, prec);
          r.kernel = t.narrow ? TK_KERNEL_TC_HALO_NARROW : t.mode;
          r.precision = t.precision;
          r.cta_group = t.cta_group;
          r.tile_m = t.tile_m;
          r.tile_n = t.tile_n;
          r.splits = t.splits;
          r.tail_pieces = t.tail_pieces;
          r.imgs = t.imgs;
          r.flat = t.flat;
          r.box_w = t.box_w;
          r.box_h = t.box_h;
          r.halo_resident = t.halo_resident;
        }
        break;
      case 1:
        check_tiled_params(s, params);
        if (prec != TK_PREC_FP32_EXACT)
          fail(TK_ERR_CAPABILITY, "conv2d: algorithm \"tiled\" is FP32-exact only; use im2col or "
                                  "winograd for tensor cores");
        exact(tiled_launch(params, g));
        break;
      case 3: {
        const int m = check_winograd(s, params);
        r.kernel = TK_KERNEL_WINOGRAD;
        r.winograd_m = m;
        const bool tc = prec != TK_PREC_FP32_EXACT && g.C % 4 == 0;
        // The transform-domain operands are fp32 scratch: kind::tf32 for
        // every tensor-core request (3xTF32 splits them).
        r.precision = !tc ? TK_PREC_FP32_EXACT : prec == TK_PREC_3XTF32 ? TK_PREC_3XTF32 : TK_PREC_TF32;
        break;
      }
      default:
        fail(TK_ERR_CONTRACT, "conv2d: unknown algorithm");
    }
    *out = r;
  });
}

int tk_tuning_db_load(const char* path, const char* device, size_t* records) {
  return guarded([&] {
    if (!path) fail(TK_ERR_CONTRACT, "tuning_db_load: path must not be NULL");
    const size_t kept = tuning_db_load(path, device ? device : "");
    if (records) *records = kept;
  });
}

int tk_tuning_db_clear(void) {
  return guarded([&] { tuning_db_clear(); });
}

int tk_tuning_db_size(size_t* entries) {
  return guarded([&] {
    if (!entries) fail(TK_ERR_CONTRACT, "tuning_db_size: NULL argument");
    *entries = tuning_db_size();
  });
}

int tk_bench_gemm(const tk_gemm_shape* shape, const tk_gemm_config* cfg, const tk_exec_options* opts,
                  const float* a, const float* b, const float* c, int warmup, int samples,
                  int64_t* ns) {
  return guarded([&] {
    KnobScope knobs(opts);
    const tilekit::GemmShape g = gemm_shape(shape);
    cudaStream_t st = host_stream();
    const size_t na = g.m * g.k, nb = g.k * g.n, nc = g.m * g.n;
    const bool read_c = g.beta != 0.0f;
    DevBuf da(4 * na, st), db(4 * nb, st), dc(read_c ? 4 * nc : 0, st), dd(4 * nc, st);
    h2d(da.p, a, 4 * na, st);
    h2d(db.p, b, 4 * nb, st);
    if (read_c) h2d(dc.p, c, 4 * nc, st);
    const int prec = precision_of(opts);
    const ExactLaunch L = cfg ? exact_launch_of(gemm_config(cfg)) : exact_auto((long long)g.m, (long long)g.n);
    const int tile = tuned_gemm_tile(g, opts);
    auto run = [&] {
      if (prec == TK_PREC_FP32_EXACT) {
        launch_exact(gemm_args(g, da.f(), db.f(), dc.f(), dd.f()), L, false, 1, st);
      } else {
        launch_tc_colmajor_gemm(g.m, g.n, g.k, g.alpha, g.beta, g.op_a == tilekit::Op::Transpose,
                                g.op_b == tilekit::Op::Transpose, da.f(), db.f(), dc.f(), dd.f(),
                                prec, tile, st);
      }
    };
    time_samples(run, warmup, samples, ns, st);
  });
}

int tk_bench_conv2d(const tk_conv_shape* shape, const tk_conv_params* params,
                    const tk_exec_options* opts, const float* in, const float* filt, int warmup,
                    int samples, int64_t* ns) {
  return guarded([&] {
    KnobScope knobs(opts);
    if (!params) fail(TK_ERR_CONTRACT, "bench: params must not be NULL");
    const tilekit::ConvShape s = conv_shape(shape);
    const ConvGeom g = conv_geom(s);
    if (params->algo == 1) check_tiled_params(s, params);
    if (params->algo == 3) check_winograd(s, params);
    apply_tuned_conv(s, params, opts);
    const int prec = precision_of(opts);
    cudaStream_t st = host_stream();
    DevBuf din(4 * in_elems(g), st), dfl(4 * filt_elems(g), st), dout(4 * out_elems(g), st);
    DevBuf ws(conv_workspace(g, params, prec), st);
    h2d(din.p, in, 4 * in_elems(g), st);
    h2d(dfl.p, filt, 4 * filt_elems(g), st);
    auto run = [&] { conv_dev(s, params, prec, din.f(), dfl.f(), dout.f(), ws.p, st); };
    time_samples(run, warmup, samples, ns, st);
  });
}

}  // extern "C"

/*
 * tk_oracle.c -- CPU restatement of the tilekit hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the B200
 * kernels in paper_1904_05347_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path never links or calls it.
 *
 * Parity is PINNED: tests/test_oracle.py checks every function here against
 * (a) the golden vectors of the reference's own tests (test_gemm.cpp,
 * test_conv.cpp, test_winograd.cpp) and (b) fixtures produced by the
 * reference headers themselves (tests/golden/make_golden.py compiles
 * oracle/ref_shim.cpp against /root/reference/proj/include).
 *
 * Must be compiled with -ffp-contract=off: the reference relies on separate
 * multiply and add roundings.
 *
 * All matrices are column-major (element (i,j) at i + j*rows,
 * tensor.hpp:12-14 of the reference); 4-D tensors are row-major over their
 * four dimensions (NHWC inputs, HWCK filters).
 */
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define TKO_API __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* Random fill: std::mt19937_64 + std::uniform_real_distribution<float>(-1,1)
 * as libstdc++ 13 implements them (reference tests/helpers.hpp:11-15 and
 * tuner.hpp:293-297).  generate_canonical<float,24> draws one 64-bit word,
 * converts it to float, scales by 2^-64 and clamps below 1.              */
/* ------------------------------------------------------------------------ */

typedef struct {
  uint64_t s[312];
  int idx;
} mt64_t;

static void mt64_seed(mt64_t* g, uint64_t seed) {
  g->s[0] = seed;
  for (int i = 1; i < 312; ++i) {
    uint64_t p = g->s[i - 1];
    g->s[i] = 6364136223846793005ULL * (p ^ (p >> 62)) + (uint64_t)i;
  }
  g->idx = 312;
}

static void mt64_twist(mt64_t* g) {
  const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
  for (int i = 0; i < 312; ++i) {
    uint64_t y = (g->s[i] & upper) | (g->s[(i + 1) % 312] & lower);
    uint64_t v = g->s[(i + 156) % 312] ^ (y >> 1);
    if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
    g->s[i] = v;
  }
  g->idx = 0;
}

static uint64_t mt64_next(mt64_t* g) {
  if (g->idx >= 312) mt64_twist(g);
  uint64_t z = g->s[g->idx++];
  z ^= (z >> 29) & 0x5555555555555555ULL;
  z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
  z ^= (z << 37) & 0xFFF7EEE000000000ULL;
  z ^= (z >> 43);
  return z;
}

TKO_API void tko_fill_random(float* data, size_t count, uint64_t seed) {
  mt64_t* g = (mt64_t*)malloc(sizeof(mt64_t));
  mt64_seed(g, seed);
  const float two64 = 18446744073709551616.0f;
  for (size_t i = 0; i < count; ++i) {
    float u = (float)mt64_next(g) / two64;
    if (u >= 1.0f) u = nextafterf(1.0f, 0.0f);
    float scaled = u * 2.0f;
    data[i] = scaled + -1.0f;
  }
  free(g);
}

/* FNV-1a over the problem key (tuner.hpp:284-291). */
TKO_API uint64_t tko_fnv1a(const char* text) {
  uint64_t h = 1469598103934665603ULL;
  for (const unsigned char* p = (const unsigned char*)text; *p; ++p) {
    h ^= *p;
    h *= 1099511628211ULL;
  }
  return h;
}

/* ------------------------------------------------------------------------ */
/* GEMM                                                                     */
/* ------------------------------------------------------------------------ */

/* gemm_naive (gemm.hpp:194-213).  out(i,j) = alpha*r (+ beta*C(i,j) when
 * beta != 0), r = sum over ascending kk of OPa(A)(i,kk)*OPb(B)(kk,j).
 * C is not read when beta == 0.  The loop nest is reordered for cache
 * behaviour but each element's own summation order is unchanged, so the
 * result is bit-identical to the reference loop. */
TKO_API void tko_gemm_naive(size_t m, size_t n, size_t k, float alpha,
                            float beta, int trans_a, int trans_b,
                            const float* a, const float* b, const float* c,
                            float* out) {
  const size_t lda = trans_a ? k : m; /* rows of the stored A */
  const size_t ldb = trans_b ? n : k;
#pragma omp parallel
  {
    float* acc = (float*)malloc(sizeof(float) * (m ? m : 1));
#pragma omp for schedule(static)
    for (size_t j = 0; j < n; ++j) {
      for (size_t i = 0; i < m; ++i) acc[i] = 0.0f;
      if (!trans_a) {
        for (size_t kk = 0; kk < k; ++kk) {
          const float bv = trans_b ? b[j + kk * ldb] : b[kk + j * ldb];
          const float* acol = a + kk * lda;
          for (size_t i = 0; i < m; ++i) acc[i] += acol[i] * bv;
        }
      } else {
        for (size_t i = 0; i < m; ++i) {
          float r = 0.0f;
          const float* arow = a + i * lda; /* A stored k x m */
          for (size_t kk = 0; kk < k; ++kk) {
            const float bv = trans_b ? b[j + kk * ldb] : b[kk + j * ldb];
            r += arow[kk] * bv;
          }
          acc[i] = r;
        }
      }
      for (size_t i = 0; i < m; ++i) {
        const float r = acc[i];
        if (beta == 0.0f) {
          out[i + j * m] = alpha * r;
        } else {
          const float p = alpha * r;
          const float q = beta * c[i + j * m];
          out[i + j * m] = p + q;
        }
      }
    }
    free(acc);
  }
}

/* gemm_batched_strided (gemm.hpp:451-479): C_g = A_g * B_g, packed
 * column-major, C zeroed first.  Returns the multiply count. */
TKO_API uint64_t tko_gemm_batched_strided(const float* a, size_t stride_a,
                                          const float* b, size_t stride_b,
                                          float* c, size_t stride_c,
                                          size_t batch, size_t m, size_t n,
                                          size_t k) {
#pragma omp parallel for schedule(static)
  for (size_t g = 0; g < batch; ++g) {
    const float* ag = a + g * stride_a;
    const float* bg = b + g * stride_b;
    float* cg = c + g * stride_c;
    for (size_t j = 0; j < n; ++j) {
      float* col = cg + j * m;
      for (size_t i = 0; i < m; ++i) col[i] = 0.0f;
      for (size_t kk = 0; kk < k; ++kk) {
        const float bj = bg[kk + j * k];
        const float* acol = ag + kk * m;
        for (size_t i = 0; i < m; ++i) col[i] += acol[i] * bj;
      }
    }
  }
  return (uint64_t)batch * m * n * k;
}

/* ------------------------------------------------------------------------ */
/* Convolution geometry (config.hpp:137-195)                                */
/* ------------------------------------------------------------------------ */

typedef struct {
  size_t batch, in_rows, in_cols, channels, features;
  size_t window_rows, window_cols, stride;
  int same; /* 1 = Padding::Same, 0 = Padding::Valid */
} tko_conv_shape;

static size_t out_extent(size_t in, size_t win, size_t stride, int same) {
  if (!same) return in < win ? 0 : (in - win) / stride + 1;
  return (in + stride - 1) / stride;
}

static ptrdiff_t pad_before(size_t in, size_t win, size_t stride, int same) {
  if (!same) return 0;
  size_t out = out_extent(in, win, stride, same);
  size_t span = (out > 0 ? (out - 1) * stride : 0) + win;
  size_t total = span > in ? span - in : 0;
  return (ptrdiff_t)(total / 2); /* smaller half first */
}

TKO_API size_t tko_out_rows(const tko_conv_shape* s) {
  return out_extent(s->in_rows, s->window_rows, s->stride, s->same);
}
TKO_API size_t tko_out_cols(const tko_conv_shape* s) {
  return out_extent(s->in_cols, s->window_cols, s->stride, s->same);
}
TKO_API ptrdiff_t tko_pad_top(const tko_conv_shape* s) {
  return pad_before(s->in_rows, s->window_rows, s->stride, s->same);
}
TKO_API ptrdiff_t tko_pad_left(const tko_conv_shape* s) {
  return pad_before(s->in_cols, s->window_cols, s->stride, s->same);
}

/* conv2d_naive (conv.hpp:74-113): one ordered sum per output over ascending
 * (x, y, c); out-of-range taps skipped.  The k loop is hoisted inside the
 * tap loops (vectorisable) without changing any element's summation order. */
TKO_API void tko_conv2d_naive(const tko_conv_shape* s, const float* in,
                              const float* filt, float* out) {
  const size_t oh_n = tko_out_rows(s), ow_n = tko_out_cols(s);
  const ptrdiff_t pr = tko_pad_top(s), pc = tko_pad_left(s);
  const size_t C = s->channels, K = s->features;
#pragma omp parallel for collapse(2) schedule(static)
  for (size_t n = 0; n < s->batch; ++n) {
    for (size_t oh = 0; oh < oh_n; ++oh) {
      for (size_t ow = 0; ow < ow_n; ++ow) {
        float* dst = out + ((n * oh_n + oh) * ow_n + ow) * K;
        for (size_t k = 0; k < K; ++k) dst[k] = 0.0f;
        for (size_t x = 0; x < s->window_rows; ++x) {
          const ptrdiff_t ih = (ptrdiff_t)(oh * s->stride + x) - pr;
          if (ih < 0 || ih >= (ptrdiff_t)s->in_rows) continue;
          for (size_t y = 0; y < s->window_cols; ++y) {
            const ptrdiff_t iw = (ptrdiff_t)(ow * s->stride + y) - pc;
            if (iw < 0 || iw >= (ptrdiff_t)s->in_cols) continue;
            const float* px =
                in + ((n * s->in_rows + (size_t)ih) * s->in_cols + (size_t)iw) * C;
            const float* fx = filt + (x * s->window_cols + y) * C * K;
            for (size_t c = 0; c < C; ++c) {
              const float v = px[c];
              const float* fk = fx + c * K;
              for (size_t k = 0; k < K; ++k) dst[k] += v * fk[k];
            }
          }
        }
      }
    }
  }
}

/* im2col (conv.hpp:255-300): patch matrix (N*OH*OW) x (R*S*C), column-major,
 * row (n*OH+oh)*OW+ow, column (x*S+y)*C+c, zero outside the input. */
TKO_API void tko_im2col(const tko_conv_shape* s, const float* in,
                        float* patches) {
  const size_t oh_n = tko_out_rows(s), ow_n = tko_out_cols(s);
  const ptrdiff_t pr = tko_pad_top(s), pc = tko_pad_left(s);
  const size_t rows = oh_n * ow_n * s->batch;
  const size_t C = s->channels;
#pragma omp parallel for collapse(2) schedule(static)
  for (size_t n = 0; n < s->batch; ++n) {
    for (size_t oh = 0; oh < oh_n; ++oh) {
      for (size_t ow = 0; ow < ow_n; ++ow) {
        const size_t row = (n * oh_n + oh) * ow_n + ow;
        for (size_t x = 0; x < s->window_rows; ++x) {
          const ptrdiff_t ih = (ptrdiff_t)(oh * s->stride + x) - pr;
          for (size_t y = 0; y < s->window_cols; ++y) {
            const ptrdiff_t iw = (ptrdiff_t)(ow * s->stride + y) - pc;
            const int inside = ih >= 0 && iw >= 0 && ih < (ptrdiff_t)s->in_rows &&
                               iw < (ptrdiff_t)s->in_cols;
            for (size_t c = 0; c < C; ++c) {
              const size_t col = (x * s->window_cols + y) * C + c;
              patches[row + col * rows] =
                  inside ? in[((n * s->in_rows + (size_t)ih) * s->in_cols +
                               (size_t)iw) * C + c]
                         : 0.0f;
            }
          }
        }
      }
    }
  }
}

/* filter_matrix (conv.hpp:304-317): HWCK -> column-major (R*S*C) x K. */
TKO_API void tko_filter_matrix(size_t r, size_t s, size_t c, size_t k,
                               const float* filt, float* mat) {
  const size_t rows = r * s * c;
  for (size_t i = 0; i < rows; ++i)
    for (size_t j = 0; j < k; ++j) mat[i + j * rows] = filt[i * k + j];
}

/* ------------------------------------------------------------------------ */
/* Winograd (winograd.hpp:50-301)                                           */
/* ------------------------------------------------------------------------ */

/* Cook-Toom matrices, row-major, exactly the reference's float constants
 * (winograd.hpp:62-77 for F(2x2,3x3), :86-107 for F(4x4,3x3)). */
static const float F2_BT[16] = {1, 0, -1, 0, 0, 1, 1, 0, 0, -1, 1, 0, 0, 1, 0, -1};
static const float F2_G[12] = {1, 0, 0, 0.5f, 0.5f, 0.5f, 0.5f, -0.5f, 0.5f, 0, 0, 1};
static const float F2_AT[8] = {1, 1, 1, 0, 0, 1, -1, -1};
static const float F4_BT[36] = {4, 0, -5, 0,  1, 0, 0, -4, -4, 1,  1, 0,
                                0, 4, -4, -1, 1, 0, 0, -2, -1, 2,  1, 0,
                                0, 2, -1, -2, 1, 0, 0, 4,  0,  -5, 0, 1};
static const float F4_G[18] = {1.0f / 4,  0,          0,
                               -1.0f / 6, -1.0f / 6,  -1.0f / 6,
                               -1.0f / 6, 1.0f / 6,   -1.0f / 6,
                               1.0f / 24, 1.0f / 12,  1.0f / 6,
                               1.0f / 24, -1.0f / 12, 1.0f / 6,
                               0,         0,          1};
static const float F4_AT[24] = {1, 1, 1,  1, 1,  0, 0, 1, -1, 2, -2, 0,
                                0, 1, 1,  4, 4,  0, 0, 1, -1, 8, -8, 1};

/* Copies a plan matrix (row-major) into dst; returns 0 if no plan. */
TKO_API int tko_winograd_plan(size_t m, size_t r, float* bt, float* g,
                              float* at) {
  if (r != 3) return 0;
  if (m == 2) {
    memcpy(bt, F2_BT, sizeof F2_BT);
    memcpy(g, F2_G, sizeof F2_G);
    memcpy(at, F2_AT, sizeof F2_AT);
    return 1;
  }
  if (m == 4) {
    memcpy(bt, F4_BT, sizeof F4_BT);
    memcpy(g, F4_G, sizeof F4_G);
    memcpy(at, F4_AT, sizeof F4_AT);
    return 1;
  }
  return 0;
}

/* transform_tile (winograd.hpp:125-147): dst (p x p) = T src T^T with T
 * p x q (row-major) and src q x q, two ordered passes. */
static void transform_tile(const float* t, size_t p, size_t q, const float* src,
                           float* dst) {
  float tmp[36];
  for (size_t i = 0; i < p; ++i)
    for (size_t j = 0; j < q; ++j) {
      float sum = 0.0f;
      for (size_t kk = 0; kk < q; ++kk) sum += t[i * q + kk] * src[kk * q + j];
      tmp[i * q + j] = sum;
    }
  for (size_t i = 0; i < p; ++i)
    for (size_t j = 0; j < p; ++j) {
      float sum = 0.0f;
      for (size_t kk = 0; kk < q; ++kk) sum += tmp[i * q + kk] * t[j * q + kk];
      dst[i * p + j] = sum;
    }
}

/* conv2d_winograd (winograd.hpp:169-301), stride 1, m in {2,4}, 3x3 window.
 * Returns -1 on unsupported arguments, else 0.  multiplies/tiles mirror
 * WinogradStats. */
TKO_API int tko_conv2d_winograd(const tko_conv_shape* s, size_t m,
                                const float* in, const float* filt, float* out,
                                uint64_t* multiplies, size_t* tiles_out) {
  float bt[36], g[18], at[24];
  if (s->stride != 1 || s->window_rows != 3 || s->window_cols != 3) return -1;
  if (!tko_winograd_plan(m, 3, bt, g, at)) return -1;
  const size_t t = m + 2, spots = t * t;
  const size_t oh_n = tko_out_rows(s), ow_n = tko_out_cols(s);
  const size_t tiles_r = (oh_n + m - 1) / m, tiles_c = (ow_n + m - 1) / m;
  const size_t num_tiles = tiles_r * tiles_c * s->batch;
  const size_t C = s->channels, K = s->features;
  const ptrdiff_t pr = tko_pad_top(s), pc = tko_pad_left(s);

  float* v = (float*)malloc(sizeof(float) * spots * num_tiles * C);
  float* u = (float*)malloc(sizeof(float) * spots * C * K);
  float* prod = (float*)malloc(sizeof(float) * spots * num_tiles * K);
  if (!v || !u || !prod) {
    free(v); free(u); free(prod);
    return -2;
  }

  /* Stage 1: input transform + scatter, v[s][tile + c*num_tiles]. */
#pragma omp parallel for schedule(static)
  for (size_t tile = 0; tile < num_tiles; ++tile) {
    const size_t b = tile / (tiles_r * tiles_c);
    const size_t ti = (tile / tiles_c) % tiles_r;
    const size_t tj = tile % tiles_c;
    const ptrdiff_t r0 = (ptrdiff_t)(ti * m) - pr, c0 = (ptrdiff_t)(tj * m) - pc;
    float patch[36], tr[36];
    for (size_t c = 0; c < C; ++c) {
      for (size_t i = 0; i < t; ++i) {
        const ptrdiff_t ih = r0 + (ptrdiff_t)i;
        for (size_t j = 0; j < t; ++j) {
          const ptrdiff_t iw = c0 + (ptrdiff_t)j;
          const int inside = ih >= 0 && iw >= 0 && ih < (ptrdiff_t)s->in_rows &&
                             iw < (ptrdiff_t)s->in_cols;
          patch[i * t + j] =
              inside ? in[((b * s->in_rows + (size_t)ih) * s->in_cols + (size_t)iw) * C + c]
                     : 0.0f;
        }
      }
      transform_tile(bt, t, t, patch, tr);
      for (size_t sp = 0; sp < spots; ++sp)
        v[sp * num_tiles * C + tile + c * num_tiles] = tr[sp];
    }
  }

  /* Stage 2: filter transform + scatter, u[s][c + k*C]. */
#pragma omp parallel for schedule(static)
  for (size_t k = 0; k < K; ++k) {
    float gg[9], tr[36];
    for (size_t c = 0; c < C; ++c) {
      for (size_t x = 0; x < 3; ++x)
        for (size_t y = 0; y < 3; ++y) gg[x * 3 + y] = filt[((x * 3 + y) * C + c) * K + k];
      transform_tile(g, t, 3, gg, tr);
      for (size_t sp = 0; sp < spots; ++sp) u[sp * C * K + c + k * C] = tr[sp];
    }
  }

  /* Stage 3: batched GEMM over spots. */
  const uint64_t mults = tko_gemm_batched_strided(
      v, num_tiles * C, u, C * K, prod, num_tiles * K, spots, num_tiles, K, C);

  /* Stage 4: gather + output transform, clipped at the plane edge. */
#pragma omp parallel for schedule(static)
  for (size_t tile = 0; tile < num_tiles; ++tile) {
    const size_t b = tile / (tiles_r * tiles_c);
    const size_t ti = (tile / tiles_c) % tiles_r;
    const size_t tj = tile % tiles_c;
    float gathered[36], to[16];
    const size_t rh = oh_n - ti * m < m ? oh_n - ti * m : m;
    const size_t cw = ow_n - tj * m < m ? ow_n - tj * m : m;
    for (size_t k = 0; k < K; ++k) {
      for (size_t sp = 0; sp < spots; ++sp)
        gathered[sp] = prod[sp * num_tiles * K + tile + k * num_tiles];
      transform_tile(at, m, t, gathered, to);
      for (size_t i = 0; i < rh; ++i)
        for (size_t j = 0; j < cw; ++j)
          out[((b * oh_n + ti * m + i) * ow_n + tj * m + j) * K + k] = to[i * m + j];
    }
  }

  if (multiplies) *multiplies = mults;
  if (tiles_out) *tiles_out = num_tiles;
  free(v);
  free(u);
  free(prod);
  return 0;
}

/* ------------------------------------------------------------------------ */
/* Parity metrics (numeric.hpp:14-56)                                       */
/* ------------------------------------------------------------------------ */

TKO_API double tko_max_rel_error(const float* values, const float* ref,
                                 size_t count, double floor_) {
  double worst = 0.0;
  for (size_t i = 0; i < count; ++i) {
    double d = fabs((double)ref[i]);
    if (d < floor_) d = floor_;
    double e = fabs((double)values[i] - (double)ref[i]) / d;
    if (e > worst) worst = e;
  }
  return worst;
}

TKO_API double tko_max_scaled_error(const float* values, const float* ref,
                                    size_t count, double floor_) {
  double scale = floor_;
  for (size_t i = 0; i < count; ++i) {
    double a = fabs((double)ref[i]);
    if (a > scale) scale = a;
  }
  double worst = 0.0;
  for (size_t i = 0; i < count; ++i) {
    double e = fabs((double)values[i] - (double)ref[i]) / scale;
    if (e > worst) worst = e;
  }
  return worst;
}

// exact_gemm.cuh -- bit-exact FP32 SIMT tiled GEMM / implicit-GEMM conv.
//
// One kernel family implements every exact path of the reference:
//   gemm_naive / gemm_tiled        (gemm.hpp:194-213, 308-445)
//   gemm_batched_strided           (gemm.hpp:451-479; gridDim.z = batch)
//   conv2d_naive / _tiled / _im2col (conv.hpp:74-113, 136-248, 320-362) as an
//       implicit GEMM whose K index runs over window taps (x, y, c) in the
//       reference order (x*S + y)*C + c, gathered straight from NHWC input.
//
// Parity contract: every output element is one
// running sum started at +0 and updated acc = fadd_rn(acc, fmul_rn(a, b)) in
// ascending k; out = alpha*acc (beta == 0, C never read) or
// alpha*acc + beta*C.  Zero-filled tails and halos add +0 and leave the bits
// unchanged, so the result equals the reference bit for bit whatever the
// tiling.  No FFMA, no split-K.
//
// Parameterisation follows GemmConfig: each thread owns an H x W register
// tile (reg_rows x reg_cols), a CTA is wg_rows x wg_cols threads, "loc"
// stages K-slabs of BK = 32 elements (one 128-byte line, the paper's X)
// through shared memory with cp.async, "db" deepens that to a multi-stage
// ring, "noloc" reads operands straight from global memory.
#pragma once

#include "common.cuh"

namespace tkb {

constexpr int kExactBK = 32;

enum OperandMajor : int { kMN = 0, kK = 1 };

// Element (m, k) of A lives at a[m*a_sm + k*a_sk]; (k, n) of B at
// b[k*b_sk + n*b_sn]; (m, n) of C/D at d[m*d_sm + n*d_sn].  In conv mode A is
// the implicit patch matrix of an NHWC input.
struct ExactArgs {
  int M, N, K;
  const float* a;
  long long a_sm, a_sk, a_batch;
  const float* b;
  long long b_sk, b_sn, b_batch;
  const float* c;
  float* d;
  long long d_sm, d_sn, d_batch;
  float alpha, beta;
  int read_c;   // beta != 0
  int tx_on_m;  // lane-fast thread index runs along M (column-major output)
  // conv geometry (CONV instantiations only)
  int H, W, C, OH, OW, R, S, stride, pad_t, pad_l;
  // conv2d_tiled's 2-D pixel patches (0 = linear pixel rows): each thread's
  // register rows are a t2_rows x t2_cols patch, the CTA's wg_r threads a
  // t2_pr x t2_pc grid of patches of one image; t2_blk_r x t2_blk_c CTAs
  // per image (blockIdx.x = image * blocks + block).
  int t2_rows, t2_cols, t2_pr, t2_pc, t2_blk_r, t2_blk_c;
};

// Ownership of register-tile rows: MN-major operands hand each thread runs of
// 4 consecutive indices (16-byte shared loads, conflict-free), K-major
// operands interleave single indices (row stride 36 words spreads banks).
template <int T, int LAYOUT>
__device__ __forceinline__ int own_index(int t, int threads, int u) {
  if constexpr (LAYOUT == kMN) {
    if constexpr (T >= 4) {
      return (u >> 2) * (threads * 4) + t * 4 + (u & 3);
    } else {
      return t * T + u;
    }
  } else {
    return u * threads + t;
  }
}

// Shared-memory geometry of one operand slab (BK deep, E wide).
template <int LAYOUT>
struct SlabGeom {
  // MN-major: [BK][E+4]; K-major: [E][BK+4]
  static __device__ __forceinline__ int off(int e, int k, int E) {
    if constexpr (LAYOUT == kMN) return k * (E + 4) + e;
    else return e * (kExactBK + 4) + k;
  }
  static __host__ __device__ __forceinline__ int words(int E) {
    return LAYOUT == kMN ? kExactBK * (E + 4) : E * (kExactBK + 4);
  }
};

// ---------------------------------------------------------------------------
// Global -> shared staging of one K-slab.
// ---------------------------------------------------------------------------

// Plain strided operand (GEMM and batched GEMM).  `e` indexes the M (or N)
// extent, k the depth.  stride_e / stride_k are element strides.
template <int LAYOUT>
__device__ __forceinline__ void stage_matrix(float* sm, const float* g, long long stride_e,
                                             long long stride_k, int e0, int E, int e_lim, int k0,
                                             int k_lim, int tid, int nthreads) {
  // Vector chunks of 4 along the contiguous direction of the operand (rows
  // of an MN-major slab are padded by 4 words, so a ragged last chunk lands
  // in the padding).
  const int chunks = LAYOUT == kMN ? ((E + 3) >> 2) * kExactBK : E * (kExactBK >> 2);
  for (int ch = tid; ch < chunks; ch += nthreads) {
    int e, k;
    if constexpr (LAYOUT == kMN) {
      const int per_row = (E + 3) >> 2;
      k = ch / per_row;
      e = (ch - k * per_row) << 2;
    } else {
      k = (ch & 7) << 2;  // BK/4 = 8 chunks per row
      e = ch >> 3;
    }
    const int ge = e0 + e, gk = k0 + k;
    float* dst = sm + SlabGeom<LAYOUT>::off(e, k, E);
    if constexpr (LAYOUT == kMN) {
      const float* src = g + (long long)ge * stride_e + (long long)gk * stride_k;
      const bool full = gk < k_lim && ge + 3 < e_lim && stride_e == 1 &&
                        ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
      if (full) {
        cp_async16(dst, src, true);
      } else {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const bool ok = gk < k_lim && ge + v < e_lim;
          cp_async4(dst + v, ok ? src + (long long)v * stride_e : g, ok);
        }
      }
    } else {
      const float* src = g + (long long)ge * stride_e + (long long)gk * stride_k;
      const bool full = ge < e_lim && gk + 3 < k_lim && stride_k == 1 &&
                        ((reinterpret_cast<uintptr_t>(src) & 15) == 0);
      if (full) {
        cp_async16(dst, src, true);
      } else {
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const bool ok = ge < e_lim && gk + v < k_lim;
          cp_async4(dst + v, ok ? src + (long long)v * stride_k : g, ok);
        }
      }
    }
  }
}

// Implicit patch matrix of an NHWC input: row m = (n*OH + oh)*OW + ow,
// column k = (x*S + y)*C + c.  Taps outside the input stage as zero.
__device__ __forceinline__ void stage_patches(float* sm, const ExactArgs& p, int m0, int BM,
                                              int k0, int tid, int nthreads) {
  const int chunks = BM * (kExactBK >> 2);
  const bool vec_ok = (p.C & 3) == 0;
  for (int ch = tid; ch < chunks; ch += nthreads) {
    const int kq = (ch & 7) << 2;
    const int e = ch >> 3;
    const int m = m0 + e;
    const int k = k0 + kq;
    float* dst = sm + SlabGeom<kK>::off(e, kq, BM);
    int n = 0, oh = 0, ow = 0;
    const bool row_ok = m < p.M;
    if (row_ok) {
      ow = m % p.OW;
      const int t = m / p.OW;
      oh = t % p.OH;
      n = t / p.OH;
    }
    if (vec_ok && k + 3 < p.K) {
      // Four consecutive channels of one tap.
      const int c = k % p.C;
      const int tap = k / p.C;
      const int y = tap % p.S, x = tap / p.S;
      const int ih = oh * p.stride + x - p.pad_t;
      const int iw = ow * p.stride + y - p.pad_l;
      const bool ok = row_ok && ih >= 0 && iw >= 0 && ih < p.H && iw < p.W;
      const float* src = ok ? p.a + (((long long)n * p.H + ih) * p.W + iw) * p.C + c : p.a;
      if ((reinterpret_cast<uintptr_t>(src) & 15) == 0) {
        cp_async16(dst, src, ok);
      } else {
#pragma unroll
        for (int v = 0; v < 4; ++v) cp_async4(dst + v, ok ? src + v : p.a, ok);
      }
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int kk = k + v;
        bool ok = row_ok && kk < p.K;
        const float* src = p.a;
        if (ok) {
          const int c = kk % p.C;
          const int tap = kk / p.C;
          const int y = tap % p.S, x = tap / p.S;
          const int ih = oh * p.stride + x - p.pad_t;
          const int iw = ow * p.stride + y - p.pad_l;
          ok = ih >= 0 && iw >= 0 && ih < p.H && iw < p.W;
          if (ok) src = p.a + (((long long)n * p.H + ih) * p.W + iw) * p.C + c;
        }
        cp_async4(dst + v, src, ok);
      }
    }
  }
}

// Per-CTA pixel table for the implicit patch matrix: row e of the CTA tile
// -> {element offset of (n, ih0, iw0, 0) in the NHWC input, ih0, iw0}, with
// ih0 = oh*stride - pad_t, iw0 = ow*stride - pad_l (rows past M get an ih0
// that fails every bounds test).  Built once per CTA so the slab loop does
// no divisions.
struct PixRow {
  long long base;
  int ih0, iw0;
};

// wg_r: threads along M (row e = u * wg_r + t of the K-major register
// ownership is element u of thread t's patch in 2-D mode).
// out[e]: element offset of row e's output pixel (pixel * d_sm), -1 if none
// (a separate table: the staging loop reads only the 16-byte PixRow).
__device__ __forceinline__ void build_pix_rows(PixRow* rows, long long* out, const ExactArgs& p,
                                               int m0, int BM, int wg_r, int tid, int nthreads) {
  int n2 = 0, oh2 = 0, ow2 = 0;
  if (p.t2_rows > 0) {
    const int per_img = p.t2_blk_r * p.t2_blk_c;
    n2 = blockIdx.x / per_img;
    const int rem = blockIdx.x - n2 * per_img;
    oh2 = (rem / p.t2_blk_c) * p.t2_rows * p.t2_pr;
    ow2 = (rem % p.t2_blk_c) * p.t2_cols * p.t2_pc;
  }
  for (int e = tid; e < BM; e += nthreads) {
    PixRow r{0, -(1 << 28), 0};
    long long o = -1;
    int n, oh, ow;
    bool ok;
    if (p.t2_rows > 0) {
      const int u = e / wg_r, t = e - (e / wg_r) * wg_r;
      n = n2;
      oh = oh2 + (t / p.t2_pc) * p.t2_rows + u / p.t2_cols;
      ow = ow2 + (t % p.t2_pc) * p.t2_cols + u % p.t2_cols;
      ok = oh < p.OH && ow < p.OW;
    } else {
      const int m = m0 + e;
      ok = m < p.M;
      ow = m % p.OW;
      const int t = m / p.OW;
      oh = t % p.OH;
      n = t / p.OH;
    }
    if (ok) {
      r.ih0 = oh * p.stride - p.pad_t;
      r.iw0 = ow * p.stride - p.pad_l;
      r.base = (((long long)n * p.H + r.ih0) * p.W + r.iw0) * p.C;
      o = (((long long)n * p.OH + oh) * p.OW + ow) * p.d_sm;
    }
    rows[e] = r;
    out[e] = o;
  }
}

// Stage a K-slab of the implicit patch matrix using the pixel table.  A
// thread's chunks always cover the same 4 consecutive k of the slab (the
// chunk index advances by nthreads, a multiple of 8), so the tap
// decomposition is done once per slab and thread.
__device__ __forceinline__ void stage_patches_fast(float* sm, const ExactArgs& p, const PixRow* rows,
                                                   int BM, int k0, int tid, int nthreads) {
  const int kq = (tid & 7) << 2;
  const int k = k0 + kq;
  int kx[4], ky[4], kc[4];
  bool kv[4];
  if (p.C % kExactBK == 0) {
    // The whole 32-deep slab is one tap's channel run: one division pair
    // per slab instead of four per thread (integer division was ~4% of the
    // exact conv's instructions).
    const int tap = k0 / p.C, x = tap / p.S;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      kv[v] = k + v < p.K;
      kc[v] = k0 - tap * p.C + kq + v;
      ky[v] = tap - x * p.S;
      kx[v] = x;
    }
  } else {
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int kk = k + v;
      kv[v] = kk < p.K;
      const int c = kk % p.C, tap = kk / p.C;
      kc[v] = c;
      ky[v] = tap % p.S;
      kx[v] = tap / p.S;
    }
  }
  const bool vec = (p.C & 3) == 0 && kv[3] &&  // four channels of one tap, 16B aligned
                   (reinterpret_cast<uintptr_t>(p.a) & 15) == 0;
  const long long koff = ((long long)kx[0] * p.W + ky[0]) * p.C + kc[0];
  for (int e = tid >> 3; e < BM; e += nthreads >> 3) {
    const PixRow r = rows[e];
    float* dst = sm + SlabGeom<kK>::off(e, kq, BM);
    if (vec) {
      const int ih = r.ih0 + kx[0], iw = r.iw0 + ky[0];
      const bool ok = (unsigned)ih < (unsigned)p.H && (unsigned)iw < (unsigned)p.W;
      cp_async16(dst, ok ? p.a + r.base + koff : p.a, ok);
    } else {
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int ih = r.ih0 + kx[v], iw = r.iw0 + ky[v];
        const bool ok = kv[v] && (unsigned)ih < (unsigned)p.H && (unsigned)iw < (unsigned)p.W;
        cp_async4(dst + v,
                  ok ? p.a + r.base + ((long long)kx[v] * p.W + ky[v]) * p.C + kc[v] : p.a, ok);
      }
    }
  }
}

// Load the register fragment of one depth step from a staged slab.
template <int T, int LAYOUT>
__device__ __forceinline__ void load_frag(float (&f)[T], const float* sm, int t, int threads,
                                          int E, int k) {
  if constexpr (LAYOUT == kMN && T >= 4) {
#pragma unroll
    for (int q = 0; q < T / 4; ++q) {
      const float4 v = *reinterpret_cast<const float4*>(
          sm + SlabGeom<kMN>::off(own_index<T, kMN>(t, threads, q * 4), k, E));
      f[q * 4 + 0] = v.x;
      f[q * 4 + 1] = v.y;
      f[q * 4 + 2] = v.z;
      f[q * 4 + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int u = 0; u < T; ++u) f[u] = sm[SlabGeom<LAYOUT>::off(own_index<T, LAYOUT>(t, threads, u), k, E)];
  }
}

// Fragments of four consecutive depth steps k0..k0+3 (k0 % 4 == 0): one
// 16-byte shared load per row for K-major slabs (the four k are contiguous),
// one per 4 rows and step for MN-major slabs.  f[kk][u].
template <int T, int LAYOUT>
__device__ __forceinline__ void load_frag4(float (&f)[4][T], const float* sm, int t, int threads,
                                           int E, int k0);
template <int T, int LAYOUT>
__device__ __forceinline__ void load_frag4(float (&f)[4][T], const float* sm, int t, int threads,
                                           int E, int k0) {
  if constexpr (LAYOUT == kK) {
#pragma unroll
    for (int u = 0; u < T; ++u) {
      const float4 v = *reinterpret_cast<const float4*>(
          sm + SlabGeom<kK>::off(own_index<T, kK>(t, threads, u), k0, E));
      f[0][u] = v.x;
      f[1][u] = v.y;
      f[2][u] = v.z;
      f[3][u] = v.w;
    }
  } else {
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      float g[T];
      load_frag<T, kMN>(g, sm, t, threads, E, k0 + kk);
#pragma unroll
      for (int u = 0; u < T; ++u) f[kk][u] = g[u];
    }
  }
}

// ---------------------------------------------------------------------------
// The kernel.  H x W register tile, blockDim.x = r*c threads.
// ---------------------------------------------------------------------------
template <int H, int W, int AL, int BL, bool CONV>
__global__ void exact_gemm_loc_kernel(ExactArgs p, int wg_r, int wg_c, int stages) {
  extern __shared__ __align__(16) float smem[];
  const int tid = threadIdx.x;
  const int nthreads = wg_r * wg_c;
  const int BM = H * wg_r, BN = W * wg_c;
  const int tm = p.tx_on_m ? tid % wg_r : tid / wg_c;
  const int tn = p.tx_on_m ? tid / wg_r : tid % wg_c;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int z = blockIdx.z;

  const float* ga = p.a + (CONV ? 0 : (long long)z * p.a_batch);
  const float* gb = p.b + (long long)z * p.b_batch;

  const int a_words = SlabGeom<AL>::words(BM), b_words = SlabGeom<BL>::words(BN);
  const int stage_words = a_words + b_words;
  PixRow* pix_rows = reinterpret_cast<PixRow*>(smem + stages * stage_words);
  long long* pix_out = reinterpret_cast<long long*>(pix_rows + BM);
  if constexpr (CONV) {
    build_pix_rows(pix_rows, pix_out, p, m0, BM, wg_r, tid, nthreads);
    __syncthreads();
  }

  float acc[H][W];
#pragma unroll
  for (int i = 0; i < H; ++i)
#pragma unroll
    for (int j = 0; j < W; ++j) acc[i][j] = 0.0f;

  const int nslabs = (p.K + kExactBK - 1) / kExactBK;

  auto issue = [&](int s) {
    float* sa = smem + (s % stages) * stage_words;
    float* sb = sa + a_words;
    const int k0 = s * kExactBK;
    if constexpr (CONV) {
      if ((nthreads & 7) == 0) stage_patches_fast(sa, p, pix_rows, BM, k0, tid, nthreads);
      else stage_patches(sa, p, m0, BM, k0, tid, nthreads);
    } else {
      stage_matrix<AL>(sa, ga, p.a_sm, p.a_sk, m0, BM, p.M, k0, p.K, tid, nthreads);
    }
    stage_matrix<BL>(sb, gb, p.b_sn, p.b_sk, n0, BN, p.N, k0, p.K, tid, nthreads);
  };

  // Prologue: stages-1 slabs in flight.
  for (int s = 0; s < stages - 1; ++s) {
    if (s < nslabs) issue(s);
    cp_async_commit();
  }
  for (int s = 0; s < nslabs; ++s) {
    if (stages == 1) {
      issue(s);
      cp_async_commit();
      cp_async_wait<0>();
    } else {
      const int nxt = s + stages - 1;
      if (nxt < nslabs) issue(nxt);
      cp_async_commit();
      cp_async_wait_dyn(stages - 1);
    }
    __syncthreads();
    const float* sa = smem + (s % stages) * stage_words;
    const float* sb = sa + a_words;
    // Slab entries past K are staged as zeros on both operands; their +0
    // products leave every running sum's bits unchanged (a sum started at
    // +0 is never -0), so the last slab runs in whole groups of four too.
    const int depth4 = (min(kExactBK, p.K - s * kExactBK) + 3) & ~3;
#pragma unroll 1
    for (int k0 = 0; k0 < depth4; k0 += 4) {
      // K-major operands: one 16-byte load per row covers all four steps;
      // MN-major operands are loaded per step (bounds register pressure).
      float a4[AL == kK ? 4 : 1][H], b4[BL == kK ? 4 : 1][W];
      if constexpr (AL == kK) load_frag4<H, kK>(a4, sa, tm, wg_r, BM, k0);
      if constexpr (BL == kK) load_frag4<W, kK>(b4, sb, tn, wg_c, BN, k0);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        float fa[H], fb[W];
        if constexpr (AL == kK) {
#pragma unroll
          for (int i = 0; i < H; ++i) fa[i] = a4[kk][i];
        } else {
          load_frag<H, kMN>(fa, sa, tm, wg_r, BM, k0 + kk);
        }
        if constexpr (BL == kK) {
#pragma unroll
          for (int j = 0; j < W; ++j) fb[j] = b4[kk][j];
        } else {
          load_frag<W, kMN>(fb, sb, tn, wg_c, BN, k0 + kk);
        }
#pragma unroll
        for (int i = 0; i < H; ++i)
#pragma unroll
          for (int j = 0; j < W; ++j) acc[i][j] = mac_exact(acc[i][j], fa[i], fb[j]);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  // Epilogue: alpha*acc (+ beta*C), clipped to the extent.
  float* gd = p.d + (long long)z * p.d_batch;
  const float* gc = p.c ? p.c + (long long)z * p.d_batch : nullptr;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    long long row_off;
    if constexpr (CONV) {
      row_off = pix_out[own_index<H, AL>(tm, wg_r, i)];  // linear or 2-D patch row
      if (row_off < 0) continue;
    } else {
      const int m = m0 + own_index<H, AL>(tm, wg_r, i);
      if (m >= p.M) continue;
      row_off = (long long)m * p.d_sm;
    }
#pragma unroll
    for (int j = 0; j < W; ++j) {
      const int n = n0 + own_index<W, BL>(tn, wg_c, j);
      if (n >= p.N) continue;
      const long long off = row_off + (long long)n * p.d_sn;
      TKB_DCHECK(off >= 0 && (!CONV || off < (long long)p.M * p.N));
      float v = __fmul_rn(p.alpha, acc[i][j]);
      if (p.read_c) v = __fadd_rn(v, __fmul_rn(p.beta, gc[off]));
      gd[off] = v;
    }
  }
}

// "noloc": same slab walk and accumulation order, operands read straight
// from global memory (the reference's direct path, gemm.hpp:408-430).
template <int H, int W, bool CONV>
__global__ void exact_gemm_noloc_kernel(ExactArgs p, int wg_r, int wg_c) {
  const int tid = threadIdx.x;
  const int BM = H * wg_r, BN = W * wg_c;
  const int tm = p.tx_on_m ? tid % wg_r : tid / wg_c;
  const int tn = p.tx_on_m ? tid / wg_r : tid % wg_c;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int z = blockIdx.z;
  const float* ga = p.a + (CONV ? 0 : (long long)z * p.a_batch);
  const float* gb = p.b + (long long)z * p.b_batch;

  int rows[H], cols[W];
#pragma unroll
  for (int i = 0; i < H; ++i) rows[i] = m0 + i * wg_r + tm;
#pragma unroll
  for (int j = 0; j < W; ++j) cols[j] = n0 + j * wg_c + tn;

  // Conv row decomposition, once.
  int pn[H], pih[H], piw[H];
  if constexpr (CONV) {
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const int m = min(rows[i], p.M - 1);
      const int ow = m % p.OW, t = m / p.OW;
      pn[i] = t / p.OH;
      pih[i] = (t % p.OH) * p.stride - p.pad_t;
      piw[i] = ow * p.stride - p.pad_l;
    }
  }

  float acc[H][W];
#pragma unroll
  for (int i = 0; i < H; ++i)
#pragma unroll
    for (int j = 0; j < W; ++j) acc[i][j] = 0.0f;

  int c = 0, y = 0, x = 0;  // conv tap walk
  for (int k = 0; k < p.K; ++k) {
    float fa[H], fb[W];
#pragma unroll
    for (int i = 0; i < H; ++i) {
      float v = 0.0f;
      if (rows[i] < p.M) {
        if constexpr (CONV) {
          const int ih = pih[i] + x, iw = piw[i] + y;
          if (ih >= 0 && iw >= 0 && ih < p.H && iw < p.W)
            v = __ldg(p.a + (((long long)pn[i] * p.H + ih) * p.W + iw) * p.C + c);
        } else {
          v = __ldg(ga + (long long)rows[i] * p.a_sm + (long long)k * p.a_sk);
        }
      }
      fa[i] = v;
    }
#pragma unroll
    for (int j = 0; j < W; ++j)
      fb[j] = cols[j] < p.N ? __ldg(gb + (long long)k * p.b_sk + (long long)cols[j] * p.b_sn) : 0.0f;
#pragma unroll
    for (int i = 0; i < H; ++i)
#pragma unroll
      for (int j = 0; j < W; ++j) acc[i][j] = mac_exact(acc[i][j], fa[i], fb[j]);
    if constexpr (CONV) {
      if (++c == p.C) {
        c = 0;
        if (++y == p.S) {
          y = 0;
          ++x;
        }
      }
    }
  }

  float* gd = p.d + (long long)z * p.d_batch;
  const float* gc = p.c ? p.c + (long long)z * p.d_batch : nullptr;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    if (rows[i] >= p.M) continue;
#pragma unroll
    for (int j = 0; j < W; ++j) {
      if (cols[j] >= p.N) continue;
      const long long off = (long long)rows[i] * p.d_sm + (long long)cols[j] * p.d_sn;
      float v = __fmul_rn(p.alpha, acc[i][j]);
      if (p.read_c) v = __fadd_rn(v, __fmul_rn(p.beta, gc[off]));
      gd[off] = v;
    }
  }
}

// Host launcher (exact_gemm.cu).  h/w in {1,2,4,8}; r*c <= 1024.
struct ExactLaunch {
  int h, w, r, c;
  bool loc;
  int stages;  // 1 (loc), 2..3 (loc_db)
  // Runtime register tile (exact_gen.cuh): any h, w; conv2d_tiled's patch
  // geometry when tile_rows > 0; cvec = channel_vector of the staging.
  bool gen = false;
  int tile_rows = 0, tile_cols = 0, cvec = 4;
  bool shrink_ok = false;  // library-shaped (conv2d_tiled): r may shrink to fit
};
void launch_exact(const ExactArgs& p, const ExactLaunch& L, bool conv, int batch,
                  cudaStream_t stream);

}  // namespace tkb

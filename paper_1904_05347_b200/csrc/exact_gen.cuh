// exact_gen.cuh -- runtime register tile for the exact FP32 family.
//
// The reference's microkernel_generic (gemm.hpp:247-292) accepts ANY h x w
// register tile; the tuned kernels of exact_gemm.cuh instantiate h, w in
// {1, 2, 4, 8} only.  This kernel takes h and w at run time inside a
// compile-time bound (HM x WM accumulators, HM * WM <= 64; the host picks
// the smallest bound that holds the tile, and splits tiles of more than 64
// outputs over several GPU threads -- the CTA tile h*r x w*c is kept).  The
// arithmetic is the family's: one ascending-k running sum per output,
// acc = fadd_rn(acc, fmul_rn(a, b)), so the bits equal the reference's for
// every h, w.
//
// It also carries conv2d_tiled's own geometry (conv.hpp:136-248): with
// tile_rows x tile_cols set, a thread's h = tile_rows * tile_cols rows are a
// 2-D patch of output pixels (the reference's per-thread tile), the CTA's
// r threads along M tile a pr x pc grid of such patches of one image, w =
// feature_vector features per thread, and the input is staged channel_vector
// channels per copy.
#pragma once

#include "exact_gemm.cuh"

namespace tkb {

// Extra geometry of the generic kernel (kept out of ExactArgs so the tuned
// kernels' parameter block is unchanged).
struct GenGeom {
  int h, w;                // runtime register tile
  int tile_rows, tile_cols;  // conv2d_tiled patch per thread (0: linear rows)
  int pr, pc;              // patch grid of the CTA (pr * pc = wg_r)
  int blk_r, blk_c;        // CTA blocks per image (rows, cols)
  int cvec;                // channel_vector: elements per staging copy (1, 2, 4)
};

// Row e of the CTA tile -> input pixel + output offset.
struct GenRow {
  long long base;  // element offset of (n, ih0, iw0, 0) in the NHWC input
  long long out;   // element offset of the output pixel, -1 if outside
  int ih0, iw0;
};

__device__ __forceinline__ void gen_rows_conv(GenRow* rows, const ExactArgs& p, const GenGeom& q,
                                              int blk, int BM, int wg_r, int tid, int nthreads) {
  const int per_img = q.blk_r * q.blk_c;
  const int n = blk / per_img;
  const int rem = blk - n * per_img;
  const int br = rem / q.blk_c, bc = rem - (rem / q.blk_c) * q.blk_c;
  const int BR = q.tile_rows * q.pr, BC = q.tile_cols * q.pc;
  for (int e = tid; e < BM; e += nthreads) {
    int oh, ow;
    if (q.tile_rows > 0) {
      const int u = e / wg_r, tm = e - (e / wg_r) * wg_r;  // element u of thread tm's patch
      oh = br * BR + (tm / q.pc) * q.tile_rows + u / q.tile_cols;
      ow = bc * BC + (tm % q.pc) * q.tile_cols + u % q.tile_cols;
    } else {
      const int m = blk * BM + e;
      ow = m % p.OW;
      oh = (m / p.OW) % p.OH;
    }
    GenRow r{0, -1, -(1 << 28), 0};
    const int nn = q.tile_rows > 0 ? n : (blk * BM + e) / (p.OW * p.OH);
    const bool ok = q.tile_rows > 0 ? (oh < p.OH && ow < p.OW) : (blk * BM + e < p.M);
    if (ok) {
      r.ih0 = oh * p.stride - p.pad_t;
      r.iw0 = ow * p.stride - p.pad_l;
      r.base = (((long long)nn * p.H + r.ih0) * p.W + r.iw0) * p.C;
      r.out = (((long long)nn * p.OH + oh) * p.OW + ow) * p.d_sm;
    }
    rows[e] = r;
  }
}

// K-slab of the implicit patch matrix through the row table, cvec
// consecutive channels of one tap per copy (channel_vector).
__device__ __forceinline__ void gen_stage_patches(float* sm, const ExactArgs& p, const GenRow* rows,
                                                  int BM, int k0, int cvec, int tid, int nthreads) {
  const int groups = kExactBK / cvec;  // copies per row of the slab
  if (nthreads % groups == 0) {
    // Every copy of this thread is the same cvec-channel group of the slab:
    // decompose its k into (tap, channel) once.
    const int kq = (tid % groups) * cvec;
    const int k = k0 + kq;
    const int c = k % p.C, tap = k / p.C;
    const int y = tap % p.S, x = tap / p.S;
    const bool whole = c + cvec <= p.C && k + cvec <= p.K &&
                       (reinterpret_cast<uintptr_t>(p.a) & (4 * cvec - 1)) == 0 && (p.C % cvec) == 0;
    const long long koff = ((long long)x * p.W + y) * p.C + c;
    for (int e = tid / groups; e < BM; e += nthreads / groups) {
      const GenRow r = rows[e];
      float* dst = sm + SlabGeom<kK>::off(e, kq, BM);
      if (whole) {
        const int ih = r.ih0 + x, iw = r.iw0 + y;
        const bool in = r.out >= 0 && (unsigned)ih < (unsigned)p.H && (unsigned)iw < (unsigned)p.W;
        const float* src = in ? p.a + r.base + koff : p.a;
        if (cvec == 4) cp_async16(dst, src, in);
        else if (cvec == 2) cp_async8(dst, src, in);
        else cp_async4(dst, src, in);
      } else {
        for (int v = 0; v < cvec; ++v) {
          const int kk = k + v;
          bool ok = r.out >= 0 && kk < p.K;
          const float* s = p.a;
          if (ok) {
            const int cc = kk % p.C, tp = kk / p.C;
            const int yy = tp % p.S, xx = tp / p.S;
            const int ih2 = r.ih0 + xx, iw2 = r.iw0 + yy;
            ok = (unsigned)ih2 < (unsigned)p.H && (unsigned)iw2 < (unsigned)p.W;
            if (ok) s = p.a + r.base + ((long long)xx * p.W + yy) * p.C + cc;
          }
          cp_async4(dst + v, s, ok);
        }
      }
    }
    return;
  }
  for (int ch = tid; ch < BM * groups; ch += nthreads) {
    const int e = ch / groups;
    const int kq = (ch - e * groups) * cvec;
    const GenRow r = rows[e];
    float* dst = sm + SlabGeom<kK>::off(e, kq, BM);
    const int k = k0 + kq;
    const int c = k % p.C, tap = k / p.C;
    const int y = tap % p.S, x = tap / p.S;
    const bool whole = cvec > 1 && c + cvec <= p.C && k + cvec <= p.K;
    const int ih = r.ih0 + x, iw = r.iw0 + y;
    const bool in = r.out >= 0 && (unsigned)ih < (unsigned)p.H && (unsigned)iw < (unsigned)p.W;
    const float* src = p.a + r.base + ((long long)x * p.W + y) * p.C + c;
    if (whole && cvec == 4 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
      cp_async16(dst, in ? src : p.a, in);
    } else if (whole && cvec == 2 && (reinterpret_cast<uintptr_t>(src) & 7) == 0) {
      cp_async8(dst, in ? src : p.a, in);
    } else {
      for (int v = 0; v < cvec; ++v) {
        const int kk = k + v;
        bool ok = r.out >= 0 && kk < p.K;
        const float* s = p.a;
        if (ok) {
          const int cc = kk % p.C, tp = kk / p.C;
          const int yy = tp % p.S, xx = tp / p.S;
          const int ih2 = r.ih0 + xx, iw2 = r.iw0 + yy;
          ok = (unsigned)ih2 < (unsigned)p.H && (unsigned)iw2 < (unsigned)p.W;
          if (ok) s = p.a + r.base + ((long long)xx * p.W + yy) * p.C + cc;
        }
        cp_async4(dst + v, s, ok);
      }
    }
  }
}

// SMALL: work-groups of at most 256 threads, two CTAs per SM (<= 128
// registers: the staging wait of one CTA overlaps the other's MACs).
template <int HM, int WM, int AL, int BL, bool CONV, bool SMALL>
__global__ void __launch_bounds__(SMALL ? 256 : 1024, SMALL ? 2 : 1)
    exact_gemm_gen_kernel(ExactArgs p, GenGeom q, int wg_r, int wg_c, int stages) {
  extern __shared__ __align__(16) float smem[];
  const int tid = threadIdx.x;
  const int nthreads = wg_r * wg_c;
  const int h = q.h, w = q.w;
  const int BM = h * wg_r, BN = w * wg_c;
  const int tm = p.tx_on_m ? tid % wg_r : tid / wg_c;
  const int tn = p.tx_on_m ? tid / wg_r : tid % wg_c;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int z = blockIdx.z;
  const float* ga = p.a + (CONV ? 0 : (long long)z * p.a_batch);
  const float* gb = p.b + (long long)z * p.b_batch;

  const int a_words = SlabGeom<AL>::words(BM), b_words = SlabGeom<BL>::words(BN);
  const int stage_words = a_words + b_words;
  GenRow* rows = reinterpret_cast<GenRow*>(smem + stages * stage_words);
  if constexpr (CONV) {
    gen_rows_conv(rows, p, q, blockIdx.x, BM, wg_r, tid, nthreads);
    __syncthreads();
  }

  float acc[HM][WM];
#pragma unroll
  for (int i = 0; i < HM; ++i)
#pragma unroll
    for (int j = 0; j < WM; ++j) acc[i][j] = 0.0f;

  const int nslabs = (p.K + kExactBK - 1) / kExactBK;
  auto issue = [&](int s) {
    float* sa = smem + (s % stages) * stage_words;
    float* sb = sa + a_words;
    const int k0 = s * kExactBK;
    if constexpr (CONV) gen_stage_patches(sa, p, rows, BM, k0, q.cvec, tid, nthreads);
    else stage_matrix<AL>(sa, ga, p.a_sm, p.a_sk, m0, BM, p.M, k0, p.K, tid, nthreads);
    stage_matrix<BL>(sb, gb, p.b_sn, p.b_sk, n0, BN, p.N, k0, p.K, tid, nthreads);
  };
  for (int s = 0; s < stages - 1; ++s) {
    if (s < nslabs) issue(s);
    cp_async_commit();
  }
  for (int s = 0; s < nslabs; ++s) {
    const int nxt = s + stages - 1;
    if (nxt < nslabs) issue(nxt);
    cp_async_commit();
    cp_async_wait_dyn(stages - 1);
    __syncthreads();
    const float* sa = smem + (s % stages) * stage_words;
    const float* sb = sa + a_words;
    const int depth = min(kExactBK, p.K - s * kExactBK);
    // Runtime h, w inside the HM x WM bound: rows run in groups of 4 and
    // columns in pairs behind warp-uniform branches (h, w are kernel
    // arguments); inside a group every MAC is unconditional, rows / columns
    // past h / w read a clamped (valid) slab entry and their sums are never
    // stored.  Depth advances 4 steps at a time (slab entries past K are
    // zeros on both operands: +0 products leave the sums' bits unchanged);
    // K-major operands load those 4 steps with one 16-byte read per row.
    // Per output the recurrence is the family's ascending-k sum.
    constexpr int RG = HM >= 4 ? 4 : HM, CG = WM >= 2 ? 2 : WM;
    const int depth4 = (depth + 3) & ~3;
#pragma unroll 1
    for (int k0 = 0; k0 < depth4; k0 += 4) {
      // Narrow tiles (WM <= 8) load B's 4 steps once; wide ones (HM <= 4:
      // a single row group) load B per step inside the group.
      constexpr bool kB4 = WM <= 8;
      float fb4[kB4 ? 4 : 1][kB4 ? WM : 1];
      if constexpr (kB4) {
#pragma unroll
        for (int j = 0; j < WM; ++j) {
          const float* bcol = sb + SlabGeom<BL>::off(min(j, w - 1) * wg_c + tn, k0, BN);
          if constexpr (BL == kK) {
            const float4 v = *reinterpret_cast<const float4*>(bcol);
            fb4[0][j] = v.x;
            fb4[1][j] = v.y;
            fb4[2][j] = v.z;
            fb4[3][j] = v.w;
          } else {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) fb4[kk][j] = bcol[kk * (BN + 4)];
          }
        }
      }
#pragma unroll
      for (int i0 = 0; i0 < HM; i0 += RG) {
        if (i0 < h) {
          const float* arow[RG];
#pragma unroll
          for (int i = 0; i < RG; ++i)
            arow[i] = sa + SlabGeom<AL>::off(min(i0 + i, h - 1) * wg_r + tm, k0, BM);
          float fa4[AL == kK ? 4 : 1][RG];
          if constexpr (AL == kK) {
#pragma unroll
            for (int i = 0; i < RG; ++i) {
              const float4 v = *reinterpret_cast<const float4*>(arow[i]);
              fa4[0][i] = v.x;
              fa4[1][i] = v.y;
              fa4[2][i] = v.z;
              fa4[3][i] = v.w;
            }
          }
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            float fa[RG], fb[WM];
#pragma unroll
            for (int i = 0; i < RG; ++i)
              fa[i] = AL == kK ? fa4[AL == kK ? kk : 0][i] : arow[i][kk * (BM + 4)];
#pragma unroll
            for (int j = 0; j < WM; ++j) {
              if constexpr (kB4) {
                fb[j] = fb4[kk][j];
              } else {
                const float* bcol = sb + SlabGeom<BL>::off(min(j, w - 1) * wg_c + tn, k0 + kk, BN);
                fb[j] = *bcol;
              }
            }
#pragma unroll
            for (int j0 = 0; j0 < WM; j0 += CG) {
              if (j0 < w) {
#pragma unroll
                for (int i = 0; i < RG; ++i)
#pragma unroll
                  for (int j = 0; j < CG; ++j)
                    acc[i0 + i][j0 + j] = mac_exact(acc[i0 + i][j0 + j], fa[i], fb[j0 + j]);
              }
            }
          }
        }
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();

  float* gd = p.d + (long long)z * p.d_batch;
  const float* gc = p.c ? p.c + (long long)z * p.d_batch : nullptr;
#pragma unroll
  for (int i = 0; i < HM; ++i) {
    if (i >= h) break;
    const int e = i * wg_r + tm;
    long long row_off;
    if constexpr (CONV) {
      row_off = rows[e].out;
      if (row_off < 0) continue;
    } else {
      const int m = m0 + e;
      if (m >= p.M) continue;
      row_off = (long long)m * p.d_sm;
    }
#pragma unroll
    for (int j = 0; j < WM; ++j) {
      if (j >= w) break;
      const int n = n0 + j * wg_c + tn;
      if (n >= p.N) continue;
      const long long off = row_off + (long long)n * p.d_sn;
      TKB_DCHECK(off >= 0 && (!CONV || off < (long long)p.M * p.N));
      float v = __fmul_rn(p.alpha, acc[i][j]);
      if (p.read_c) v = __fadd_rn(v, __fmul_rn(p.beta, gc[off]));
      gd[off] = v;
    }
  }
}

// Host launcher (exact_gemm.cu): any h, w >= 1 (tiles over 64 outputs are
// split over several GPU threads, CTA tile kept); conv2d_tiled geometry when
// tile_rows > 0.
struct GenLaunch {
  int h, w, r, c, stages;
  int tile_rows = 0, tile_cols = 0, cvec = 4;
  // Library-shaped launch (conv2d_tiled): r may shrink to fit the register
  // file; a caller's GemmConfig that does not fit is a ConfigError instead.
  bool shrink_ok = false;
};
void launch_exact_gen(const ExactArgs& p, const GenLaunch& L, bool conv, int batch,
                      cudaStream_t stream);

}  // namespace tkb

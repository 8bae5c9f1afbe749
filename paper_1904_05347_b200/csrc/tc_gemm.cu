// tc_gemm.cu -- tcgen05 tensor-core GEMM and implicit-GEMM convolution.
//
// One persistent, warp-specialised kernel family (192 threads per CTA, one
// CTA per SM), templated on
//   MODE  operand sources (plain GEMM / conv with pixels on N / on M)
//   CG    CTA group: 1 = one SM, UMMA M = 128; 2 = an SM pair (cluster of 2)
//         issuing tcgen05.mma.cta_group::2 with UMMA M = 256 -- each SM
//         stages half of A (128 rows) and half of B (BN/2 rows), which halves
//         the per-SM shared-memory operand traffic per MAC
//   TF32  kind::tf32 on fp32 operands (32 elements per 128-byte K-slab) or
//         kind::f16 on bf16 operands (64 elements per slab)
// Roles:
//   warp 0      TMA producer (both CTAs): STAGES-deep ring of 128-byte-
//               swizzled K-slabs; completion is signalled on the leader CTA's
//               `full` barrier (cp.async.bulk.tensor.cta_group::2)
//   warp 1      MMA issuer (leader CTA only): 4 x tcgen05.mma per slab into a
//               TMEM accumulator; tcgen05.commit (multicast to the pair)
//               frees the slab in both CTAs / publishes the accumulator
//   warps 2..5  epilogue (both CTAs): tcgen05.ld 32x32b -> registers ->
//               global; two TMEM accumulators (2 x 256 columns) let the MMA
//               run the next tile while the epilogue drains this one
// Operand sources:
//   plain GEMM : A [M][K], B [N][K] via 3-D TMA (K, rows, batch)
//   conv       : the filter repacked to [Kout][R*S*C] via 2-D TMA; the
//                activations via a 4-D TMA box {slab, Wb, Hb, 1} of the NHWC
//                input per (tap, channel chunk) shifted by the tap offset.
//                Rows/cols of the box outside the input are zero-filled by
//                the TMA unit, which is exactly Same padding.
// K order of the conv slabs is (x, y, c), the reference's im2col column order
// (conv.hpp:286-292).
#include <cuda.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>
#include <cstdio>

#include "common.cuh"
#include "experiments.cuh"
#include "launch_cache.cuh"
#include "tc_gemm.cuh"
#include "tc_ptx.cuh"

namespace tkb {

TcKnobs& tc_knobs() {
  thread_local TcKnobs k;
  return k;
}

namespace {

constexpr int kRows = 128;       // A rows staged per CTA (UMMA M per SM)
constexpr int kSlabBytes = 128;  // bytes of K per operand row per stage
constexpr int kThreads = 192;
constexpr int kAccCols = 256;  // TMEM: 2 x 256 fp32 columns allocated
constexpr int kMaxAcc = 8;     // accumulator slots when BN <= 64 (512 / 64)
constexpr int kMaxStages = 8;
constexpr int kMaxSplits = 16;
constexpr int kHaloPitch = 16;  // halo modes: virtual pitch of the pixel rows (TMEM lanes)  // split-K partials summed by splitk_reduce
constexpr int kMaxNarrowMma = 32;  // narrow halo: MMAs per tile (two taps each, 7x7 -> 25)

enum TcMode : int {
  kPlain = 0,
  kConvPixN = 1,
  kConvPixM = 2,
  kConvGather = 3,
  kConvHalo = 4,
  kConvIm2col = 5,  // plain GEMM whose A rows are output pixels loaded by im2col-mode TMA
  kConvHaloNarrow = 6  // halo mode on 16-byte pixels (the C = 3 first layers), see TcArgs::nphase
};
// Halo-family modes (halo box operand + shifted-view taps, halo epilogue).
template <int MODE>
constexpr bool halo_like() {
  return MODE == kConvHalo || MODE == kConvHaloNarrow;
}
// Modes with the plain GEMM's unit decode, split-K partials and tail pieces.
template <int MODE>
constexpr bool plain_like() {
  return MODE == kPlain || MODE == kConvIm2col;
}

#ifndef TKB_GATHER_GROUPS
#define TKB_GATHER_GROUPS 2
#endif
// Gather mode adds kGatherGroups x 4 producer warps (6..) that build the
// pixel operand; groups take alternate K-slabs so their load latencies
// overlap.
constexpr int kGatherGroups = TKB_GATHER_GROUPS;
// Epilogue warpgroups: two (warps 2..5 and 6..9, alternate tiles) except in
// gather mode, whose warps 6.. are producers.  The second group runs only
// when TcArgs::epi_groups == 2 (epilogue-bound tiles).
#ifndef TKB_EPI_GROUPS
#define TKB_EPI_GROUPS 2
#endif
#ifndef TKB_TMEM_PAIRS
#define TKB_TMEM_PAIRS 1
#endif
template <int MODE>
constexpr int epi_groups_of() {
  // (only the narrow halo: a second group on the other modes measured no
  // better for short-K tiles and costs every launch 128 threads)
  return MODE == kConvHaloNarrow ? TKB_EPI_GROUPS : 1;
}
template <int MODE>
constexpr int threads_of() {
  return MODE == kConvGather ? kThreads + 128 * kGatherGroups : kThreads + 128 * (epi_groups_of<MODE>() - 1);
}
// Epilogue group g's named barrier: ptx::epi_sync(g) (ids 1 / 2; gather mode,
// whose producer groups use 2.., has one epilogue group).

// n / d for 0 <= n < 2^31 by multiply-shift (Granlund-Montgomery with a
// 33-bit magic split as m + 2^32): l = ceil(log2 d), m = 2^32 (2^l - d) / d
// + 1, n / d = (umulhi(n, m) + n) >> l.
struct FDiv {
  uint32_t m;
  int l;
};
inline FDiv make_fdiv(int d) {
  if (d < 1) d = 1;
  int l = 0;
  while ((1ll << l) < (long long)d) ++l;
  const unsigned long long m = ((1ull << 32) * ((1ull << l) - (unsigned long long)d)) / (unsigned)d + 1;
  return FDiv{(uint32_t)m, l};
}
__device__ __forceinline__ int fdiv(int n, FDiv f) {
  return (int)((__umulhi((uint32_t)n, f.m) + (uint32_t)n) >> f.l);
}

struct TcArgs {
  int M, N, K;
  int BN;                      // UMMA N (columns of the tile)
  int num_m, num_n, batch, num_kb, stages;
  int ek;                      // K elements per slab (32 tf32 / 64 bf16)
  float* d;
  const float* c;
  long long d_sm, d_sn, d_batch;
  float alpha, beta;
  int read_c;
  int store_tma;               // epilogue via swizzled smem tile + TMA store
  int epi_bytes;               // bytes of epilogue staging
  int epi_bufs;                // staging buffers for the TMA-store epilogue
  int epi_ring;                // > 0: staging slots of epi_ring 32-column chunks (tma_store_epilogue)
  int epi_slots;               // staging slots in the ring (2..8): bulk stores in flight per CTA
  int direct_store;            // epilogue: st.global straight from the TMEM registers (no TMA store)
  int epi_groups;              // epilogue warpgroups in use (1 or 2); staging split between them
  int out_bf16;                // output written as bf16 (TK_IO_OUT_BF16; kernels with OB = true)
  // TMEM accumulator ring: acc_slots slots of acc_cols columns (512 / slots);
  // more slots for narrow tiles let the MMA run further ahead of the
  // epilogue, decoupling their per-tile handshakes.
  int acc_slots, acc_cols, acc_shift;  // acc_slots = 1 << acc_shift
  // conv geometry
  int OH, OW, Kout, Wb, tileH, boxH, tiles_w, tiles_h, pad_t, pad_l, cchunks, S;
  // pixN on small planes: one pixel tile = `imgs` whole images (box
  // {slab, Wb, tileH, imgs / CG} per CTA); Nimg = batch for the edge check.
  int imgs, Nimg;
  // pixN "flat rows": batch x output rows as one row space of N*OH rows;
  // tile t = rows [t*tileH, +tileH), each CTA boxes boxH full-width rows
  // that lie in one image (OH % boxH == 0) -- no row padding per image.
  int flat;
  // halo mode: virtual pitch P, TH rows per CTA, TW useful columns, R*S taps
  int P, TH, TW, taps, halo_bytes;
  int resident;                // halo mode: this CTA's filter slice lives in smem
  // gather mode: input geometry
  const float* in;
  int H, W, C, R, stride, Kreal;
  // split-K (plain mode): unit t covers K-slabs [sp*kb_per, sp*kb_per +
  // kb_per) of its tile, sp = t / (num_m*num_n*batch); partial tiles are
  // stored at batch coordinate sp*batch + z and summed by splitk_reduce.
  int splits, kb_per;
  // With splits > 1 every unit stores its partial tile at part +
  // sp*part_stride (the output's own layout); splitk_reduce then sums the
  // partials in split order (deterministic, no atomics) into the output.
  float* part;
  long long part_stride;
  // L2-aware raster (plain / pixN): tiles are visited in groups of `raster`
  // M-blocks, N-blocks within a group, so a wave of CTAs shares A and B tiles.
  int raster;
  // Plain TF32 GEMM with A MN-major (TcGemm::a_mn): A stages are 4 boxes of
  // 32 M x 32 K (box {32, 32, 4} of the view {32, K, M/32}), 4 KiB apart,
  // 128B_ATOM_32B-swizzled (ptx::desc_sw128_mn).
  int a_mn;
  // Narrow halo (kConvHaloNarrow): window taps R*S of the 16-byte-pixel
  // first layers (C <= 4 tf32 / 8 bf16 channels, input padded once).
  int narrow_taps;
  // Narrow halo (kConvHalo with 16-byte pixels): stride^2 phase boxes of
  // phase_bytes each (stride 2: the even/odd rows x columns of the input,
  // TMA traversal stride 2), taps ordered by (phase, row, column) so each
  // MMA's two taps are increasing addresses (desc_none's LBO = their gap).
  int nphase, phase_bytes;
  int halo_tx;  // bytes the narrow halo's boxes deliver (halo_bytes: that, 1024-aligned)
  // Balanced tail (plain / pixN, splits == 1; stream-K over the last partial
  // wave): the tail_W = (tiles - tail_start) x num_kb slab-steps of the
  // tiles >= tail_start are dealt to the tail_P SM pairs as equal contiguous
  // ranges [p W / P, (p+1) W / P) in (tile, slab) order.  Pair p's range is
  // cut at tile boundaries into at most tail_kb segments, visited as units
  // tail_start + j P + p.  A tile covered by one segment is stored directly;
  // otherwise every segment stores its partial tile column-major (tile-
  // local, [BN][128] per CTA) in slot tile * tail_q + piece of tail_part, and
  // tail_reduce sums the pieces in order into the output (deterministic).
  int tail_start, tail_q, tail_kb, tail_P;
  long long tail_W;
  float* tail_part;
  // Timeline probe (TK_TC_TRACE=1, experiments only): per CTA, globaltimer
  // stamps of kTraceEvents milestones.
  unsigned long long* trace;
  // Multiply-shift divisors of the unit decode (set by run_kernel): a chain
  // of runtime integer divisions per tile sat on the epilogue's critical
  // path of one-slab tiles (narrow halo).
  FDiv fd_per, fd_span, fd_raster, fd_num_m, fd_num_n, fd_batch, fd_per_img, fd_tiles_w;
};

constexpr int kTraceEvents = 21;
constexpr int kTraceUnit = 8;  // steady-state unit probed by events 10..17
__device__ __forceinline__ void trace_mark(const TcArgs& p, int ev) {
  if (p.trace) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
    p.trace[blockIdx.x * kTraceEvents + ev] = t;
  }
}

// Work unit t -> (m_blk, n_blk, z, split) and its K-slab range.
struct Unit {
  int m_blk, n_blk, z, sp, kb0, kb1;
  int slot;  // tail piece slot (-1: a whole tile)
};

// Tile t -> (m_blk, n_blk, z, split) with the split's K-slab range.
__device__ __forceinline__ Unit decode_tile(const TcArgs& p, int t) {
  Unit u;
  u.slot = -1;
  const int per = p.num_m * p.num_n;
  const int rest = fdiv(t, p.fd_per);
  const int t2 = t - rest * per;
  if (p.raster > 1) {
    const int span = p.raster * p.num_n;
    const int group = fdiv(t2, p.fd_span);
    const int first_m = group * p.raster;
    const int gsize = min(p.num_m - first_m, p.raster);
    const int local = t2 - group * span;
    const int nb = gsize == p.raster ? fdiv(local, p.fd_raster) : local / gsize;
    u.m_blk = first_m + local - nb * gsize;
    u.n_blk = nb;
  } else {
    const int nb = fdiv(t2, p.fd_num_m);
    u.m_blk = t2 - nb * p.num_m;
    u.n_blk = nb;
  }
  u.sp = fdiv(rest, p.fd_batch);
  u.z = rest - u.sp * p.batch;
  TKB_DCHECK(u.sp < p.splits && u.m_blk < p.num_m && u.n_blk < p.num_n);
  u.kb0 = u.sp * p.kb_per;
  u.kb1 = min(p.num_kb, u.kb0 + p.kb_per);
  return u;
}

// Balanced tail: the pair whose range holds slab-step s (ranges [b_p,
// b_{p+1}), b_p = floor(p W / P)) is ceil((s + 1) P / W) - 1.
__device__ __forceinline__ int tail_owner(const TcArgs& p, long long s) {
  return (int)(((s + 1) * p.tail_P + p.tail_W - 1) / p.tail_W) - 1;
}

// Unit t -> tile and K-slab range; tail units may be empty (kb0 == kb1).
__device__ __forceinline__ Unit decode_unit(const TcArgs& p, int t) {
  if (p.tail_q > 1 && t >= p.tail_start) {
    const int d = t - p.tail_start;
    const int pr = d % p.tail_P, j = d / p.tail_P;
    const long long nk = p.num_kb;
    const long long b1 = (long long)(pr + 1) * p.tail_W / p.tail_P;
    long long s = (long long)pr * p.tail_W / p.tail_P;
    for (int i = 0; i < j && s < b1; ++i) s = (s / nk + 1) * nk;
    if (s >= b1) {
      Unit e = decode_tile(p, p.tail_start);
      e.kb0 = e.kb1 = 0;
      return e;
    }
    const int r = (int)(s / nk);
    const long long e = min(b1, (long long)(r + 1) * nk);
    Unit u = decode_tile(p, p.tail_start + r);
    u.kb0 = (int)(s - r * nk);
    u.kb1 = (int)(e - r * nk);
    const int p0 = tail_owner(p, r * nk), p1 = tail_owner(p, (r + 1) * nk - 1);
    u.slot = p0 == p1 ? -1 : r * p.tail_q + (pr - p0);
    return u;
  }
  return decode_tile(p, t);
}

__host__ __device__ inline long long total_tiles_of_dev(const TcArgs& p) {
  return (long long)p.num_m * p.num_n * p.batch;
}

// Tail piece epilogue: this thread's accumulator row (TMEM lane `row`) into
// the slot's column-major [BN][128] partial tile (lanes = consecutive rows:
// coalesced 128-byte stores per column).
__device__ __forceinline__ void store_tail_piece(const TcArgs& p, uint32_t taddr, int slot,
                                                 uint32_t rank, int cg, int row) {
  TKB_DCHECK(slot >= 0 && slot < (int)(total_tiles_of_dev(p) - p.tail_start) * p.tail_q);
  float* dst = p.tail_part + ((long long)slot * cg + rank) * ((long long)p.BN * 128);
  for (int col = 0; col < p.BN; col += 32) {
    float v[32];
    ptx::tmem_ld32(taddr + col, v);
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (col + j < p.BN) dst[(long long)(col + j) * 128 + row] = v[j];
  }
}



struct PixTile {
  int img, oh0, ow0;
};

__device__ __forceinline__ PixTile pix_tile(const TcArgs& p, int t) {
  PixTile r;
  const int per_img = p.tiles_w * p.tiles_h;
  const int ti = fdiv(t, p.fd_per_img);
  r.img = ti * (p.imgs > 1 ? p.imgs : 1);
  const int rem = t - ti * per_img;
  const int th = fdiv(rem, p.fd_tiles_w);
  r.oh0 = th * p.tileH;
  r.ow0 = (rem - th * p.tiles_w) * p.Wb;
  return r;
}

// Epilogue through shared memory + TMA store: each of the 128 epilogue
// threads owns one accumulator row (TMEM lane); it writes the row into a
// 128-byte-swizzled [128 rows][32 fp32] staging tile per 32-column chunk
// (conflict-free: 16-byte chunk c of row r lands at c ^ (r % 8)), then one
// thread issues the bulk tensor store(s).  Rows/columns outside the output
// tensor are clipped by the TMA unit.  Two staging buffers alternate, so the
// store of tile i overlaps the TMEM drain of tile i+1.
// BF16 output: one staging chunk = 64 accumulator columns = one 128-byte
// bf16 row per pixel, in the fp32 chunk's swizzled layout (TMA box {64, ...}
// of a bf16 map).  All lanes load (tcgen05.ld is warp-collective).
__device__ __forceinline__ void stage_chunk_bf16(const TcArgs& p, uint32_t taddr, uint8_t* buf,
                                                 int srow) {
  uint32_t r[2][32];
  ptx::tmem_ld32_async(taddr, r[0]);
  ptx::tmem_ld32_async(taddr + 32, r[1]);
  ptx::tmem_wait_ld();
  if (srow < 0) return;
  const uint32_t rowp = ptx::smem(buf + srow * kSlabBytes);
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = 8 * c + 2 * q;
      __nv_bfloat162 b = __floats2bfloat162_rn(p.alpha * __uint_as_float(r[e >> 5][e & 31]),
                                               p.alpha * __uint_as_float(r[(e + 1) >> 5][(e + 1) & 31]));
      w[q] = *reinterpret_cast<uint32_t*>(&b);
    }
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};\n" ::"r"(rowp + ((c ^ (srow & 7)) << 4)),
                 "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3])
                 : "memory");
  }
}

template <int CG, bool OB = false>
__device__ __forceinline__ void tma_store_epilogue(const TcArgs& p, uint32_t taddr, uint8_t* stage,
                                                   int local, uint32_t warp, uint32_t lane, int row,
                                                   int srow,
                                                   uint32_t empty_cluster_addr, uint64_t* empty_local,
                                                   const CUtensorMap* map_d, int c0, int c1, int c2,
                                                   int c3, int rank_dims, int& ring) {
  constexpr int CW = OB ? 64 : 32;  // output columns per staging chunk (one 128-byte row)
  const int nchunks = (p.BN + CW - 1) / CW;
  const bool issuer = warp == 2 && lane == 0;
  if (p.epi_ring) {
    // Staging in two halves of epi_ring 32-column chunks each (as little as
    // 2 x 16 KiB whatever the tile width): the chunks go out in batches of
    // epi_ring, each batch one bulk group; a batch waits only for the batch
    // before the previous one to have been read.  epi_ring >= nchunks is the
    // whole-tile double buffer.
    const int bs = p.epi_ring;
    for (int j0 = 0; j0 < nchunks; j0 += bs) {
      const int nb = min(bs, nchunks - j0);
      uint8_t* half = stage + (ring & 1) * bs * kRows * kSlabBytes;
      ++ring;
      if (issuer) ptx::bulk_wait_read<1>();
      ptx::named_sync(1, 128);
      if constexpr (OB) {
        for (int jj = 0; jj < nb; ++jj)
          stage_chunk_bf16(p, taddr + (j0 + jj) * 64, half + jj * kRows * kSlabBytes, srow);
      } else
      for (int jj = 0; jj < nb; ++jj) {
        float v[32];
        ptx::tmem_ld32(taddr + (j0 + jj) * 32, v);
        if (srow < 0) continue;
        const uint32_t rowp = ptx::smem(half + jj * kRows * kSlabBytes + srow * kSlabBytes);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(rowp + ((c ^ (srow & 7)) << 4)),
                       "f"(p.alpha * v[4 * c]), "f"(p.alpha * v[4 * c + 1]),
                       "f"(p.alpha * v[4 * c + 2]), "f"(p.alpha * v[4 * c + 3])
                       : "memory");
        }
      }
      const bool last = j0 + nb == nchunks;
      if (last) ptx::tc_fence_before();
      ptx::fence_proxy_async();
      ptx::named_sync(1, 128);
      if (issuer) {
        if (last) {
          if constexpr (CG == 2) ptx::mbar_arrive_remote(empty_cluster_addr);
          else ptx::mbar_arrive(empty_local);
        }
        for (int jj = 0; jj < nb; ++jj) {
          const uint8_t* src = half + jj * kRows * kSlabBytes;
          if (rank_dims == 4) ptx::tma_store_4d(map_d, src, c0 + CW * (j0 + jj), c1, c2, c3);
          else ptx::tma_store_3d(map_d, src, c0 + CW * (j0 + jj), c1, c2);
        }
        ptx::bulk_commit();
      }
    }
    return;
  }
  const int buf_bytes = nchunks * kRows * kSlabBytes;
  uint8_t* sbuf = stage + (p.epi_bufs > 1 ? (local & 1) : 0) * buf_bytes;
  if (issuer) {
    if (p.epi_bufs > 1) ptx::bulk_wait_read<1>();
    else ptx::bulk_wait_read<0>();
  }
  ptx::named_sync(1, 128);
  if constexpr (OB) {
    for (int j = 0; j < nchunks; ++j)
      stage_chunk_bf16(p, taddr + j * 64, sbuf + j * kRows * kSlabBytes, srow);
  } else
  for (int j = 0; j < nchunks; ++j) {
    float v[32];
    ptx::tmem_ld32(taddr + j * 32, v);
    if (srow < 0) continue;  // virtual row without an output pixel
    const uint32_t rowp = ptx::smem(sbuf + j * kRows * kSlabBytes + srow * kSlabBytes);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(rowp + ((c ^ (srow & 7)) << 4)),
                   "f"(p.alpha * v[4 * c]), "f"(p.alpha * v[4 * c + 1]),
                   "f"(p.alpha * v[4 * c + 2]), "f"(p.alpha * v[4 * c + 3])
                   : "memory");
    }
  }
  if (local == 0 && issuer) trace_mark(p, 8);  // TMEM drained to smem (first unit)
  if (local == kTraceUnit && issuer) trace_mark(p, 14);
  ptx::tc_fence_before();
  if (local == kTraceUnit && issuer) trace_mark(p, 18);
  ptx::fence_proxy_async();
  if (local == kTraceUnit && issuer) trace_mark(p, 19);
  ptx::named_sync(1, 128);
  if (issuer) {
    // Accumulator fully read by all 128 threads: hand TMEM back to the MMA.
    if constexpr (CG == 2) ptx::mbar_arrive_remote(empty_cluster_addr);
    else ptx::mbar_arrive(empty_local);
    if (local == kTraceUnit) trace_mark(p, 20);  // (overrides: after the TMEM release)
    for (int j = 0; j < nchunks; ++j) {
      const uint8_t* src = sbuf + j * kRows * kSlabBytes;
      if (rank_dims == 4) ptx::tma_store_4d(map_d, src, c0 + CW * j, c1, c2, c3);
      else ptx::tma_store_3d(map_d, src, c0 + CW * j, c1, c2);
    }
    ptx::bulk_commit();
    if (local == 0) trace_mark(p, 9);  // stores issued (first unit)
    if (local == kTraceUnit) trace_mark(p, 15);
  }
}

// The narrow halo's epilogue (kConvHaloNarrow): the same staging / TMA
// store, for one of two epilogue groups (own slots, barrier, bulk groups),
// with epi_slots staging slots and two TMEM loads per wait.  (Kept apart:
// these run-time generalities measured 10-20% slower on the other modes.)
template <int CG, bool OB = false>
__device__ __forceinline__ void tma_store_epilogue_multi(const TcArgs& p, uint32_t taddr, uint8_t* stage,
                                                         int local, uint32_t warp, uint32_t lane, int row,
                                                   int srow,
                                                   uint32_t empty_cluster_addr, uint64_t* empty_local,
                                                   const CUtensorMap* map_d, int c0, int c1, int c2,
                                                   int c3, int rank_dims, int& ring, uint32_t bar) {
  constexpr int CW = OB ? 64 : 32;  // output columns per staging chunk (one 128-byte row)
  const int nchunks = (p.BN + CW - 1) / CW;
  const bool issuer = (warp & 3) == 2 && lane == 0;  // group leader: warp 2 or 6
  if (p.epi_ring) {
    // Staging in two halves of epi_ring 32-column chunks each (as little as
    // 2 x 16 KiB whatever the tile width): the chunks go out in batches of
    // epi_ring, each batch one bulk group; a batch waits only for the batch
    // before the previous one to have been read.  epi_ring >= nchunks is the
    // whole-tile double buffer.
    // epi_slots slots: up to epi_slots - 1 batches' stores stay in flight
    // while the next is drained (the write-out of an HBM-bound layer needs
    // several tiles of stores outstanding per SM).
    const int bs = p.epi_ring;
    for (int j0 = 0; j0 < nchunks; j0 += bs) {
      const int nb = min(bs, nchunks - j0);
      uint8_t* half = stage + ring * bs * kRows * kSlabBytes;
      TKB_DCHECK(ring < p.epi_slots && (ring + 1) * bs * kRows * kSlabBytes <= p.epi_bytes / p.epi_groups);
      if (++ring == p.epi_slots) ring = 0;
      if (issuer) ptx::bulk_wait_read_dyn(p.epi_slots - 1);
      ptx::epi_sync(bar);
      // TKB_TMEM_PAIRS: two TMEM loads in flight per wait.
      if constexpr (OB) {
        for (int jj = 0; jj < nb; ++jj)
          stage_chunk_bf16(p, taddr + (j0 + jj) * 64, half + jj * kRows * kSlabBytes, srow);
      } else {
#if TKB_TMEM_PAIRS
      for (int jj = 0; jj < nb; jj += 2) {
        uint32_t r[2][32];
        ptx::tmem_ld32_async(taddr + (j0 + jj) * 32, r[0]);
        if (jj + 1 < nb) ptx::tmem_ld32_async(taddr + (j0 + jj + 1) * 32, r[1]);
        ptx::tmem_wait_ld();
        if (srow < 0) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (jj + h >= nb) break;
          const uint32_t rowp =
              ptx::smem(half + (jj + h) * kRows * kSlabBytes + srow * kSlabBytes);
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(rowp + ((c ^ (srow & 7)) << 4)),
                         "f"(p.alpha * __uint_as_float(r[h][4 * c])),
                         "f"(p.alpha * __uint_as_float(r[h][4 * c + 1])),
                         "f"(p.alpha * __uint_as_float(r[h][4 * c + 2])),
                         "f"(p.alpha * __uint_as_float(r[h][4 * c + 3]))
                         : "memory");
          }
        }
      }
#else
      for (int jj = 0; jj < nb; ++jj) {
        float v[32];
        ptx::tmem_ld32(taddr + (j0 + jj) * 32, v);
        if (srow < 0) continue;
        const uint32_t rowp = ptx::smem(half + jj * kRows * kSlabBytes + srow * kSlabBytes);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(rowp + ((c ^ (srow & 7)) << 4)),
                       "f"(p.alpha * v[4 * c]), "f"(p.alpha * v[4 * c + 1]),
                       "f"(p.alpha * v[4 * c + 2]), "f"(p.alpha * v[4 * c + 3])
                       : "memory");
        }
      }
#endif
      }
      const bool last = j0 + nb == nchunks;
      if (last) ptx::tc_fence_before();
      ptx::fence_proxy_async();
      ptx::epi_sync(bar);
      if (issuer) {
        if (last) {
          if constexpr (CG == 2) ptx::mbar_arrive_remote(empty_cluster_addr);
          else ptx::mbar_arrive(empty_local);
        }
        for (int jj = 0; jj < nb; ++jj) {
          const uint8_t* src = half + jj * kRows * kSlabBytes;
          if (rank_dims == 4) ptx::tma_store_4d(map_d, src, c0 + CW * (j0 + jj), c1, c2, c3);
          else ptx::tma_store_3d(map_d, src, c0 + CW * (j0 + jj), c1, c2);
        }
        ptx::bulk_commit();
      }
    }
    return;
  }
  const int buf_bytes = nchunks * kRows * kSlabBytes;
  uint8_t* sbuf = stage + (p.epi_bufs > 1 ? (local & 1) : 0) * buf_bytes;
  if (issuer) {
    if (p.epi_bufs > 1) ptx::bulk_wait_read<1>();
    else ptx::bulk_wait_read<0>();
  }
  ptx::epi_sync(bar);
  if constexpr (OB) {
    for (int j = 0; j < nchunks; ++j)
      stage_chunk_bf16(p, taddr + j * 64, sbuf + j * kRows * kSlabBytes, srow);
  } else
  for (int j = 0; j < nchunks; ++j) {
    float v[32];
    ptx::tmem_ld32(taddr + j * 32, v);
    if (srow < 0) continue;  // virtual row without an output pixel
    const uint32_t rowp = ptx::smem(sbuf + j * kRows * kSlabBytes + srow * kSlabBytes);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(rowp + ((c ^ (srow & 7)) << 4)),
                   "f"(p.alpha * v[4 * c]), "f"(p.alpha * v[4 * c + 1]),
                   "f"(p.alpha * v[4 * c + 2]), "f"(p.alpha * v[4 * c + 3])
                   : "memory");
    }
  }
  if (local == 0 && issuer) trace_mark(p, 8);  // TMEM drained to smem (first unit)
  if (local == kTraceUnit && issuer) trace_mark(p, 14);
  ptx::tc_fence_before();
  if (local == kTraceUnit && issuer) trace_mark(p, 18);
  ptx::fence_proxy_async();
  if (local == kTraceUnit && issuer) trace_mark(p, 19);
  ptx::epi_sync(bar);
  if (issuer) {
    // Accumulator fully read by all 128 threads: hand TMEM back to the MMA.
    if constexpr (CG == 2) ptx::mbar_arrive_remote(empty_cluster_addr);
    else ptx::mbar_arrive(empty_local);
    if (local == kTraceUnit) trace_mark(p, 20);  // (overrides: after the TMEM release)
    for (int j = 0; j < nchunks; ++j) {
      const uint8_t* src = sbuf + j * kRows * kSlabBytes;
      if (rank_dims == 4) ptx::tma_store_4d(map_d, src, c0 + CW * j, c1, c2, c3);
      else ptx::tma_store_3d(map_d, src, c0 + CW * j, c1, c2);
    }
    ptx::bulk_commit();
    if (local == 0) trace_mark(p, 9);  // stores issued (first unit)
    if (local == kTraceUnit) trace_mark(p, 15);
  }
}

// Gather producer (conv fallback for channel counts / strides the TMA box
// cannot express): 128 threads build the 128-pixel x 32-element fp32 K-slab
// of the implicit patch matrix directly in the 128-byte-swizzled layout the
// UMMA descriptor expects, reading the NHWC input through the read-only
// cache (neighbouring pixels share most taps, so it is served from L1/L2).
// K order is the reference's (x, y, c) (conv.hpp:286-292); K is zero-padded
// to whole slabs.  Thread t owns 16-byte chunk q = t % 8 of rows
// t / 8 + 16 i; completion is an mbarrier arrival (count 128 per CTA) on the
// leader's `full` barrier after a proxy fence.
template <int CG>
__device__ __forceinline__ void gather_producer(const TcArgs& p, uint8_t* base, int stage_bytes,
                                                uint64_t* full, uint64_t* empty,
                                                const int2* ktab, uint32_t warp, uint32_t lane,
                                                uint32_t rank, int unit, int nunits, int total) {
  const int group = (int)(warp - 6) / 4;
  const int t = (int)((warp - 6) & 3) * 32 + (int)lane;
  const int q = t & 7;
  const int r0 = t >> 3;
  const uint32_t sbase = ptx::smem(base);
  // Groups take alternate K-slabs of the CTA's slab sequence.  (Owning
  // alternate *tiles* would let a group run more than one phase ahead on a
  // stage barrier once a tile has more slabs than stages, and the mbarrier
  // parity test cannot tell those phases apart.)
  int local = 0;
  for (int tt = unit; tt < total; tt += nunits, ++local) {
    const int seq0 = local * p.num_kb;
    if (p.num_kb == 1 && (seq0 % kGatherGroups) != group) continue;
    const int m_blk = tt % p.num_m;
    // Pixel geometry of this thread's 8 rows (rows r0 + 16 i), walked
    // incrementally from the first row: no per-row division.
    const float* rowp[8];
    int ih0[8], iw0[8];
    {
      int m = m_blk * kRows * CG + (int)rank * kRows + r0;
      int ow = m % p.OW;
      int rest = m / p.OW;
      int oh = rest % p.OH;
      int n = rest / p.OH;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const bool ok = m < p.M;
        ih0[i] = ok ? oh * p.stride - p.pad_t : -(1 << 28);
        iw0[i] = ow * p.stride - p.pad_l;
        rowp[i] = p.in + (((long long)n * p.H + ih0[i]) * p.W + iw0[i]) * p.C;
        m += 16;
        ow += 16;
        while (ow >= p.OW) {
          ow -= p.OW;
          if (++oh == p.OH) {
            oh = 0;
            ++n;
          }
        }
      }
    }
    for (int kb = 0; kb < p.num_kb; ++kb) {
      const int seq = seq0 + kb;  // slab sequence of this CTA
      if (seq % kGatherGroups != group) continue;
      const int stage = seq % p.stages;
      const uint32_t phase = (uint32_t)(seq / p.stages) & 1u;
      int2 kd[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) kd[u] = ktab[kb * 32 + q * 4 + u];
      // Loads first (they do not touch the stage), then wait for the slot.
      float v[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int x = kd[u].y >> 16, y = (kd[u].y << 16) >> 16;
          const int ih = ih0[i] + x, iw = iw0[i] + y;
          v[i][u] = ((unsigned)ih < (unsigned)p.H && (unsigned)iw < (unsigned)p.W)
                        ? __ldg(rowp[i] + kd[u].x)
                        : 0.0f;
        }
      }
      if (local == kTraceUnit && t == 0) trace_mark(p, 16);
      ptx::mbar_wait_sleep(&empty[stage], phase ^ 1);
      const uint32_t sa = sbase + stage * stage_bytes;
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int r = r0 + 16 * i;
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};\n" ::"r"(
                         sa + r * kSlabBytes + ((q ^ (r & 7)) << 4)),
                     "f"(v[i][0]), "f"(v[i][1]), "f"(v[i][2]), "f"(v[i][3])
                     : "memory");
      }
      ptx::fence_proxy_async();
      ptx::named_sync(2 + group, 128);
      if (t == 0) {
        // Cluster-scope release: the leader's MMA reads these generic-proxy
        // writes (CTA-scope would not order them for another CTA's observer).
        if constexpr (CG == 2) ptx::mbar_arrive_cluster(ptx::map_to_rank(ptx::smem(&full[stage]), 0));
        else ptx::mbar_arrive(&full[stage]);
        if (local == kTraceUnit) trace_mark(p, 17);
      }
    }
  }
}

template <int MODE, int CG, bool TF32, bool OB>
__global__ void __launch_bounds__(threads_of<MODE>(), 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ CUtensorMap map_d, TcArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  constexpr int BM = kRows * CG;
  const int a_bytes = halo_like<MODE>() ? p.halo_bytes : kRows * kSlabBytes;
  const int b_rows = p.BN / CG;
  const int b_bytes = b_rows * kSlabBytes;
  const int stage_bytes =
      a_bytes + (halo_like<MODE>() ? (p.resident ? 0 : p.taps) : 1) * b_bytes;
  // resident filter (halo mode): taps x cchunks slabs after the stages
  uint8_t* fres = base + p.stages * stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(
      base + p.stages * stage_bytes + (p.resident ? p.taps * p.cchunks * b_bytes : 0));
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStages;
  uint64_t* tmem_full = bars + 2 * kMaxStages;
  uint64_t* tmem_empty = tmem_full + kMaxAcc;
  uint64_t* fbar = tmem_empty + kMaxAcc;  // resident-filter barrier
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fbar + 1);
  // TMA-store staging: epi_bufs x (BN/32) swizzled 128-row x 128-byte tiles
  uint8_t* epi_stage = reinterpret_cast<uint8_t*>(bars) + 1024;
  // gather mode: K -> {element offset (x*W + y)*C + c, (x << 16) | y} table,
  // K padded to whole slabs with out-of-window markers.
  int2* ktab = reinterpret_cast<int2*>(epi_stage + p.epi_bytes);
#if TKB_CHECKED
  if (threadIdx.x == 0) {
    uint32_t dsmem;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dsmem));
    const long long end = (reinterpret_cast<uint8_t*>(ktab) - smem_raw) +
                          (MODE == kConvGather ? (long long)p.num_kb * 32 * 8 : 0);
    TKB_DCHECK(end <= (long long)dsmem);                        // layout fits the allocation
    TKB_DCHECK(reinterpret_cast<uint8_t*>(tmem_slot + 1) <= epi_stage);  // barriers before staging
    TKB_DCHECK(stage_bytes % 1024 == 0 && (reinterpret_cast<uintptr_t>(base) & 1023) == 0);
    TKB_DCHECK(p.stages >= 2 && p.stages <= kMaxStages && p.acc_slots <= kMaxAcc);
    TKB_DCHECK(p.acc_slots * p.acc_cols <= 2 * kAccCols && p.BN <= p.acc_cols);  // TMEM ring
    TKB_DCHECK(p.splits >= 1 && p.splits <= kMaxSplits);
  }
#endif

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  const uint32_t rank = CG == 2 ? ptx::cluster_rank() : 0;
  const bool leader = rank == 0;
  if (threadIdx.x == 0) trace_mark(p, 0);  // entry

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&map_a);
    ptx::prefetch_tmap(&map_b);
    if (p.store_tma) ptx::prefetch_tmap(&map_d);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      ptx::mbar_init(&full[s], MODE == kConvGather ? 1 + CG : 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < p.acc_slots; ++a) {
      ptx::mbar_init(&tmem_full[a], 1);
      ptx::mbar_init(&tmem_empty[a], CG);
    }
    ptx::mbar_init(fbar, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_cg<CG, 2 * kAccCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // Programmatic dependent launch: the setup above overlapped the previous
  // kernel's tail; nothing below may touch global memory before it is done.
  // The next kernel may be scheduled as soon as SMs free up.
  ptx::griddep_launch_dependents();
  ptx::griddep_wait();
  if (threadIdx.x == 0) trace_mark(p, 1);  // barriers + TMEM ready

  const int total = p.tail_q > 1 ? p.tail_start + p.tail_kb * p.tail_P
                                  : p.num_m * p.num_n * p.batch * p.splits;
  const int unit = blockIdx.x / CG, nunits = gridDim.x / CG;

  if (halo_like<MODE>() && warp == 0) {
    // ---------------- TMA producer, halo mode ----------------
    // One super-stage per (tile, channel chunk): the (TH+R) x P halo box of
    // this CTA's output rows plus the R*S filter slabs of the chunk.
    if (ptx::elect_one()) {
      if (p.resident) {
        // Every tile of this CTA has the same feature block (host ensures
        // nunits % num_n == 0): stage its filter slice once.
        uint32_t fb = ptx::smem(fbar);
        if constexpr (CG == 2) fb = ptx::map_to_rank(fb, 0);
        if (leader) ptx::mbar_arrive_expect_tx(fbar, CG * p.taps * p.cchunks * b_bytes);
        const int n_blk = unit % p.num_n;
        for (int tap = 0; tap < p.taps; ++tap)
          for (int ch = 0; ch < p.cchunks; ++ch)
            ptx::tma2<CG>(fres + (tap * p.cchunks + ch) * b_bytes, &map_b, fb,
                          tap * p.cchunks * p.ek + ch * p.ek, n_blk * p.BN + rank * b_rows);
      }
      int stage = 0;
      uint32_t phase = 0;
      for (int t = unit; t < total; t += nunits) {
        const int m_blk = fdiv(t, p.fd_num_n);
        const int n_blk = t - m_blk * p.num_n;
        const PixTile pt = pix_tile(p, m_blk);
        for (int ch = 0; ch < p.cchunks; ++ch) {
          ptx::mbar_wait_sleep(&empty[stage], phase ^ 1);
          uint8_t* sa = base + stage * stage_bytes;
          uint32_t fb = ptx::smem(&full[stage]);
          if constexpr (CG == 2) fb = ptx::map_to_rank(fb, 0);
          if (leader)
            ptx::mbar_arrive_expect_tx(
                &full[stage],
                CG * (MODE == kConvHaloNarrow ? stage_bytes - a_bytes + p.halo_tx : stage_bytes));
          const int c0 = ch * p.ek;
          if constexpr (MODE == kConvHaloNarrow) {
            if (t == unit + kTraceUnit * nunits) trace_mark(p, 16);
            // Phase-split input [N][H][s][W2][cp] (pad_phase_kernel): phase
            // (px, py) of the tile = the 16-pixel run of column phase py
            // from w2 = ow0, rows oh*s - pad_t + px stepping by s -- each
            // box row one contiguous 256-byte run.
            for (int ph = 0; ph < p.nphase; ++ph) {
              const int px = p.stride == 1 ? 0 : ph >> 1, py = p.stride == 1 ? 0 : ph & 1;
              ptx::tma4<CG>(sa + ph * p.phase_bytes, &map_a, fb, pt.ow0 * p.C, py,
                            (pt.oh0 + rank * p.TH) * p.stride - p.pad_t + px, pt.img);
            }
          } else {
            ptx::tma4<CG>(sa, &map_a, fb, c0, pt.ow0 - p.pad_l, pt.oh0 + rank * p.TH - p.pad_t,
                          pt.img);
          }
          if (!p.resident)
            for (int tap = 0; tap < p.taps; ++tap)
              ptx::tma2<CG>(sa + a_bytes + tap * b_bytes, &map_b, fb, tap * p.cchunks * p.ek + c0,
                            n_blk * p.BN + rank * b_rows);
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (halo_like<MODE>() && warp == 1) {
    // ---------------- MMA issuer, halo mode (leader CTA) ----------------
    // Tap (x, y) reads the halo from row x*P + y on: output row v = h*P + w
    // needs halo pixel (h + x, w + y), a constant shift in the virtual
    // pitch-P layout.
    if (leader) {
      const uint32_t idesc = ptx::idesc(BM, p.BN, TF32);
      if (p.resident) ptx::mbar_wait(fbar, 0);
      const uint32_t fres_s = ptx::smem(fres);
      const uint64_t kdesc = ptx::desc_sw128(0);
      uint64_t tap_off[9];  // halo row shift of tap (x, y), in 16-byte units
#pragma unroll
      for (int tap = 0; tap < 9; ++tap) {
        const int x = tap / p.S, y = tap - (tap / p.S) * p.S;
        tap_off[tap] = (uint64_t)((x * p.P + y) * (kSlabBytes / 16));
      }
      // Narrow halo: taps in (phase, row, column) order, two per MMA.
      uint32_t mma_off[kMaxNarrowMma], mma_lbo[kMaxNarrowMma];
      int n_mma = 0;
      if (MODE == kConvHaloNarrow) {
        const int s = p.stride;
        int q = 0;
        for (int ph = 0; ph < p.nphase; ++ph) {
          const int px = ph / s, py = ph - (ph / s) * s;
          for (int x = px; x < p.R; x += s)
            for (int y = py; y < p.S; y += s) {
              const uint32_t off = ph * p.phase_bytes + ((x / s) * p.P + y / s) * 16;
              TKB_DCHECK((q >> 1) < kMaxNarrowMma && off < (uint32_t)p.halo_tx);
              if ((q & 1) == 0) {
                mma_off[q >> 1] = off;
                mma_lbo[q >> 1] = 0;  // (odd last tap: paired with zero filter rows)
              } else {
                mma_lbo[q >> 1] = off - mma_off[q >> 1];
              }
              ++q;
            }
        }
        n_mma = (q + 1) >> 1;
      }
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = unit; t < total; t += nunits, ++local) {
        const int acc = local & (p.acc_slots - 1);
        const uint32_t acc_phase = (uint32_t)(local >> p.acc_shift) & 1u;
        ptx::mbar_wait_sleep(&tmem_empty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * p.acc_cols;
        if (local == kTraceUnit && lane == 0) trace_mark(p, 10);
        for (int ch = 0; ch < p.cchunks; ++ch) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (local == 0 && lane == 0) trace_mark(p, 2);
          if (local == kTraceUnit && lane == 0) trace_mark(p, 11);
          if constexpr (MODE == kConvHaloNarrow) {
            // Two taps (2 x 16-byte pixels = one 32-byte K step) per MMA:
            // A = the pair's shifted halo views (start = first tap, LBO =
            // gap to the second), B = the filter's K rows of the pair.  The
            // (start offset, LBO) of every MMA is tabulated once per CTA.
            if (ptx::elect_one()) {
              const uint32_t sa = ptx::smem(base + stage * stage_bytes);
              const uint64_t bd0 = kdesc + ((p.resident ? fres_s : sa + (uint32_t)a_bytes) >> 4);
              for (int kk = 0; kk < n_mma; ++kk) {
                const uint64_t bd = bd0 + (uint64_t)(kk >> 2) * (b_bytes >> 4) + 2 * (kk & 3);
                ptx::mma_cg<CG, TF32>(d_tmem, ptx::desc_none(sa + mma_off[kk], mma_lbo[kk], 128), bd,
                                      idesc, kk != 0);
              }
              ptx::commit_cg<CG>(&empty[stage]);
              ptx::commit_cg<CG>(&tmem_full[acc]);
              if (local == kTraceUnit) trace_mark(p, 12);
            }
            __syncwarp();
            if (++stage == p.stages) {
              stage = 0;
              phase ^= 1;
            }
            continue;
          }
          if (ptx::elect_one()) {
            // Descriptors are linear in the 16-byte address field: build
            // the stage bases once, then every MMA is two 64-bit adds.
            const uint32_t sa = ptx::smem(base + stage * stage_bytes);
            const uint64_t ad0 = kdesc + (sa >> 4);
            const uint64_t bd0 = kdesc + ((p.resident ? fres_s + (uint32_t)(ch * b_bytes)
                                                      : sa + (uint32_t)a_bytes) >> 4);
            const uint64_t b_tap = (uint64_t)((p.resident ? p.cchunks : 1) * b_bytes) >> 4;
#pragma unroll
            for (int tap = 0; tap < 9; ++tap) {
              if (tap < p.taps) {
                const uint64_t ad = ad0 + tap_off[tap];
                const uint64_t bd = bd0 + b_tap * tap;
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)
                  ptx::mma_cg<CG, TF32>(d_tmem, ad + 2 * kk, bd + 2 * kk, idesc,
                                        (ch | tap | kk) != 0);
              }
            }
            ptx::commit_cg<CG>(&empty[stage]);
            if (ch == p.cchunks - 1) ptx::commit_cg<CG>(&tmem_full[acc]);
          }
          __syncwarp();
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 0) {
    // ---------------- TMA producer (every CTA) ----------------
    if (ptx::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = unit; t < total; t += nunits) {
        const Unit u = decode_unit(p, t);
        const int m_blk = u.m_blk, n_blk = u.n_blk, z = u.z;
        PixTile pt{0, 0, 0};
        int i2c_w = 0, i2c_h = 0, i2c_n = 0;  // im2col: traversal start of the CTA's rows
        if constexpr (MODE == kConvIm2col) {
          const int m0 = m_blk * BM + rank * kRows;
          const int plane = p.OH * p.OW;
          i2c_n = m0 / plane;
          const int r = m0 - i2c_n * plane;
          const int oh = r / p.OW;
          i2c_h = oh * p.stride - p.pad_t;
          i2c_w = (r - oh * p.OW) * p.stride - p.pad_l;
        }
        if constexpr (MODE == kConvPixN) pt = pix_tile(p, n_blk);
        if constexpr (MODE == kConvPixM) pt = pix_tile(p, m_blk);
        for (int kb = u.kb0; kb < u.kb1; ++kb) {
          ptx::mbar_wait_sleep(&empty[stage], phase ^ 1);
          uint8_t* sa = base + stage * stage_bytes;
          uint8_t* sb = sa + a_bytes;
          uint32_t fb = ptx::smem(&full[stage]);
          if constexpr (CG == 2) fb = ptx::map_to_rank(fb, 0);
          if (leader)
            ptx::mbar_arrive_expect_tx(&full[stage],
                                       CG * (MODE == kConvGather ? b_bytes : stage_bytes));
          const int k0 = kb * p.ek;
          int c0 = 0, dy = 0, dx = 0;
          if constexpr (MODE != kPlain) {
            const int tap = kb / p.cchunks;
            c0 = (kb - tap * p.cchunks) * p.ek;
            dy = tap % p.S - p.pad_l;
            dx = tap / p.S - p.pad_t;
          }
          if constexpr (MODE == kPlain) {
            if (p.a_mn)  // MN-major A: M blocks of 32 tf32 / 64 bf16 (128 bytes)
              ptx::tma3<CG>(sa, &map_a, fb, 0, k0, (m_blk * BM + rank * kRows) / (TF32 ? 32 : 64));
            else ptx::tma3<CG>(sa, &map_a, fb, k0, m_blk * BM + rank * kRows, z);
            ptx::tma3<CG>(sb, &map_b, fb, k0, n_blk * p.BN + rank * b_rows, z);
          } else if constexpr (MODE == kConvIm2col) {
            // 128 consecutive output pixels (across rows and images) from
            // the traversal start of this CTA's first pixel, shifted by the tap.
            const int tap = kb / p.cchunks;
            const int ty = tap % p.S;
            ptx::tma4_im2col<CG>(sa, &map_a, fb, c0, i2c_w, i2c_h, i2c_n, (uint16_t)ty,
                                 (uint16_t)(tap / p.S));
            ptx::tma2<CG>(sb, &map_b, fb, k0, n_blk * p.BN + rank * b_rows);
          } else if constexpr (MODE == kConvPixN) {
            ptx::tma2<CG>(sa, &map_a, fb, k0, m_blk * BM + rank * kRows);
            if (p.flat) {
              const int r = n_blk * p.tileH + (int)rank * p.boxH;
              ptx::tma4<CG>(sb, &map_b, fb, c0, dy, (r % p.OH) * p.stride + dx, r / p.OH);
            } else if (p.imgs > 1)  // each CTA boxes its imgs / CG whole images
              ptx::tma4<CG>(sb, &map_b, fb, c0, pt.ow0 * p.stride + dy, pt.oh0 * p.stride + dx,
                            pt.img + (int)rank * (p.imgs / CG));
            else
              ptx::tma4<CG>(sb, &map_b, fb, c0, pt.ow0 * p.stride + dy,
                            (pt.oh0 + rank * p.boxH) * p.stride + dx, pt.img);
          } else if constexpr (MODE == kConvPixM) {
            ptx::tma4<CG>(sa, &map_a, fb, c0, pt.ow0 * p.stride + dy,
                          (pt.oh0 + rank * p.boxH) * p.stride + dx, pt.img);
            ptx::tma2<CG>(sb, &map_b, fb, k0, n_blk * p.BN + rank * b_rows);
          } else {
            ptx::tma2<CG>(sb, &map_b, fb, k0, n_blk * p.BN + rank * b_rows);
          }
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA) ----------------
    if (leader) {
      const bool a_mn = MODE == kPlain && p.a_mn;
      const uint32_t idesc = ptx::idesc(BM, p.BN, TF32) | (a_mn ? (1u << 15) : 0u);
      const uint64_t kdesc = ptx::desc_sw128(0);
      const uint64_t kdesc_mn =
          TF32 ? ptx::desc_sw128_mn(0, 4096, 512) : ptx::desc_sw128_mn16(0, 8192, 1024);
      int stage = 0;
      uint32_t phase = 0;
      int nlocal = 0;
      for (int t = unit; t < total; t += nunits) {
        const Unit u = decode_unit(p, t);
        if (u.kb0 >= u.kb1) continue;  // empty tail segment
        const int local = nlocal++;
        const int acc = local & (p.acc_slots - 1);
        const uint32_t acc_phase = (uint32_t)(local >> p.acc_shift) & 1u;
        ptx::mbar_wait_sleep(&tmem_empty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        if (local == kTraceUnit && lane == 0) trace_mark(p, 10);
        const uint32_t d_tmem = tmem_base + acc * p.acc_cols;
        for (int kb = u.kb0; kb < u.kb1; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (local == 0 && kb == u.kb0 && lane == 0) trace_mark(p, 2);  // first slab landed
          if (local == 0 && kb == u.kb1 - 1 && lane == 0) trace_mark(p, 3);  // last slab landed
          if (local == kTraceUnit && kb == u.kb0 && lane == 0) trace_mark(p, 11);
          if (ptx::elect_one()) {
            const uint32_t sa = ptx::smem(base + stage * stage_bytes);
            const uint64_t ad = (a_mn ? kdesc_mn : kdesc) + (sa >> 4);
            const uint64_t bd = kdesc + ((sa + (uint32_t)a_bytes) >> 4);
            // K step of one MMA (32 bytes of K): MN-major tf32 two 512-B
            // atoms (1 KiB), MN-major bf16 two 1-KiB atoms (2 KiB), K-major 32 B
            const uint64_t a_step = a_mn ? (TF32 ? 64 : 128) : 2;
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)
              ptx::mma_cg<CG, TF32>(d_tmem, ad + a_step * kk, bd + 2 * kk, idesc,
                                    (kb != u.kb0 || kk != 0));
            ptx::commit_cg<CG>(&empty[stage]);
            if (kb == u.kb1 - 1) ptx::commit_cg<CG>(&tmem_full[acc]);
            if (kb == u.kb1 - 1 && local == kTraceUnit) trace_mark(p, 12);
          }
          __syncwarp();
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (MODE == kConvGather && warp >= 6) {
    // ---------------- pixel gather (warps 6.., every CTA) ----------------
    {
      const int tid = (int)(warp - 6) * 32 + (int)lane;
      for (int k = tid; k < p.num_kb * 32; k += 128 * kGatherGroups) {
        int2 e;
        if (k < p.Kreal) {
          const int c = k % p.C, tap = k / p.C;
          const int y = tap % p.S, x = tap / p.S;
          e.x = (x * p.W + y) * p.C + c;
          e.y = (x << 16) | (y & 0xFFFF);
        } else {
          e.x = 0;
          e.y = (1 << 30);  // x huge: always outside the input
        }
        ktab[k] = e;
      }
      ptx::named_sync(2 + kGatherGroups, 128 * kGatherGroups);  // after the group barriers
    }
    gather_producer<CG>(p, base, stage_bytes, full, empty, ktab, warp, lane, rank, unit, nunits,
                        total);
  } else {
    // ---------------- epilogue (warps 2..5, every CTA) ----------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    uint32_t empty_base = ptx::smem(&tmem_empty[0]);
    if constexpr (CG == 2) empty_base = ptx::map_to_rank(empty_base, 0);
    int nlocal = 0;
    int ering = 0;  // staging chunk sequence (chunk-ring epilogue)
    // Epilogue group eg takes the CTA's tiles local % epi_groups == eg, with
    // its own half of the staging area, bulk groups and named barrier.
    constexpr bool kMulti = MODE == kConvHaloNarrow;  // two epilogue groups
    const int eg = kMulti ? (int)(warp - 2) >> 2 : 0;
    const uint32_t ebar = (uint32_t)eg;
    const bool elead = kMulti ? ((warp & 3) == 2 && lane == 0) : (warp == 2 && lane == 0);
    uint8_t* const epi_mine =
        epi_stage + (kMulti && p.epi_groups > 1 ? eg * (p.epi_bytes / 2) : 0);
    auto esync = [&]() {
      if constexpr (kMulti) ptx::epi_sync(ebar);
      else ptx::named_sync(1, 128);
    };
    for (int t = unit; t < total; t += nunits) {
      const Unit u = decode_unit(p, t);
      if (u.kb0 >= u.kb1) continue;  // empty tail segment
      const int local = nlocal++;
      if constexpr (kMulti) {
        if (eg >= p.epi_groups || (local & (p.epi_groups - 1)) != eg) continue;  // 1 or 2 groups
      }
      const int m_blk = u.m_blk, n_blk = u.n_blk, z = u.z;
      const int acc = local & (p.acc_slots - 1);
      const uint32_t acc_phase = (uint32_t)(local >> p.acc_shift) & 1u;
      ptx::mbar_wait_sleep(&tmem_full[acc], acc_phase);
      ptx::tc_fence_after();
      if (local == 0 && warp == 2 && lane == 0) trace_mark(p, 4);  // first accumulator ready
      if (local == 1 && warp == 2 && lane == 0) trace_mark(p, 5);  // second accumulator ready
      if (local == kTraceUnit && warp == 2 && lane == 0) trace_mark(p, 13);
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * p.acc_cols;

      if ((plain_like<MODE>() || MODE == kConvPixN) && u.slot >= 0) {
        store_tail_piece(p, taddr, u.slot, rank, CG, row);
        ptx::tc_fence_before();
        esync();
        if (elead) {
          if constexpr (CG == 2) ptx::mbar_arrive_remote(empty_base + 8u * acc);
          else ptx::mbar_arrive(&tmem_empty[acc]);
        }
        continue;
      }
      if constexpr (halo_like<MODE>()) {
        const int hm = fdiv(t, p.fd_num_n), hn = t - hm * p.num_n;
        const PixTile pt = pix_tile(p, hm);
        const int h = row / kHaloPitch, w = row % kHaloPitch;
        const int srow = w < p.TW ? h * p.TW + w : -1;
        if (p.direct_store) {
          // Each thread owns one output pixel (TMEM lane): its BN features
          // leave as 16-byte streaming stores straight from the registers
          // (no staging, no bulk store; L2 merges the lanes' lines).
          const int oh = pt.oh0 + rank * p.TH + h, ow = pt.ow0 + w;
          const bool ok = srow >= 0 && oh < p.OH && ow < p.OW;
          float* dst = p.d + (((long long)pt.img * p.OH + oh) * p.OW + ow) * p.Kout + hn * p.BN;
          for (int col = 0; col < p.BN; col += 32) {
            float v[32];
            ptx::tmem_ld32(taddr + col, v);
            if (ok) {
#pragma unroll
              for (int q = 0; q < 8; ++q)
                __stcs(reinterpret_cast<float4*>(dst + col) + q,
                       make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
            }
          }
          ptx::tc_fence_before();
          esync();
          if (elead) {
            if constexpr (CG == 2) ptx::mbar_arrive_remote(empty_base + 8u * acc);
            else ptx::mbar_arrive(&tmem_empty[acc]);
          }
          continue;
        }
        if constexpr (kMulti)
          tma_store_epilogue_multi<CG, OB>(p, taddr, epi_mine, local, warp, lane, row, srow,
                                       empty_base + 8u * acc, &tmem_empty[acc], &map_d, hn * p.BN,
                                       pt.ow0, pt.oh0 + rank * p.TH, pt.img, 4, ering, ebar);
        else
          tma_store_epilogue<CG, OB>(p, taddr, epi_mine, local, warp, lane, row, srow,
                                 empty_base + 8u * acc, &tmem_empty[acc], &map_d, hn * p.BN,
                                 pt.ow0, pt.oh0 + rank * p.TH, pt.img, 4, ering);
        continue;
      } else if constexpr (MODE == kConvGather) {
        tma_store_epilogue<CG, OB>(p, taddr, epi_mine, local, warp, lane, row, row, empty_base + 8u * acc,
                               &tmem_empty[acc], &map_d, n_blk * p.BN, m_blk * BM + rank * kRows,
                               0, 0, 3, ering);
        continue;
      } else if constexpr (plain_like<MODE>()) {
        const int m = m_blk * BM + rank * kRows + row;
        // Split-K partials (non-TMA path: dense column-major output, batch 1)
        // land at part + sp * part_stride in the output's own layout.
        float* dz = (p.splits > 1 ? p.part + u.sp * p.part_stride : p.d) + (long long)z * p.d_batch;
        const float* cz = p.read_c ? p.c + (long long)z * p.d_batch : nullptr;
        if (p.store_tma) {
          tma_store_epilogue<CG, OB>(p, taddr, epi_mine, local, warp, lane, row, row, empty_base + 8u * acc,
                                 &tmem_empty[acc], &map_d, n_blk * p.BN,
                                 m_blk * BM + rank * kRows, u.sp * p.batch + z, 0, 3, ering);
          continue;
        }
        for (int col = 0; col < p.BN; col += 32) {
          float v[32];
          ptx::tmem_ld32(taddr + col, v);
          const int n0 = n_blk * p.BN + col;
          if (!p.read_c && p.d_sm == 1 && n0 + 32 <= p.N && col + 32 <= p.BN) {
            // Column-major C, whole 32-column chunk in range: lanes = 32
            // consecutive rows, each j one coalesced 128-byte store; no
            // per-element predicates or 64-bit index math.
            if (m < p.M) {
              float* dst = dz + m + (long long)n0 * p.d_sn;
#pragma unroll
              for (int j = 0; j < 32; ++j) dst[(long long)j * p.d_sn] = p.alpha * v[j];
            }
            continue;
          }
          if (m < p.M) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int n = n0 + j;
              if (col + j < p.BN && n < p.N) {
                const long long off = (long long)m * p.d_sm + (long long)n * p.d_sn;
                float r = p.alpha * v[j];
                if (p.read_c) r = fmaf(p.beta, cz[off], r);
                dz[off] = r;
              }
            }
          }
        }
      } else if constexpr (MODE == kConvPixN) {
        const PixTile pt = pix_tile(p, n_blk);
        const int m = m_blk * BM + rank * kRows + row;  // output feature
        const bool m_ok = m < p.Kout;
        for (int col = 0; col < p.BN; col += 32) {
          float v[32];
          ptx::tmem_ld32(taddr + col, v);
          // Lane l resolves column col + l to its NHWC pixel offset once; the
          // warp then walks the 32 columns with shuffles (one coalesced
          // 128-byte store of 32 consecutive features per column).
          const int n = col + (int)lane;
          int oh, ow, img;
          if (p.flat) {
            const int r = n_blk * p.tileH + n / p.Wb;
            img = r / p.OH;
            oh = r - img * p.OH;
            ow = n - (n / p.Wb) * p.Wb;
          } else {
            const int per = p.Wb * p.tileH;  // columns per image of the tile
            const int ii = n / per, nn = n - (n / per) * per;
            const int h = nn / p.Wb, w = nn - (nn / p.Wb) * p.Wb;
            oh = pt.oh0 + h;
            ow = pt.ow0 + w;
            img = pt.img + ii;
          }
          const bool ok = n < p.BN && oh < p.OH && ow < p.OW && img < p.Nimg;
          const long long pix_off =
              ok ? (((long long)img * p.OH + oh) * p.OW + ow) * p.Kout : -1ll;
          float* dst = p.splits > 1 ? p.part + u.sp * p.part_stride : p.d;
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const long long o = __shfl_sync(0xffffffffu, pix_off, j);
            if constexpr (OB) {  // (OB kernels run only without split partials)
              if (o >= 0 && m_ok) reinterpret_cast<__nv_bfloat16*>(p.d)[o + m] = __float2bfloat16_rn(v[j]);
            } else {
              if (o >= 0 && m_ok) dst[o + m] = v[j];
            }
          }
        }

      } else {
        const PixTile pt = pix_tile(p, m_blk);
        tma_store_epilogue<CG, OB>(p, taddr, epi_mine, local, warp, lane, row, row, empty_base + 8u * acc,
                               &tmem_empty[acc], &map_d, n_blk * p.BN, pt.ow0,
                               pt.oh0 + rank * p.boxH, pt.img, 4, ering);
        continue;
      }
      ptx::tc_fence_before();
      esync();
      if (elead) {
        if constexpr (CG == 2) ptx::mbar_arrive_remote(empty_base + 8u * acc);
        else ptx::mbar_arrive(&tmem_empty[acc]);
      }
    }
  }

  if ((warp == 2 || (MODE == kConvHaloNarrow && warp == 6)) && lane == 0 && p.store_tma)
    ptx::bulk_wait<0>();
  if (warp == 2 && lane == 0) trace_mark(p, 6);  // epilogue stores complete
  ptx::tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) trace_mark(p, 7);  // exit
  if constexpr (CG == 2) ptx::cluster_sync();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc_cg<CG, 2 * kAccCols>(tmem_base);
  }
}

// ---------------------------------------------------------------------------
// Host: tensor maps via the driver entry point (no libcuda link needed).
// ---------------------------------------------------------------------------
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                   CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  if (!fn) fail(TK_ERR_CUDA, "cuTensorMapEncodeTiled unavailable from the driver");
  return fn;
}

// Tensor maps are memoised per calling thread on every argument of the
// encode (base pointer included): a repeated call with the same buffers pays
// a hash lookup instead of a driver encode (~1-2 us each, three per launch).
struct MapKey {
  const void* base;
  int kind, esize, rank, swz;
  cuuint64_t dims[5], strides[4];
  cuuint32_t box[5], trav[5];
  int lower[2], upper[2];
  cuuint32_t chans, pixels;
};

struct MapMemo {
  std::unordered_map<std::string, CUtensorMap> maps;
  static std::string key(const MapKey& k) {
    return std::string(reinterpret_cast<const char*>(&k), sizeof k);
  }
  const CUtensorMap* find(const MapKey& k) const {
    auto it = maps.find(key(k));
    return it == maps.end() ? nullptr : &it->second;
  }
  void put(const MapKey& k, const CUtensorMap& m) {
    if (maps.size() >= 4096) maps.clear();
    maps.emplace(key(k), m);
  }
};

MapMemo& map_memo() {
  thread_local MapMemo memo;
  return memo;
}

// esize: 4 (fp32 / tf32) or 2 (bf16).  dims[0] is the contiguous K axis.
CUtensorMap make_map(const void* base, int esize, int rank, const cuuint64_t* dims,
                     const cuuint64_t* strides, const cuuint32_t* box,
                     const cuuint32_t* traversal = nullptr,
                     CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  MapKey key;
  std::memset(&key, 0, sizeof key);
  key.base = base;
  key.kind = 0;
  key.esize = esize;
  key.rank = rank;
  key.swz = (int)swz;
  for (int i = 0; i < rank; ++i) {
    key.dims[i] = dims[i];
    key.box[i] = box[i];
    key.trav[i] = traversal ? traversal[i] : 1;
    if (i + 1 < rank) key.strides[i] = strides[i];
  }
  if (const CUtensorMap* hit = map_memo().find(key)) return *hit;
  CUtensorMap m;
  cuuint32_t elem_strides[5] = {1, 1, 1, 1, 1};
  if (traversal)
    for (int i = 0; i < rank; ++i) elem_strides[i] = traversal[i];
  const CUresult r = encode_fn()(
      &m, esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
      (cuuint32_t)rank, const_cast<void*>(base), dims, strides, box, elem_strides,
      CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(TK_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  map_memo().put(key, m);
  return m;
}

using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const int*, const int*,
                                    cuuint32_t, cuuint32_t, const cuuint32_t*, CUtensorMapInterleave,
                                    CUtensorMapSwizzle, CUtensorMapL2promotion,
                                    CUtensorMapFloatOOBfill);

EncodeIm2colFn encode_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(ptr);
  });
  if (!fn) fail(TK_ERR_CUDA, "cuTensorMapEncodeIm2col unavailable from the driver");
  return fn;
}

// [batch][rows][K] K-major operand, box {slab, box_rows, 1}.
CUtensorMap map_rows(const void* base, int esize, long long K, long long rows, long long batch,
                     long long batch_stride, int box_rows) {
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)K * esize,
                           (cuuint64_t)(batch_stride ? batch_stride : K * rows) * esize};
  cuuint32_t box[3] = {(cuuint32_t)(kSlabBytes / esize), (cuuint32_t)box_rows, 1};
  return make_map(base, esize, 3, dims, strides, box);
}

CUtensorMap map_rows2d(const void* base, int esize, long long K, long long rows, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * esize};
  cuuint32_t box[2] = {(cuuint32_t)(kSlabBytes / esize), (cuuint32_t)box_rows};
  return make_map(base, esize, 2, dims, strides, box);
}

// Epilogue output maps.  fp32: 32-feature boxes; bf16 activations out
// (TcArgs::out_bf16): 64-feature boxes -- the same 128-byte staging rows.
// Rows [pix][K] with the split partials as the third dimension:
CUtensorMap out_map_rows(const void* base, bool ob, int K, long long pix, int splits) {
  const int es = ob ? 2 : 4;
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)pix, (cuuint64_t)splits};
  cuuint64_t strides[2] = {(cuuint64_t)K * es, (cuuint64_t)(pix * K * es)};
  cuuint32_t box[3] = {(cuuint32_t)(ob ? 64 : 32), (cuuint32_t)kRows, 1};
  return make_map(base, es, 3, dims, strides, box);
}
// The NHWC output plane, box {32 | 64 features, bw, bh, 1}:
CUtensorMap out_map_nhwc(const void* base, bool ob, const ConvGeom& g, int bw, int bh) {
  const int es = ob ? 2 : 4;
  cuuint64_t dims[4] = {(cuuint64_t)g.K, (cuuint64_t)g.OW, (cuuint64_t)g.OH, (cuuint64_t)g.N};
  cuuint64_t strides[3] = {(cuuint64_t)g.K * es, (cuuint64_t)g.OW * g.K * es,
                           (cuuint64_t)g.OH * g.OW * g.K * es};
  cuuint32_t box[4] = {(cuuint32_t)(ob ? 64 : 32), (cuuint32_t)bw, (cuuint32_t)bh, 1};
  return make_map(base, es, 4, dims, strides, box);
}

// NHWC activations, box {slab channels, Wb, Hb, 1}.
// With stride s > 1 the box traverses W and H with element stride s: it
// spans s*wb x s*hb input pixels and lands the wb x hb pixels a stride-s
// window visits (one tap), densely, in shared memory.
CUtensorMap map_nhwc(const void* base, int esize, const ConvGeom& g, int wb, int hb,
                     int stride = 1, int nb = 1) {
  cuuint64_t dims[4] = {(cuuint64_t)g.C, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
  cuuint64_t strides[3] = {(cuuint64_t)g.C * esize, (cuuint64_t)g.W * g.C * esize,
                           (cuuint64_t)g.H * g.W * g.C * esize};
  cuuint32_t box[4] = {(cuuint32_t)(kSlabBytes / esize), (cuuint32_t)(wb * stride),
                       (cuuint32_t)(hb * stride), (cuuint32_t)nb};
  const cuuint32_t trav[4] = {1, (cuuint32_t)stride, (cuuint32_t)stride, 1};
  return make_map(base, esize, 4, dims, strides, box, stride > 1 ? trav : nullptr);
}

// NHWC activations in im2col mode: each load is `pixels` consecutive output
// pixels x one slab of channels.  The bounding box of filter origins runs
// from -pad (lower corner) to the last origin a window visits (upper corner
// = pad_after - (R-1)); the traversal steps by the stride in W and H and
// wraps across rows and images, so a tile is any run of output pixels in
// NHW order -- no per-image box padding.  Order of the corner arrays: W, H.
CUtensorMap map_nhwc_im2col(const void* base, int esize, const ConvGeom& g, int pixels) {
  const cuuint32_t chans = (cuuint32_t)(kSlabBytes / esize);
  const CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B;
  cuuint64_t dims[4] = {(cuuint64_t)g.C, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
  cuuint64_t strides[3] = {(cuuint64_t)g.C * esize, (cuuint64_t)g.W * g.C * esize,
                           (cuuint64_t)g.H * g.W * g.C * esize};
  const int pad_b = (g.OH - 1) * g.stride + g.R - g.H - g.pad_t;
  const int pad_r = (g.OW - 1) * g.stride + g.S - g.W - g.pad_l;
  const int lower[2] = {-g.pad_l, -g.pad_t};
  const int upper[2] = {pad_r - (g.S - 1), pad_b - (g.R - 1)};
  const cuuint32_t trav[4] = {1, (cuuint32_t)g.stride, (cuuint32_t)g.stride, 1};
  MapKey key;
  std::memset(&key, 0, sizeof key);
  key.base = base;
  key.kind = 1;
  key.esize = esize;
  key.rank = 4;
  for (int i = 0; i < 4; ++i) {
    key.dims[i] = dims[i];
    key.trav[i] = trav[i];
    if (i < 3) key.strides[i] = strides[i];
  }
  key.lower[0] = lower[0];
  key.lower[1] = lower[1];
  key.upper[0] = upper[0];
  key.upper[1] = upper[1];
  key.chans = chans;
  key.pixels = (cuuint32_t)pixels;
  key.swz = (int)swz;
  if (const CUtensorMap* hit = map_memo().find(key)) return *hit;
  CUtensorMap m;
  const CUresult r = encode_im2col_fn()(
      &m, esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
      const_cast<void*>(base), dims, strides, lower, upper, chans,
      (cuuint32_t)pixels, trav, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    fail(TK_ERR_CUDA, "cuTensorMapEncodeIm2col failed (" + std::to_string(r) + ")");
  // Same driver workaround as CUTLASS's im2col descriptors (drivers <= 13.1,
  // tensors under 128 KiB): clear bit 21 of the second descriptor word.
  static const int drv = [] {
    int v = 0;
    return cudaDriverGetVersion(&v) == cudaSuccess ? v : 0;
  }();
  if (drv > 0 && drv <= 13010 && (size_t)g.N * g.H * g.W * g.C * esize < 131072)
    reinterpret_cast<uint64_t*>(&m)[1] &= ~(1ull << 21);
  map_memo().put(key, m);
  return m;
}

int sm_count() {
  static int n = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  });
  return n;
}

bool pdl_enabled() { return experiments().pdl; }

// Launch of a helper kernel (reductions, conversions) as a programmatic
// dependent of the previous kernel in the stream: its CTAs may be scheduled
// while that kernel drains (they block in griddep_wait before touching
// memory), and they release their own dependents at once, so the next
// tensor-core kernel's prologue overlaps them too.
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kern)(KArgs...), unsigned grid, unsigned block, cudaStream_t st,
                Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  TKB_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
  note_launch();
}

// Sum the tail pieces of each tail tile in piece order into the output.
// Block = (tail tile r, CTA rank, 8 columns); thread = one column x 4 rows
// (float4 along the column-major partial).  pixN: row = output feature,
// column = pixel of the tile's box (features are contiguous in NHWC: float4
// stores); plain: row = M index, column = N index.
template <int MODE, int CG, bool OB>
__global__ void __launch_bounds__(256) tail_reduce_kernel(TcArgs p) {
  ptx::griddep_wait();
  ptx::griddep_launch_dependents();
  const int col_blocks = (p.BN + 7) / 8;
  const int r = blockIdx.x / (CG * col_blocks);
  const int rem = blockIdx.x - r * CG * col_blocks;
  const int rank = rem / col_blocks;
  const int col = (rem - rank * col_blocks) * 8 + threadIdx.x / 32;
  const int row = (threadIdx.x % 32) * 4;
  // The tile's piece count and decode, once per block (64-bit owner
  // arithmetic per thread made this pass 15 us on VGG conv5).
  __shared__ int s_pieces;
  __shared__ Unit s_u;
  if (threadIdx.x == 0) {
    const long long nk = p.num_kb;
    s_pieces = tail_owner(p, (r + 1) * nk - 1) - tail_owner(p, r * nk) + 1;
    s_u = decode_tile(p, p.tail_start + r);
  }
  __syncthreads();
  const int pieces = s_pieces;
  const Unit u = s_u;
  if (pieces < 2 || col >= p.BN) return;  // stored directly by its only segment
  const long long tile = (long long)p.BN * 128;
  const float* src =
      p.tail_part + ((long long)r * p.tail_q * CG + rank) * tile + (long long)col * 128 + row;
  float4 a = __ldcs(reinterpret_cast<const float4*>(src));
  for (int q = 1; q < pieces; ++q) {
    const float4 b = __ldcs(reinterpret_cast<const float4*>(src + (long long)q * CG * tile));
    a.x += b.x;
    a.y += b.y;
    a.z += b.z;
    a.w += b.w;
  }
  const int m = u.m_blk * kRows * CG + rank * kRows + row;
  if constexpr (MODE == kConvPixN) {
    const PixTile pt = pix_tile(p, u.n_blk);
    int oh, ow, img;
    if (p.flat) {
      const int r = u.n_blk * p.tileH + col / p.Wb;
      img = r / p.OH;
      oh = r - img * p.OH;
      ow = col - (col / p.Wb) * p.Wb;
    } else {
      const int per = p.Wb * p.tileH;
      const int ii = col / per, cc = col - (col / per) * per;
      oh = pt.oh0 + cc / p.Wb;
      ow = pt.ow0 + cc - (cc / p.Wb) * p.Wb;
      img = pt.img + ii;
    }
    if (oh >= p.OH || ow >= p.OW || img >= p.Nimg) return;
    if constexpr (OB) {
      __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(p.d) +
                         (((long long)img * p.OH + oh) * p.OW + ow) * p.Kout + m;
      const float v[4] = {a.x, a.y, a.z, a.w};
      for (int i = 0; i < 4; ++i)
        if (m + i < p.Kout) o[i] = __float2bfloat16_rn(v[i]);
      return;
    }
    float* o = p.d + (((long long)img * p.OH + oh) * p.OW + ow) * p.Kout + m;
    if (m + 3 < p.Kout && (p.Kout & 3) == 0) {
      *reinterpret_cast<float4*>(o) = a;
    } else {
      const float v[4] = {a.x, a.y, a.z, a.w};
      for (int i = 0; i < 4; ++i)
        if (m + i < p.Kout) o[i] = v[i];
    }
  } else {
    const int n = u.n_blk * p.BN + col;
    if (n >= p.N) return;
    const float v[4] = {a.x, a.y, a.z, a.w};
    for (int i = 0; i < 4; ++i)
      if (m + i < p.M) {
        const long long off =
            (long long)u.z * p.d_batch + (long long)(m + i) * p.d_sm + (long long)n * p.d_sn;
        if constexpr (OB) reinterpret_cast<__nv_bfloat16*>(p.d)[off] = __float2bfloat16_rn(p.alpha * v[i]);
        else p.d[off] = p.alpha * v[i];
      }
  }
}

inline long long total_tiles_of(const TcArgs& p) { return (long long)p.num_m * p.num_n * p.batch; }

// Sustained dense TF32 tensor-core rate per SM and clock the cost models use:
// the measured 827 TF/s (1/2 of the bf16 burst in MEASURED_PEAKS.json) over
// 148 SMs at 1.9 GHz (the nominal 1.1 PF would be 3782).
constexpr double kTcFlopPerClk = 2941.0;

struct TailPlan {
  int start = 0, q = 0, kb = 0, P = 0;  // q: max pieces per tile, kb: segments per pair
  long long W = 0;
  size_t bytes = 0;
  double cost_us = 0;                   // modelled time of the whole launch with this tail
};

// Per-slab time of an SM pair (us): max(MMA, operand feed) -- the constants
// of choose_splits.
// A slab is 128 bytes of K (32 tf32 / 64 bf16: the same tensor-core time);
// each SM of the group does 2 * (bm / cg) * bn * 32 tf32-equivalent flops
// and stages (bm + bn) / cg operand rows of 128 bytes at ~70 B/clk.
inline double slab_time_us(int cg, int bn) {
  const int bm = kRows * cg;
  const double mma_clk = 64.0 * (double)bm * bn / (cg * kTcFlopPerClk);
  const double feed_clk = (double)(bm + bn) / cg * 128 / 70.0;
  return std::max(mma_clk, feed_clk) / 1900.0;
}

// Modelled time (us) of `tiles` whole tiles of num_kb slabs in waves.
inline double waves_cost_us(long long tiles, int num_kb, int cg, int bn) {
  const long long pairs = sm_count() / cg;
  return (double)((tiles + pairs - 1) / pairs) * (num_kb * slab_time_us(cg, bn) + 1.0);
}

// Wave-quantisation tail, stream-K style: with T tiles on P SM pairs the
// last T % P tiles (all of them when T < P) would run as a partial wave as
// long as a full one; instead their slab-steps are dealt evenly to all P
// pairs (see TcArgs::tail_*).  Taken when the cost model (per-slab max(MMA,
// operand feed), ~1 us per unit, the reduction pass over the partial tiles
// at ~4 TB/s + launch) says it pays.
TailPlan plan_tail(long long tiles, int num_kb, int cg, int bn) {
  TailPlan t;
  const bool off = !experiments().tail;
  const long long pairs = sm_count() / cg;
  const long long rem = tiles % pairs, full = tiles / pairs;
  const double base = waves_cost_us(tiles, num_kb, cg, bn);
  t.cost_us = base;
  if (off || tc_knobs().split == 1 || rem == 0 || num_kb < 4) return t;
  const long long W = rem * (long long)num_kb;
  if (W < pairs) return t;  // every pair needs a slab-step (no empty ranges)
  const double slab = slab_time_us(cg, bn);
  const double tile_bytes = (double)kRows * cg * bn * 4;
  const long long per = (W + pairs - 1) / pairs;
  const int segs = (int)((per + num_kb - 1) / num_kb) + 1;
  const int q = (int)((num_kb * pairs + W - 1) / W) + 1;  // pieces per tile, upper bound
  // pieces written: ~ one per pair plus one per tile; read once, tiles written once
  const double red_bytes = (double)(pairs + rem) * tile_bytes * 2 + (double)rem * tile_bytes;
  const double cost = (double)full * (num_kb * slab + 1.0) + per * slab + 1.0 * segs + 2.0 +
                      red_bytes / (experiments().red_gbs * 1e3);
  if (cost >= base * 0.97 && !experiments().tail_force) return t;  // a win beyond the model's noise
  t.start = (int)(tiles - rem);
  t.q = std::max(q, 2);
  t.kb = segs;
  t.P = (int)pairs;
  t.W = W;
  t.bytes = (size_t)rem * t.q * cg * bn * 128 * 4;
  t.cost_us = cost;
  return t;
}

void apply_tail(TcArgs& p, const TailPlan& t, float* buf) {
  if (t.q < 2) return;
  p.tail_start = t.start;
  p.tail_q = t.q;
  p.tail_kb = t.kb;
  p.tail_P = t.P;
  p.tail_W = t.W;
  p.tail_part = buf;
}

template <int MODE, int CG, bool TF32, bool OB = false>
void run_kernel(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& md, TcArgs p,
                int stages_req, cudaStream_t st) {
  const int b_bytes_h = (p.BN / CG) * kSlabBytes;
  const int stage_bytes = halo_like<MODE>()
                              ? p.halo_bytes + (p.resident ? 0 : p.taps) * b_bytes_h
                              : kRows * kSlabBytes + b_bytes_h;
  const int fres_bytes = (halo_like<MODE>() && p.resident) ? p.taps * p.cchunks * b_bytes_h : 0;
  const int ktab_bytes0 = MODE == kConvGather ? p.num_kb * 32 * 8 : 0;
  // Tuning experiments: TK_TC_STAGES caps the ring, TK_TC_EPI=1 forces one
  // staging buffer.
  if (tc_knobs().stages > 0) stages_req = tc_knobs().stages;
  const Experiments& xp = experiments();
  if (xp.tc_stages > 0) stages_req = xp.tc_stages;
  if (xp.tc_epi > 0) p.epi_bufs = std::min(p.epi_bufs, xp.tc_epi);
  // Chunk-ring staging (32 KiB) for tiles wider than one chunk.
  p.epi_ring = (p.store_tma && xp.epi_ring && (p.BN > 32 || MODE == kConvHaloNarrow)) ? 1 : 0;
  p.epi_slots = 2;
  p.epi_groups = 1;
  // Double-buffered TMA-store staging when it leaves room for >= 3 stages.
  if (p.store_tma && p.epi_bufs > 1 &&
      232448 - 2048 - ktab_bytes0 - 2 * ((p.BN + 31) / 32) * kRows * kSlabBytes < 3 * stage_bytes)
    p.epi_bufs = 1;
  const int ktab_bytes = MODE == kConvGather ? p.num_kb * 32 * 8 : 0;
  constexpr int kChunkBytes = kRows * kSlabBytes;
  if (p.epi_ring) {
    // Batch size: whole tiles double-buffered (two syncs per tile) when the
    // operand ring still gets every stage a unit can use, else smaller
    // batches down to single chunks.
    const int nchunks = (p.BN + 31) / 32;
    const int room = 232448 - 1024 - 1024 - ktab_bytes - fres_bytes;
    const int kb_unit = std::max(1, std::min(p.num_kb, p.splits > 1 ? p.kb_per : p.num_kb));
    const int want = std::min(kMaxStages, std::max(3, kb_unit + 1));
    int bs = (room - want * stage_bytes) / (2 * kChunkBytes);
    bs = std::max(1, std::min(nchunks, bs));
    if (xp.epi_ring_n > 0) bs = std::max(1, std::min(nchunks, xp.epi_ring_n));
    p.epi_ring = bs;
    // Slots: as many as the room left after the wanted operand stages
    // holds (2..8); short-K layers then keep several tiles of stores in flight.
    // Slots beyond two only for epilogue-bound tiles (at most two slabs of
    // MMA work per tile: the narrow first layers, short-K 1x1 layers):
    // measured, VGG conv1_1 TF32 214 -> 180 us (L2-cold), while MMA-heavy
    // tiles lose operand stages (conv1_2 208 -> 273 us with 8 slots).
    const int work_slabs = MODE == kConvHaloNarrow ? (p.narrow_taps + 7) / 8
                           : MODE == kConvHalo     ? p.taps * p.cchunks
                                                   : kb_unit;
    // Epilogue-bound tiles also get the second epilogue warpgroup (tiles
    // alternate between the groups, each with its own staging slots).
    // (narrow halo: <= 25 MMAs of K = 8 per tile -- VGG conv1_1 178 -> 121
    // us, ResNet stem 68 -> 54 us with the second group, L2-warm A/B)
    (void)work_slabs;
    const bool epi_bound = MODE == kConvHaloNarrow;  // (the only multi-slot / two-group epilogue)
    p.epi_groups = (epi_bound && epi_groups_of<MODE>() > 1) ? 2 : 1;
    if (xp.epi_groups == 1 || xp.epi_groups == 2)
      p.epi_groups = std::min(xp.epi_groups, epi_groups_of<MODE>());
    if (p.epi_groups == 2 && room - 2 * stage_bytes < 2 * 2 * bs * kChunkBytes) p.epi_groups = 1;
    const int per_slot = p.epi_groups * bs * kChunkBytes;
    p.epi_slots = epi_bound ? std::max(2, std::min(8, (room - want * stage_bytes) / per_slot)) : 2;
    if (xp.epi_slots > 0)  // (capped at what leaves two operand stages)
      p.epi_slots = std::max(2, std::min({8, xp.epi_slots, (room - 2 * stage_bytes) / per_slot}));
  }
  const int epi_bytes = !p.store_tma ? 0
                       : p.epi_ring ? p.epi_groups * p.epi_slots * p.epi_ring * kChunkBytes
                                    : p.epi_bufs * ((p.BN + 31) / 32) * kChunkBytes;
  p.epi_bytes = epi_bytes;
  const int budget = 232448 - 1024 - 1024 - epi_bytes - ktab_bytes - fres_bytes;
  int stages = budget / stage_bytes;
  if (stages > kMaxStages) stages = kMaxStages;
  if (stages_req > 0 && stages_req < stages) stages = stages_req;
  if (stages < 2) fail(TK_ERR_CAPABILITY, "tc_gemm: tile too large for shared memory");
  if (stage_bytes % 1024 != 0 || fres_bytes % 1024 != 0)  // swizzle-atom alignment of every buffer
    fail(TK_ERR_CAPABILITY, "tc_gemm: stage of " + std::to_string(stage_bytes) +
                                " bytes is not a multiple of 1024");
  p.stages = stages;
  const size_t smem =
      1024 + (size_t)stages * stage_bytes + fres_bytes + 1024 + epi_bytes + ktab_bytes;
  if (OB && !p.store_tma && MODE != kConvPixN)
    fail(TK_ERR_CAPABILITY, "tc_gemm: bf16 output needs the TMA-store epilogue");
  if (OB && p.BN % 64 != 0 && MODE != kConvPixN)
    fail(TK_ERR_CAPABILITY, "tc_gemm: bf16 output needs tiles of 64-feature multiples");
  auto fn = tc_gemm_kernel<MODE, CG, TF32, OB>;
  func_smem((const void*)fn, smem);
  {
    const int forced = xp.tc_acc;
    p.acc_slots = p.BN <= 64 ? 8 : (p.BN <= 128 ? 4 : 2);
    if (forced == 2 || forced == 4 || forced == 8) p.acc_slots = std::min(p.acc_slots, forced);
    p.acc_cols = 2 * kAccCols / p.acc_slots;
    p.acc_shift = p.acc_slots == 8 ? 3 : (p.acc_slots == 4 ? 2 : 1);
  }
  if (p.splits < 1 || (!plain_like<MODE>() && MODE != kConvPixN)) {
    p.splits = 1;
    p.kb_per = p.num_kb;
  }
  {
    const int raster = xp.raster;
    const long long units_all = (long long)p.num_m * p.num_n * p.batch * p.splits;
    // Grouping only pays once tiles queue up behind the resident wave.
    p.raster = ((plain_like<MODE>() || MODE == kConvPixN) && units_all > 2LL * (sm_count() / CG))
                   ? raster
                   : 0;
  }
  if (p.tail_q > 1 && (p.splits > 1 || (!plain_like<MODE>() && MODE != kConvPixN))) p.tail_q = 0;
  p.fd_per = make_fdiv(p.num_m * p.num_n);
  p.fd_span = make_fdiv(p.raster * p.num_n);
  p.fd_raster = make_fdiv(p.raster);
  p.fd_num_m = make_fdiv(p.num_m);
  p.fd_num_n = make_fdiv(p.num_n);
  p.fd_batch = make_fdiv(p.batch);
  p.fd_per_img = make_fdiv(p.tiles_w * p.tiles_h);
  p.fd_tiles_w = make_fdiv(p.tiles_w);
  const long long total = p.tail_q > 1 ? (long long)p.tail_start + (long long)p.tail_kb * p.tail_P
                                       : (long long)p.num_m * p.num_n * p.batch * p.splits;
  const int units = sm_count() / CG;
  int used = (int)(total < units ? total : units);
  // Halo mode with a resident filter: every CTA must keep one feature block.
  if (halo_like<MODE>() && p.resident) used -= used % p.num_n;
  const int grid = used * CG;
  if (grid <= 0) return;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(threads_of<MODE>());
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = xp.pdl ? 2 : 1;
  unsigned long long* trace = nullptr;
  if (xp.trace) {
    TKB_CUDA(cudaMalloc(&trace, (size_t)grid * kTraceEvents * 8));
    TKB_CUDA(cudaMemset(trace, 0, (size_t)grid * kTraceEvents * 8));
    p.trace = trace;
  }
  TKB_CUDA(cudaLaunchKernelEx(&cfg, fn, ma, mb, md, p));
  note_launch();
  if constexpr (plain_like<MODE>() || MODE == kConvPixN) {
    if (p.tail_q > 1) {
      const long long rem = total_tiles_of(p) - p.tail_start;
      const long long blocks = rem * CG * ((p.BN + 7) / 8);
      launch_pdl(tail_reduce_kernel<MODE, CG, OB>, (unsigned)blocks, 256, st, p);
    }
  }
  if (trace) {
    std::vector<unsigned long long> h((size_t)grid * kTraceEvents);
    TKB_CUDA(cudaStreamSynchronize(st));
    TKB_CUDA(cudaMemcpy(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost));
    cudaFree(trace);
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < grid; ++b) t0 = std::min(t0, h[(size_t)b * kTraceEvents]);
    static const char* names[kTraceEvents] = {
        "entry", "setup", "slab0", "slabN", "acc0", "acc1", "stored", "exit", "drained", "issued",
        "u8:mma_acc_free", "u8:mma_slab_in", "u8:mma_commit", "u8:epi_acc_in", "u8:epi_drained",
        "u8:epi_issued", "u8:gather_loaded", "u8:gather_arrived", "u8:epi_tmem_fence",
        "u8:epi_proxy_fence", "u8:epi_released"};
    std::fprintf(stderr, "tc trace MODE=%d CG=%d grid=%d units=%lld stages=%d BN=%d (us from first entry: min/med/max)\n",
                 MODE, CG, grid, total, stages, p.BN);
    for (int e = 0; e < kTraceEvents; ++e) {
      std::vector<double> v;
      for (int b = 0; b < grid; ++b) {
        const unsigned long long x = h[(size_t)b * kTraceEvents + e];
        if (x) v.push_back((double)(x - t0) / 1e3);
      }
      if (v.empty()) continue;
      std::sort(v.begin(), v.end());
      std::fprintf(stderr, "  %-7s n=%3zu  %8.2f %8.2f %8.2f\n", names[e], v.size(), v.front(),
                   v[v.size() / 2], v.back());
    }
  }
}

template <int MODE>
void dispatch(const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& md,
              const TcArgs& p, int cg, bool tf32, cudaStream_t st) {
  if constexpr (MODE != kConvGather) {
    if (p.out_bf16) {  // bf16 activations out (BF16 operands only)
      if (tf32) fail(TK_ERR_CAPABILITY, "tc_gemm: bf16 output needs BF16 precision");
      if (cg == 2) run_kernel<MODE, 2, false, true>(ma, mb, md, p, 0, st);
      else run_kernel<MODE, 1, false, true>(ma, mb, md, p, 0, st);
      return;
    }
  }
  if (cg == 2) {
    if (tf32) run_kernel<MODE, 2, true>(ma, mb, md, p, 0, st);
    else run_kernel<MODE, 2, false>(ma, mb, md, p, 0, st);
  } else {
    if (tf32) run_kernel<MODE, 1, true>(ma, mb, md, p, 0, st);
    else run_kernel<MODE, 1, false>(ma, mb, md, p, 0, st);
  }
}

void require_tc(int precision) {
  if (precision != TK_PREC_TF32 && precision != TK_PREC_BF16 && precision != TK_PREC_3XTF32)
    fail(TK_ERR_CAPABILITY, "tensor-core path: precision must be TF32, BF16 or 3xTF32");
}

// ---- 3xTF32 (split precision) ------------------------------------------------
// x = hi + lo with hi = x truncated to TF32 (what the tensor core reads from
// an fp32 operand) and lo = x - hi (exact in fp32).  A product sum then runs
// as one TF32 contraction over a tripled depth:
//   sum_k a_k b_k ~= sum_k (a_hi b_hi + a_hi b_lo + a_lo b_hi)
// by concatenating [a, a, a_lo] against [b_hi, b_lo, b_hi] along K; the
// dropped a_lo b_lo term is below 2^-22 relative.
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xffffe000u);
}

// rows x [kp] K-major fp32 -> rows x [3 kp]: pattern 0 = (x, x, lo), 1 = (hi, lo, hi).
__global__ void __launch_bounds__(256) split3_rows_kernel(const float* __restrict__ src,
                                                          long long rows, long long kp,
                                                          float* __restrict__ dst, int pattern) {
  const long long n = rows * kp;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / kp, k = i - r * kp;
    const float x = src[i], hi = tf32_hi(x), lo = x - hi;
    float* d = dst + r * 3 * kp + k;
    if (pattern == 0) {
      d[0] = x;
      d[kp] = x;
      d[2 * kp] = lo;
    } else {
      d[0] = hi;
      d[kp] = lo;
      d[2 * kp] = hi;
    }
  }
}

void split3_rows(const float* src, long long rows, long long kp, float* dst, int pattern,
                 cudaStream_t st) {
  const long long n = rows * kp;
  const int blocks = (int)std::min<long long>((n + 255) / 256, (long long)sm_count() * 16);
  split3_rows_kernel<<<blocks, 256, 0, st>>>(src, rows, kp, dst, pattern);
  note_launch();
  TKB_CUDA(cudaGetLastError());
}

// NHWC [P][C] -> [P][3C] = [x | x | lo] (activations; the tensor core
// truncates the first two copies to hi).
__global__ void __launch_bounds__(256) split3_channels_kernel(const float* __restrict__ src,
                                                              long long pix, int C,
                                                              float* __restrict__ dst) {
  const long long n = pix * C;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long q = i / C;
    const int c = (int)(i - q * C);
    const float x = src[i];
    float* d = dst + q * 3 * C + c;
    d[0] = x;
    d[C] = x;
    d[2 * C] = x - tf32_hi(x);
  }
}

// HWCK [R*S][C][K] -> [R*S][3C][K] = [hi | lo | hi] along C.
__global__ void __launch_bounds__(256) split3_filter_kernel(const float* __restrict__ src,
                                                            long long taps, int C, int K,
                                                            float* __restrict__ dst) {
  const long long n = taps * C * K;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long t = i / ((long long)C * K);
    const long long rem = i - t * C * K;  // c*K + k
    const float x = src[i], hi = tf32_hi(x);
    float* d = dst + t * 3 * C * K + rem;
    d[0] = hi;
    d[(long long)C * K] = x - hi;
    d[2LL * C * K] = hi;
  }
}

// TMA tensor maps and the vectorised pack/convert kernels address global
// memory in 16-byte units.
void require_aligned(const void* p, const char* what) {
  if (p && (reinterpret_cast<uintptr_t>(p) & 15) != 0)
    fail(TK_ERR_CAPABILITY, std::string("tensor-core path: ") + what +
                                " must be 16-byte aligned (device allocations are)");
}

// ---- packing / conversion kernels -------------------------------------------

__device__ __forceinline__ float round_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

template <typename T>
__device__ __forceinline__ T cvt_out(float v, int tf32_round);
template <>
__device__ __forceinline__ float cvt_out<float>(float v, int tf32_round) {
  return tf32_round ? round_tf32(v) : v;
}
template <>
__device__ __forceinline__ __nv_bfloat16 cvt_out<__nv_bfloat16>(float v, int) {
  return __float2bfloat16_rn(v);
}

// Pack sources: fp32 operands, or bf16 ones (bf16 operands in HBM,
// tk_exec_options.io) -- read as float, 4 consecutive elements at a time.
__device__ __forceinline__ float src_f(const float* p) { return *p; }
__device__ __forceinline__ float src_f(const __nv_bfloat16* p) { return __bfloat162float(*p); }
__device__ __forceinline__ float4 src_f4(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ float4 src_f4(const __nv_bfloat16* p) {
  const uint2 u = __ldcs(reinterpret_cast<const uint2*>(p));
  const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(&u.x);
  const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&u.y);
  return make_float4(__low2float(lo), __high2float(lo), __low2float(hi), __high2float(hi));
}

// dst[r][kk] (row length kp, zero for kk >= k) = src[r*rs + kk*ks].
template <typename T, typename S = float>
__global__ void __launch_bounds__(256) pack_kmajor_kernel(const S* __restrict__ src,
                                                          long long rs, long long ks, long long rows,
                                                          long long k, long long kp,
                                                          T* __restrict__ dst, int tf32_round) {
  __shared__ float tile[32][33];
  const long long r0 = (long long)blockIdx.y * 32, k0 = (long long)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  if (ks == 1) {
    for (int i = ty; i < 32; i += 8) {
      const long long r = r0 + i, kk = k0 + tx;
      tile[i][tx] = (r < rows && kk < k) ? src_f(src + r * rs + kk) : 0.0f;
    }
  } else {
    for (int i = ty; i < 32; i += 8) {
      const long long r = r0 + tx, kk = k0 + i;
      tile[tx][i] = (r < rows && kk < k) ? src_f(src + r * rs + kk * ks) : 0.0f;
    }
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const long long r = r0 + i, kk = k0 + tx;
    if (r < rows && kk < kp) dst[r * kp + kk] = cvt_out<T>(tile[i][tx], tf32_round);
  }
}

// Row-contiguous source (ks == 1): dst[r][kk] = src[r*rs + kk], 4 elements
// per thread, vector loads and stores, zero tail up to kp.
template <typename T, typename S = float>
__global__ void __launch_bounds__(256) pack_rows_kernel(const S* __restrict__ src, long long rs,
                                                        long long rows, long long k, long long kp,
                                                        T* __restrict__ dst, int tf32_round) {
  const long long per_row = kp / 4;
  const long long total = rows * per_row;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / per_row, kk = (i - r * per_row) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (kk + 3 < k) v = src_f4(src + r * rs + kk);
    else {
      if (kk < k) v.x = src_f(src + r * rs + kk);
      if (kk + 1 < k) v.y = src_f(src + r * rs + kk + 1);
      if (kk + 2 < k) v.z = src_f(src + r * rs + kk + 2);
    }
    T* d = dst + r * kp + kk;
    if constexpr (sizeof(T) == 4) {
      *reinterpret_cast<float4*>(d) = make_float4(cvt_out<float>(v.x, tf32_round), cvt_out<float>(v.y, tf32_round),
                                                  cvt_out<float>(v.z, tf32_round), cvt_out<float>(v.w, tf32_round));
    } else {
      __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&lo);
      u.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(d) = u;
    }
  }
}

// dst[r][kk] = src[r + kk*ks] for a 64-row x 64-k tile per block: float4
// loads along r, float4 (fp32) / 8-byte (bf16) stores along kk.
template <typename T, typename S = float>
__global__ void __launch_bounds__(256) pack_transpose_kernel(const S* __restrict__ src,
                                                             long long ks, long long rows,
                                                             long long k, long long kp,
                                                             T* __restrict__ dst, int tf32_round) {
  __shared__ float tile[64][65];  // [kk][r]
  const long long r0 = (long long)blockIdx.y * 64, k0 = (long long)blockIdx.x * 64;
  const int t = threadIdx.x;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int kk = t / 16 + 16 * j, r4 = (t % 16) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (k0 + kk < k && r0 + r4 < rows)  // rows % 4 == 0: whole float4 in range
      v = src_f4(src + (k0 + kk) * ks + r0 + r4);
    tile[kk][r4] = v.x;
    tile[kk][r4 + 1] = v.y;
    tile[kk][r4 + 2] = v.z;
    tile[kk][r4 + 3] = v.w;
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int r = t / 16 + 16 * j, kk4 = (t % 16) * 4;
    if (r0 + r >= rows || k0 + kk4 >= kp) continue;
    const float a = tile[kk4][r], b = tile[kk4 + 1][r], c = tile[kk4 + 2][r], d = tile[kk4 + 3][r];
    T* o = dst + (r0 + r) * kp + k0 + kk4;
    if constexpr (sizeof(T) == 4) {
      *reinterpret_cast<float4*>(o) = make_float4(cvt_out<float>(a, tf32_round), cvt_out<float>(b, tf32_round),
                                                  cvt_out<float>(c, tf32_round), cvt_out<float>(d, tf32_round));
    } else {
      __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&lo);
      u.y = *reinterpret_cast<uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(o) = u;
    }
  }
}

template <typename T, typename S = float>
void pack_kmajor(const S* src, long long rs, long long ks, long long rows, long long k,
                 long long kp, T* dst, bool tf32_round, cudaStream_t st) {
  // (vector paths: 4 source elements = 16 bytes fp32 / 8 bytes bf16)
  const bool src16 = (reinterpret_cast<uintptr_t>(src) & (4 * sizeof(S) - 1)) == 0;
  // Column-contiguous source (a column-major operand read along its rows):
  // 64 x 64 tiles transposed through shared memory with 16-byte accesses
  // on both sides.
  if (rs == 1 && ks % 4 == 0 && rows % 4 == 0 && kp % 4 == 0 && src16) {
    dim3 grid((unsigned)((kp + 63) / 64), (unsigned)((rows + 63) / 64));
    if (grid.y > 65535) fail(TK_ERR_CAPABILITY, "pack: too many rows");
    pack_transpose_kernel<T, S><<<grid, 256, 0, st>>>(src, ks, rows, k, kp, dst, tf32_round ? 1 : 0);
    note_launch();
    TKB_CUDA(cudaGetLastError());
    return;
  }
  if (ks == 1 && rs % 4 == 0 && kp % 4 == 0 && src16) {
    const long long n = rows * (kp / 4);
    const int blocks = (int)std::min<long long>((n + 255) / 256, (long long)sm_count() * 16);
    pack_rows_kernel<T, S><<<blocks, 256, 0, st>>>(src, rs, rows, k, kp, dst, tf32_round ? 1 : 0);
    note_launch();
    TKB_CUDA(cudaGetLastError());
    return;
  }
  dim3 grid((unsigned)((kp + 31) / 32), (unsigned)((rows + 31) / 32));
  if (grid.y > 65535) fail(TK_ERR_CAPABILITY, "pack: too many rows");
  pack_kmajor_kernel<T, S><<<grid, dim3(32, 8), 0, st>>>(src, rs, ks, rows, k, kp, dst, tf32_round);
  note_launch();
  TKB_CUDA(cudaGetLastError());
}

// HWCK filter [K][Kout] -> K-major [Kout][kp] (zero padded, TF32-rounded
// or converted to bf16) without shared memory: each thread moves a KV x 4
// block through registers, so the kernel can co-reside with a running
// tensor-core kernel (whose CTAs own the shared memory) when it is issued on
// a side stream.
template <typename T, int KV>
__global__ void __launch_bounds__(256) pack_filter_kernel(const float* __restrict__ src,
                                                          int K, int Kout, int kp,
                                                          T* __restrict__ dst, int tf32_round) {
  // Thread = KV consecutive K rows x 4 features: float4 reads along the
  // features (coalesced across the warp), and per feature KV contiguous
  // packed elements written at once (KV = 8: whole 32-byte sectors for fp32,
  // no partial-sector writes).
  const int f4n = (Kout + 3) / 4, kvn = kp / KV;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)f4n * kvn) return;
  const int f0 = (int)(idx % f4n) * 4, k0 = (int)(idx / f4n) * KV;
  float v[KV][4];  // v[k][f]
#pragma unroll
  for (int i = 0; i < KV; ++i) {
    const int k = k0 + i;
    if (k < K && f0 + 3 < Kout && (Kout & 3) == 0) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(src + (long long)k * Kout + f0));
      v[i][0] = x.x;
      v[i][1] = x.y;
      v[i][2] = x.z;
      v[i][3] = x.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j)
        v[i][j] = (k < K && f0 + j < Kout) ? __ldg(src + (long long)k * Kout + f0 + j) : 0.0f;
    }
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if (f0 + j >= Kout) break;
    T* d = dst + (long long)(f0 + j) * kp + k0;
#pragma unroll
    for (int h = 0; h < KV; h += 4) {
      if constexpr (sizeof(T) == 4) {
        *reinterpret_cast<float4*>(d + h) = make_float4(
            cvt_out<float>(v[h][j], tf32_round), cvt_out<float>(v[h + 1][j], tf32_round),
            cvt_out<float>(v[h + 2][j], tf32_round), cvt_out<float>(v[h + 3][j], tf32_round));
      } else {
        __nv_bfloat162 lo = __floats2bfloat162_rn(v[h][j], v[h + 1][j]);
        __nv_bfloat162 hi = __floats2bfloat162_rn(v[h + 2][j], v[h + 3][j]);
        uint2 u;
        u.x = *reinterpret_cast<uint32_t*>(&lo);
        u.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(d + h) = u;
      }
    }
  }
}

template <typename T>
void pack_filter(const float* filt, int K, int Kout, int kp, T* dst, bool tf32_round,
                 cudaStream_t st) {
  if (kp % 4 != 0) fail(TK_ERR_CAPABILITY, "pack_filter: padded K must be a multiple of 4");
  const int kv = 4;  // (KV = 8 measured slower: 129 vs 100 us for the 13 VGG filters, cold)
  const long long n = (long long)((Kout + 3) / 4) * (kp / kv);
  const unsigned blocks = (unsigned)((n + 255) / 256);
  if (kv == 8)
    pack_filter_kernel<T, 8><<<blocks, 256, 0, st>>>(filt, K, Kout, kp, dst, tf32_round ? 1 : 0);
  else
    pack_filter_kernel<T, 4><<<blocks, 256, 0, st>>>(filt, K, Kout, kp, dst, tf32_round ? 1 : 0);
  note_launch();
  TKB_CUDA(cudaGetLastError());
}

// Narrow-pixel im2col operands (TcArgs::narrow_taps).  Filter: HWCK ->
// [Kout][kp] with k = tap * cp + c (zero for c >= C and for the padding
// taps past R*S), TF32-rounded or bf16.
// order = 1: taps row-major (im2col); order = s > 1: the narrow halo's
// (phase, row, column) order of a stride-s window (TcArgs::nphase).
template <typename T>
__global__ void __launch_bounds__(256) pack_filter_narrow_kernel(const float* __restrict__ src,
                                                                 int R, int S, int C, int Kout, int cp,
                                                                 int kp, int order,
                                                                 T* __restrict__ dst,
                                                                 int tf32_round) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)Kout * kp) return;
  const int f = (int)(i / kp), k = (int)(i - (long long)f * kp);
  const int q = k / cp, c = k - (k / cp) * cp;
  int tap = -1;  // window tap (x * S + y) of sorted position q
  if (order <= 1) {
    tap = q < R * S ? q : -1;
  } else {
    int n = 0;
    for (int ph = 0; ph < order * order && tap < 0; ++ph)
      for (int x = ph / order; x < R && tap < 0; x += order)
        for (int y = ph % order; y < S; y += order)
          if (n++ == q) {
            tap = x * S + y;
            break;
          }
  }
  const float v = (tap >= 0 && c < C) ? __ldg(src + ((long long)tap * C + c) * Kout + f) : 0.0f;
  dst[i] = cvt_out<T>(v, tf32_round);
}

// Narrow halo input: NHWC (C channels) -> phase-split [N][H][s][W2][cp]
// with xs[n][h][py][w2] = x[n][h][s*w2 + py - pad_l] (zero outside the row,
// channels past C zero): a stride-s window's column phase is contiguous and
// the left padding is baked in (tap y reads phase y % s at w2 = ow + y / s).
template <typename T, typename S>
__global__ void __launch_bounds__(256) pad_phase_kernel(const S* __restrict__ src, int N, int H,
                                                        int W, int C, int s, int W2, int pad_l,
                                                        int cp, T* __restrict__ dst) {
  ptx::griddep_wait();
  ptx::griddep_launch_dependents();
  // U destination rows (n, h, column phase py) per block
  // iteration, their W2 16-byte pixels across the threads: every thread has
  // the loads of several rows in flight before it stores (one row's 12-byte
  // pixel per thread left the pass latency-bound at ~4.4 TB/s).
  // Block b owns the contiguous rows [b rows / B, (b + 1) rows / B): one
  // resident wave, no half-empty second one.
  constexpr int U = 4;
  const int rows_all = N * H * s;
  const int rb = (int)((long long)blockIdx.x * rows_all / gridDim.x);
  const int rows = (int)((long long)(blockIdx.x + 1) * rows_all / gridDim.x);
  for (int r0 = rb; r0 < rows; r0 += U) {
    for (int w2 = threadIdx.x; w2 < W2; w2 += blockDim.x) {
      float v[U][8];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int r = r0 + u;
        const int py = s == 1 ? 0 : (r & 1);
        const long long nh = s == 1 ? r : (r >> 1);  // n * H + h
        const int col = s * w2 + py - pad_l;
        const bool in = r < rows && col >= 0 && col < W;
        const S* px = src + (in ? (nh * W + col) * C : 0);
        TKB_DCHECK(!in || nh < (long long)N * H);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          if constexpr (sizeof(S) == 4) v[u][c] = in && c < C && c < cp ? __ldg(px + c) : 0.0f;
          else v[u][c] = in && c < C && c < cp ? __bfloat162float(px[c]) : 0.0f;
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (r0 + u >= rows) break;
        const long long i = (long long)(r0 + u) * W2 + w2;
        if constexpr (sizeof(T) == 4) {
          reinterpret_cast<float4*>(dst)[i] = make_float4(v[u][0], v[u][1], v[u][2], v[u][3]);
        } else {
          uint4 q;
          __nv_bfloat162 b0 = __floats2bfloat162_rn(v[u][0], v[u][1]),
                         b1 = __floats2bfloat162_rn(v[u][2], v[u][3]),
                         b2 = __floats2bfloat162_rn(v[u][4], v[u][5]),
                         b3 = __floats2bfloat162_rn(v[u][6], v[u][7]);
          q.x = *reinterpret_cast<uint32_t*>(&b0);
          q.y = *reinterpret_cast<uint32_t*>(&b1);
          q.z = *reinterpret_cast<uint32_t*>(&b2);
          q.w = *reinterpret_cast<uint32_t*>(&b3);
          reinterpret_cast<uint4*>(dst)[i] = q;
        }
      }
    }
  }
}

// fp32 -> bf16, 8 elements per thread (n % 8 == 0 fast path).
__global__ void __launch_bounds__(256) to_bf16_kernel(const float4* __restrict__ src,
                                                      __nv_bfloat162* __restrict__ dst,
                                                      long long n4) {
  ptx::griddep_wait();
  ptx::griddep_launch_dependents();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    const float4 v = src[i];
    dst[2 * i] = __floats2bfloat162_rn(v.x, v.y);
    dst[2 * i + 1] = __floats2bfloat162_rn(v.z, v.w);
  }
}

void to_bf16(const float* src, __nv_bfloat16* dst, long long n, cudaStream_t st) {
  if (n % 4 != 0) fail(TK_ERR_CAPABILITY, "bf16 conversion needs a multiple of 4 elements");
  const long long n4 = n / 4;
  const int blocks = (int)std::min<long long>((n4 + 255) / 256, (long long)sm_count() * 8);
  launch_pdl(to_bf16_kernel, (unsigned)blocks, 256, st, reinterpret_cast<const float4*>(src),
             reinterpret_cast<__nv_bfloat162*>(dst), n4);
}

// out[i] = sum_s part[s*stride + i] in split order (deterministic), 4
// elements per thread (n % 4 == 0, 16-byte aligned rows).
template <bool OB>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const float4* __restrict__ part,
                                                            long long stride4, int splits,
                                                            void* __restrict__ out, long long n4) {
  ptx::griddep_wait();
  ptx::griddep_launch_dependents();
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    float4 v[kMaxSplits];  // every split's load in flight before the ordered sum (host: splits <= kMaxSplits)
#pragma unroll
    for (int s = 0; s < kMaxSplits; ++s)
      if (s < splits) v[s] = __ldcs(part + s * stride4 + i);
    float4 a = v[0];
#pragma unroll
    for (int s = 1; s < kMaxSplits; ++s) {
      if (s < splits) {
        a.x += v[s].x;
        a.y += v[s].y;
        a.z += v[s].z;
        a.w += v[s].w;
      }
    }
    if constexpr (OB) {  // bf16 activations out
      const __nv_bfloat162 lo = __floats2bfloat162_rn(a.x, a.y), hi = __floats2bfloat162_rn(a.z, a.w);
      uint2 u;
      u.x = *reinterpret_cast<const uint32_t*>(&lo);
      u.y = *reinterpret_cast<const uint32_t*>(&hi);
      reinterpret_cast<uint2*>(out)[i] = u;
    } else {
      reinterpret_cast<float4*>(out)[i] = a;
    }
  }
}

void splitk_reduce(const float* part, long long n, int splits, void* out, cudaStream_t st,
                   bool out_bf16 = false) {
  if (splits < 1 || splits > kMaxSplits)
    fail(TK_ERR_CAPABILITY, "split-K: " + std::to_string(splits) + " splits (at most " +
                                std::to_string(kMaxSplits) + ")");
  const long long n4 = n / 4;
  const int blocks = (int)std::min<long long>((n4 + 255) / 256, (long long)sm_count() * 8);
  if (out_bf16)
    launch_pdl(splitk_reduce_kernel<true>, (unsigned)blocks, 256, st,
               reinterpret_cast<const float4*>(part), n4, splits, out, n4);
  else
    launch_pdl(splitk_reduce_kernel<false>, (unsigned)blocks, 256, st,
               reinterpret_cast<const float4*>(part), n4, splits, out, n4);
}

// Pointwise (1x1) conv operand: the input pixels the strided window visits,
// compacted to [N*OH*OW][C] and converted to T (fp32 copy or bf16), 4
// channels per thread.  Stride 1 + bf16 is a plain conversion.
template <typename T, typename S>
__global__ void __launch_bounds__(256) pointwise_gather_kernel(const S* __restrict__ in, ConvGeom g,
                                                               FDiv fd_c4, T* __restrict__ out) {
  // One output row (n, oh) per block iteration, its OW x C/4 chunks across
  // the threads (one division per row, multiply-shift per chunk).
  ptx::griddep_wait();
  ptx::griddep_launch_dependents();
  const int c4 = g.C / 4;
  const int per_row = g.OW * c4;
  const int rows = g.N * g.OH;
  for (int r = blockIdx.x; r < rows; r += gridDim.x) {
    const int n = r / g.OH, oh = r - n * g.OH;
    const S* src = in + ((long long)n * g.H + (long long)oh * g.stride) * g.W * g.C;
    for (int i = threadIdx.x; i < per_row; i += blockDim.x) {
      const int ow = fdiv(i, fd_c4), c = (i - ow * c4) * 4;
      const long long o = (long long)r * per_row + i;
      const S* sp = src + (long long)ow * g.stride * g.C + c;
      TKB_DCHECK(ow < g.OW && (long long)oh * g.stride < g.H && (long long)ow * g.stride < g.W &&
                 n < g.N);
      if constexpr (sizeof(S) == 2) {  // bf16 activations in: a strided copy
        const uint2 u = __ldg(reinterpret_cast<const uint2*>(sp));
        reinterpret_cast<uint2*>(out)[o] = u;
      } else {
        const float4 v = __ldg(reinterpret_cast<const float4*>(sp));
        if constexpr (sizeof(T) == 4) {
          reinterpret_cast<float4*>(out)[o] = v;
        } else {
          __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
          uint2 u;
          u.x = *reinterpret_cast<uint32_t*>(&lo);
          u.y = *reinterpret_cast<uint32_t*>(&hi);
          reinterpret_cast<uint2*>(out)[o] = u;
        }
      }
    }
  }
}

template <typename T, typename S = float>
void pointwise_gather(const S* in, const ConvGeom& g, T* out, cudaStream_t st) {
  static_assert(sizeof(S) == 4 || sizeof(T) == 2, "bf16 input compacts to bf16");
  const long long rows = (long long)g.N * g.OH;
  if (rows > 2147483647ll || (long long)g.OW * (g.C / 4) > 2147483647ll)
    fail(TK_ERR_CAPABILITY, "pointwise gather: plane too large");
  const int blocks = (int)std::min<long long>(rows, (long long)sm_count() * 16);
  launch_pdl(pointwise_gather_kernel<T, S>, (unsigned)blocks, 256, st, in, g, make_fdiv(g.C / 4), out);
}

// Row-major patch matrix [pixel][kp] (K-major, zero padded to kp): one
// thread per 4-element chunk, consecutive threads write consecutive 16-byte
// chunks.  The explicit fallback for channel counts TMA cannot box and for
// strides != 1.
__global__ void __launch_bounds__(256) patches_rm_kernel(ConvGeom g, const float* __restrict__ in,
                                                         int kp, float* __restrict__ out,
                                                         long long chunks) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= chunks) return;
  const int per_pix = kp >> 2;
  const int pix = (int)(idx / per_pix);
  const int k0 = (int)(idx - (long long)pix * per_pix) * 4;
  const int ow = pix % g.OW;
  const int t = pix / g.OW;
  const int oh = t % g.OH;
  const int n = t / g.OH;
  const int K = g.R * g.S * g.C;
  float v[4];
  int c = k0 % g.C, tap = k0 / g.C;
  int y = tap % g.S, x = tap / g.S;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    float val = 0.0f;
    if (k0 + u < K) {
      const int ih = oh * g.stride + x - g.pad_t, iw = ow * g.stride + y - g.pad_l;
      if (ih >= 0 && iw >= 0 && ih < g.H && iw < g.W)
        val = __ldg(in + (((long long)n * g.H + ih) * g.W + iw) * g.C + c);
      if (++c == g.C) {
        c = 0;
        if (++y == g.S) {
          y = 0;
          ++x;
        }
      }
    }
    v[u] = val;
  }
  reinterpret_cast<float4*>(out)[idx] = make_float4(v[0], v[1], v[2], v[3]);
}

// Pixel-tile shape for the conv box: Wb x tileH pixels per tile, loaded as
// CG boxes of Wb x boxH.
struct BoxShape {
  int wb, tileH, boxH, tiles_w, tiles_h;
};

// pix_on_n: the tile is the MMA N side (P = BN, multiple of 16*CG, <= 256);
// otherwise it is the M side (P = 128*CG, each CTA boxes 128 pixels).
BoxShape pick_box(const ConvGeom& g, bool pix_on_n, int cg) {
  BoxShape best{0, 0, 0, 0, 0};
  double best_score = 1e30;
  for (int wb = 1; wb <= 256; ++wb) {
    for (int th = 1; wb * th <= 256 * cg; ++th) {
      const int P = wb * th;
      if (pix_on_n) {
        if (P > 256 || P % (16 * cg) != 0 || P < 64 || th % cg != 0) continue;
      } else {
        if (P != kRows * cg || th % cg != 0) continue;
      }
      if (wb > 2 * g.OW + 16 || th > 2 * g.OH + 16) continue;
      if (wb * g.stride > 256 || (th / cg) * g.stride > 256) continue;  // TMA box extent
      const int tw = (g.OW + wb - 1) / wb, tt = (g.OH + th - 1) / th;
      const double waste = (double)tw * wb * tt * th / ((double)g.OW * g.OH);
      const double score = waste * (1.0 + 24.0 / P);
      if (score < best_score - 1e-9) {
        best_score = score;
        best = BoxShape{wb, th, th / cg, tw, tt};
      }
    }
  }
  return best;
}

}  // namespace

namespace {
double split_cost_us(long long units, int num_kb, long long pairs, int cg, int bn, int s,
                     size_t out_bytes);
int choose_splits(long long units, int num_kb, long long pairs, int bm, int bn, size_t out_bytes,
                  size_t cap);
}  // namespace

void launch_tc_gemm(const TcGemm& g, cudaStream_t st) {
  require_tc(g.precision);
  const bool tf32 = g.precision == TK_PREC_TF32;
  const int esize = tf32 ? 4 : 2;
  const int ek = kSlabBytes / esize;
  if ((g.K * esize) % 16 != 0) fail(TK_ERR_CAPABILITY, "tc_gemm: rows must be 16-byte multiples");
  int cg = g.M > kRows ? 2 : 1;
  if (tc_knobs().cluster == 1 || tc_knobs().cluster == 2) cg = tc_knobs().cluster;
  int bn = g.tile_n > 0 ? g.tile_n : (g.N >= 256 ? 256 : ((g.N + 15) / 16) * 16);
  // Split-K (no C read, batch 1, dense output): every split stores its
  // partial product in the output's own layout, splitk_reduce sums them in
  // split order (deterministic).
  const int num_kb_all = (g.K + ek - 1) / ek;
  const size_t out_bytes = (size_t)g.M * g.N * 4;
  const bool dense = (g.d_sm == 1 && g.d_sn == g.M) || (g.d_sn == 1 && g.d_sm == g.N);
  const bool split_ok = !(g.c != nullptr && g.beta != 0.0f) && g.batch == 1 && dense &&
                        ((long long)g.M * g.N) % 4 == 0 &&
                        (reinterpret_cast<uintptr_t>(g.d) & 15) == 0;
  const size_t split_cap = std::max<size_t>(out_bytes * 4, (size_t)64 << 20);
  int splits = 1;
  if (g.tile_n <= 0 && g.N >= 64) {
    // Library tile for a GEMM too small to fill the SMs with 256 x 256
    // tiles: the (cluster, N tile, K splits) whose modelled time (waves of
    // max(MMA, operand feed) per slab + the stream-K tail or the split-K
    // reduction) is least.
    double best = 1e30;
    for (int c : {2, 1}) {
      if (tc_knobs().cluster != 0 && c != tc_knobs().cluster) continue;
      if (c == 2 && g.M <= kRows) continue;
      for (int b : {256, 128, 64}) {
        if (b > 64 && b >= 2 * g.N) continue;
        const long long tiles = (long long)((g.M + kRows * c - 1) / (kRows * c)) *
                                ((g.N + b - 1) / b) * g.batch;
        // Candidates in order of preference (SM pairs, wide tiles: the
        // measured winners whenever the SMs fill); a later one must beat
        // the model by 15% (4096^3: the model ties cg1/cg2, hardware
        // prefers the pair, 199 vs 225 us).
        double t = plan_tail(tiles, num_kb_all, c, b).cost_us;
        int sp = 1;
        if (split_ok) {
          sp = choose_splits(tiles, num_kb_all, sm_count() / c, kRows * c, b, out_bytes, split_cap);
          if (sp > 1) t = split_cost_us(tiles, num_kb_all, sm_count() / c, c, b, sp, out_bytes);
        }
        if (t < best * 0.85) {
          best = t;
          cg = c;
          bn = b;
          splits = sp;
        }
      }
    }
  } else if (split_ok) {
    const int c = cg;
    const int b = std::min(256, (bn + 16 * c - 1) / (16 * c) * (16 * c));
    const long long tiles =
        (long long)((g.M + kRows * c - 1) / (kRows * c)) * ((g.N + b - 1) / b) * g.batch;
    splits = choose_splits(tiles, num_kb_all, sm_count() / c, kRows * c, b, out_bytes, split_cap);
  }
  if (bn > 256) bn = 256;
  const int step = 16 * cg;
  bn = (bn + step - 1) / step * step;
  if (bn < step) bn = step;
  if (g.plan) {  // dry run (tk_gemm_plan_info): the tile choice and work split, no launch
    const int num_kb = (g.K + ek - 1) / ek;
    int sp = splits;
    if (sp > 1) {
      const int per = (num_kb + sp - 1) / sp;
      sp = (num_kb + per - 1) / per;
    }
    const bool read_c = g.c != nullptr && g.beta != 0.0f;
    const TailPlan tp = (read_c || sp > 1)
                            ? TailPlan{}
                            : plan_tail((long long)((g.M + kRows * cg - 1) / (kRows * cg)) *
                                            ((g.N + bn - 1) / bn) * g.batch,
                                        num_kb, cg, bn);
    g.plan->precision = g.precision;
    g.plan->cta_group = cg;
    g.plan->tile_m = kRows * cg;
    g.plan->tile_n = bn;
    g.plan->splits = sp;
    g.plan->tail_pieces = tp.q > 1 ? tp.q : 0;
    g.plan->k_depth = g.K;
    return;
  }
  TcArgs p{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.BN = bn;
  p.ek = ek;
  p.num_m = (g.M + kRows * cg - 1) / (kRows * cg);
  p.num_n = (g.N + bn - 1) / bn;
  p.batch = g.batch;
  p.num_kb = (g.K + ek - 1) / ek;
  p.d = g.d;
  p.c = g.c;
  p.d_sm = g.d_sm;
  p.d_sn = g.d_sn;
  p.d_batch = g.d_batch;
  p.alpha = g.alpha;
  p.beta = g.beta;
  p.read_c = g.c != nullptr && g.beta != 0.0f;
  if (splits > 1) {
    p.kb_per = (p.num_kb + splits - 1) / splits;
    splits = (p.num_kb + p.kb_per - 1) / p.kb_per;  // no empty split
  }
  p.splits = splits;
  if (splits <= 1) p.kb_per = p.num_kb;
  Scratch part_buf(st, kScratchPart, splits > 1 ? (size_t)splits * out_bytes : 0);
  if (splits > 1) {
    p.part = part_buf.as<float>();
    p.part_stride = (long long)g.M * g.N;
  }
  CUtensorMap ma;
  if (g.a_mn && !tf32) {
    // bf16 MN-major A: view {64 (M inner), K (stride lda), M / 64 (stride
    // 128 B)}, box {64, 64, 2}, the canonical 128-byte swizzle
    if (g.batch != 1 || g.M % 64 != 0 || (g.lda * 2) % 16 != 0)
      fail(TK_ERR_CAPABILITY, "tc_gemm: MN-major bf16 A needs batch 1, M % 64 == 0");
    const long long ak = g.a_k > 0 ? std::min<long long>(g.a_k, g.K) : g.K;
    cuuint64_t dims[3] = {64, (cuuint64_t)ak, (cuuint64_t)(g.M / 64)};
    cuuint64_t strides[2] = {(cuuint64_t)g.lda * 2, 128};
    cuuint32_t box[3] = {64, 64, (cuuint32_t)(kRows / 64)};
    ma = make_map(g.a, 2, 3, dims, strides, box);
    p.a_mn = 1;
  } else if (g.a_mn) {
    if (!tf32 || g.batch != 1 || g.M % 32 != 0 || (g.lda * 4) % 16 != 0)
      fail(TK_ERR_CAPABILITY, "tc_gemm: MN-major A needs TF32, batch 1, M % 32 == 0");
    // view {32 (M inner), K (stride lda), M / 32 (stride 128 B)}, box {32, 32, 4}
    const long long ak = g.a_k > 0 ? std::min<long long>(g.a_k, g.K) : g.K;
    cuuint64_t dims[3] = {32, (cuuint64_t)ak, (cuuint64_t)(g.M / 32)};
    cuuint64_t strides[2] = {(cuuint64_t)g.lda * 4, 128};
    cuuint32_t box[3] = {32, 32, (cuuint32_t)(kRows / 32)};
    ma = make_map(g.a, 4, 3, dims, strides, box, nullptr, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
    p.a_mn = 1;
  } else {
    ma = map_rows(g.a, esize, g.K, g.M, g.batch, g.a_batch, kRows);
  }
  const CUtensorMap mb = map_rows(g.b, esize, g.K, g.N, g.batch, g.b_batch, bn / cg);
  // Row-major output (d_sn == 1): stage through smem and TMA-store it.
  CUtensorMap md = ma;
  if (g.d_sn == 1 && !p.read_c && (g.d_sm * 4) % 16 == 0 &&
      (reinterpret_cast<uintptr_t>(g.d) & 15) == 0 && (bn % 32 == 0 || p.num_n == 1) &&
      (g.batch == 1 || (g.d_batch * 4) % 16 == 0)) {
    // (split-K: the partials, batch coordinate = split)
    cuuint64_t dims[3] = {(cuuint64_t)g.N, (cuuint64_t)g.M, (cuuint64_t)(splits > 1 ? splits : g.batch)};
    cuuint64_t strides[2] = {(cuuint64_t)g.d_sm * 4,
                             (cuuint64_t)(splits > 1 ? p.part_stride
                                                     : (g.d_batch ? g.d_batch : g.d_sm * g.M)) * 4};
    cuuint32_t box[3] = {32, (cuuint32_t)kRows, 1};
    md = make_map(splits > 1 ? p.part : g.d, 4, 3, dims, strides, box);
    p.store_tma = 1;
    p.epi_bufs = 2;
  }
  const TailPlan tp = (p.read_c || splits > 1)
                         ? TailPlan{}
                         : plan_tail((long long)p.num_m * p.num_n * p.batch, p.num_kb, cg, bn);
  Scratch tail_buf(st, kScratchTail, tp.q > 1 ? tp.bytes : 0);
  if (tp.q > 1) apply_tail(p, tp, tail_buf.as<float>());
  dispatch<kPlain>(ma, mb, md, p, cg, tf32, st);
  if (splits > 1) splitk_reduce(p.part, (long long)g.M * g.N, splits, g.d, st);
}

void launch_split3_rows(const float* src, long long rows, long long kp, float* dst, int pattern,
                        cudaStream_t st) {
  split3_rows(src, rows, kp, dst, pattern, st);
}

void launch_tc_batched_colmajor(size_t m, size_t n, size_t k, size_t batch, const float* a,
                                long long sa, const float* b, long long sb, float* d, long long sc,
                                int precision, cudaStream_t st) {
  require_tc(precision);
  if (m > 2147483647ull || n > 2147483647ull || k > 2147483647ull || batch > 2147483647ull)
    fail(TK_ERR_CAPABILITY, "gemm_batched_strided: dimensions exceed the 32-bit index range");
  if (precision == TK_PREC_3XTF32) {  // the split-precision path, member by member
    for (size_t g = 0; g < batch; ++g)
      launch_tc_colmajor_gemm(m, n, k, 1.0f, 0.0f, false, false, a + g * sa, b + g * sb, nullptr,
                              d + g * sc, precision, 0, st);
    return;
  }
  const bool tf32 = precision == TK_PREC_TF32;
  const long long kp = tf32 ? (long long)((k + 3) / 4 * 4) : (long long)((k + 7) / 8 * 8);
  const size_t esz = tf32 ? 4 : 2;
  // B_g (k x n column-major) is K-major already: read in place when its rows
  // and batch stride are 16-byte multiples (TF32).
  const bool b_ok = tf32 && kp == (long long)k && (reinterpret_cast<uintptr_t>(b) & 15) == 0 &&
                    (sb * 4) % 16 == 0;
  Scratch spa(st, kScratchPackA, batch * m * (size_t)kp * esz);
  Scratch spb(st, kScratchPackB, b_ok ? 0 : batch * n * (size_t)kp * esz);
  char* pa = static_cast<char*>(spa.get());
  char* pb = static_cast<char*>(spb.get());
  for (size_t g = 0; g < batch; ++g) {
    const float* ag = a + g * sa;
    void* dst = pa + g * m * (size_t)kp * esz;  // A_g^T: rows m, K contiguous
    if (tf32) pack_kmajor<float>(ag, 1, (long long)m, (long long)m, (long long)k, kp, (float*)dst, false, st);
    else pack_kmajor<__nv_bfloat16>(ag, 1, (long long)m, (long long)m, (long long)k, kp, (__nv_bfloat16*)dst, false, st);
    if (!b_ok) {
      const float* bg = b + g * sb;
      void* bd = pb + g * n * (size_t)kp * esz;
      if (tf32) pack_kmajor<float>(bg, (long long)k, 1, (long long)n, (long long)k, kp, (float*)bd, false, st);
      else pack_kmajor<__nv_bfloat16>(bg, (long long)k, 1, (long long)n, (long long)k, kp, (__nv_bfloat16*)bd, false, st);
    }
  }
  TcGemm t;
  t.M = (int)m;
  t.N = (int)n;
  t.K = (int)kp;
  t.batch = (int)batch;
  t.a = reinterpret_cast<const float*>(pa);
  t.a_batch = (long long)m * kp;
  t.b = b_ok ? b : reinterpret_cast<const float*>(pb);
  t.b_batch = b_ok ? sb : (long long)n * kp;
  t.d = d;
  t.d_sm = 1;
  t.d_sn = (long long)m;
  t.d_batch = sc;
  t.precision = precision;
  launch_tc_gemm(t, st);
}

void launch_tc_colmajor_gemm(size_t m, size_t n, size_t k, float alpha, float beta, bool ta,
                             bool tb, const float* a, const float* b, const float* c, float* d,
                             int precision, int tile_n, cudaStream_t st, TcGemmPlan* plan) {
  require_tc(precision);
  if (precision == TK_PREC_3XTF32) {
    // Pack both operands K-major (fp32, unrounded), expand to the split
    // triple along K, run one TF32 GEMM of depth 3 kp.
    const long long kp = (long long)((k + 3) / 4 * 4);
    if (plan) {
      TcGemm g;
      g.M = (int)m;
      g.N = (int)n;
      g.K = (int)(3 * kp);
      g.c = c;
      g.d_sm = 1;
      g.d_sn = (long long)m;
      g.beta = beta;
      g.precision = TK_PREC_TF32;
      g.tile_n = tile_n;
      g.plan = plan;
      launch_tc_gemm(g, st);
      plan->a_in_place = plan->b_in_place = 0;
      return;
    }
    Scratch spa(st, kScratchPackA, (size_t)m * kp * 4), spb(st, kScratchPackB, (size_t)n * kp * 4);
    Scratch sa3(st, kScratchSplitA, (size_t)m * kp * 12), sb3(st, kScratchSplitB, (size_t)n * kp * 12);
    float *pa = spa.as<float>(), *pb = spb.as<float>(), *a3 = sa3.as<float>(), *b3 = sb3.as<float>();
    if (ta) pack_kmajor<float>(a, (long long)k, 1, (long long)m, (long long)k, kp, pa, false, st);
    else pack_kmajor<float>(a, 1, (long long)m, (long long)m, (long long)k, kp, pa, false, st);
    if (tb) pack_kmajor<float>(b, 1, (long long)n, (long long)n, (long long)k, kp, pb, false, st);
    else pack_kmajor<float>(b, (long long)k, 1, (long long)n, (long long)k, kp, pb, false, st);
    split3_rows(pa, (long long)m, kp, a3, 0, st);
    split3_rows(pb, (long long)n, kp, b3, 1, st);
    TcGemm g;
    g.M = (int)m;
    g.N = (int)n;
    g.K = (int)(3 * kp);
    g.a = a3;
    g.b = b3;
    g.d = d;
    g.c = c;
    g.d_sm = 1;
    g.d_sn = (long long)m;
    g.alpha = alpha;
    g.beta = beta;
    g.precision = TK_PREC_TF32;
    g.tile_n = tile_n;
    launch_tc_gemm(g, st);
    return;
  }
  const bool tf32 = precision == TK_PREC_TF32;
  const long long kp = tf32 ? (long long)((k + 3) / 4 * 4) : (long long)((k + 7) / 8 * 8);
  // TF32 operands already K-major with 16-byte rows are used in place;
  // everything else is packed (and converted for BF16).
  // bf16 operands in HBM (tk_exec_options.io, BF16 only): a and b address
  // bf16 column-major matrices; K-major ones with 16-byte rows are used in
  // place, the rest are packed bf16 -> bf16 (no conversion).
  const bool in16 = (tc_knobs().io & TK_IO_IN_BF16) != 0;
  if (in16 && tf32) fail(TK_ERR_CAPABILITY, "gemm: bf16 operands (io flags) need BF16 precision");
  auto aligned = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  const bool a_ok = (tf32 || in16) && ta && kp == (long long)k && aligned(a);
  const bool b_ok = (tf32 || in16) && !tb && kp == (long long)k && aligned(b);
  // Column-major, untransposed A is MN-major: the tensor core reads it in
  // place (no transpose pass) when M is a multiple of 32.
  const bool mn_on = experiments().a_mn;
  // (bf16 operands in HBM: the same in-place read of an untransposed A, in
  // 64-element M blocks)
  const bool a_mn = mn_on && !ta && aligned(a) && m <= (1ull << 31) &&
                    ((tf32 && m % 32 == 0) || (in16 && m % 64 == 0));
  const size_t esz = tf32 ? 4 : 2;
  if (plan) {
    TcGemm g;
    g.M = (int)m;
    g.N = (int)n;
    g.K = (int)kp;
    g.a_mn = a_mn;
    g.c = c;
    g.d_sm = 1;
    g.d_sn = (long long)m;
    g.beta = beta;
    g.precision = precision;
    g.tile_n = tile_n;
    g.plan = plan;
    launch_tc_gemm(g, st);
    plan->a_in_place = (a_ok || a_mn) ? 1 : 0;
    plan->b_in_place = b_ok ? 1 : 0;
    return;
  }
  Scratch spa(st, kScratchPackA, (!a_ok && !a_mn) ? (size_t)m * kp * esz : 0);
  Scratch spb(st, kScratchPackB, !b_ok ? (size_t)n * kp * esz : 0);
  void* pa = spa.get();
  void* pb = spb.get();
  auto pack = [&](const float* src, long long rs, long long ks, long long rows, void* dst) {
    if (tf32) pack_kmajor<float>(src, rs, ks, rows, (long long)k, kp, (float*)dst, false, st);
    else if (in16)
      pack_kmajor<__nv_bfloat16, __nv_bfloat16>(reinterpret_cast<const __nv_bfloat16*>(src), rs, ks,
                                                rows, (long long)k, kp, (__nv_bfloat16*)dst, false, st);
    else pack_kmajor<__nv_bfloat16>(src, rs, ks, rows, (long long)k, kp, (__nv_bfloat16*)dst, false, st);
  };
  if (!a_ok && !a_mn) {
    if (ta) pack(a, (long long)k, 1, (long long)m, pa);
    else pack(a, 1, (long long)m, (long long)m, pa);
  }
  if (!b_ok) {
    if (tb) pack(b, 1, (long long)n, (long long)n, pb);
    else pack(b, (long long)k, 1, (long long)n, pb);
  }
  TcGemm g;
  g.M = (int)m;
  g.N = (int)n;
  g.K = (int)kp;
  g.a = (a_ok || a_mn) ? a : (const float*)pa;
  g.a_mn = a_mn;
  g.lda = (long long)m;
  g.a_k = (long long)k;  // A holds k columns; the padded K tail reads as zeros
  g.b = b_ok ? b : (const float*)pb;
  g.d = d;
  g.c = c;
  g.d_sm = 1;
  g.d_sn = (long long)m;
  g.alpha = alpha;
  g.beta = beta;
  g.precision = precision;
  g.tile_n = tile_n;
  launch_tc_gemm(g, st);
}

namespace {

// Slab width in elements for the precision.
int slab_elems(int precision) { return precision == TK_PREC_TF32 ? 32 : 64; }

// Pixel boxes need whole slabs of channels; stride 2 through a traversal
// stride (box extent s*wb <= 256).
bool conv_boxable(const ConvGeom& g, int precision) {
  return g.C % slab_elems(precision) == 0 && (g.stride == 1 || g.stride == 2);
}

size_t align256(size_t b) { return (b + 255) / 256 * 256; }

// How a convolution runs on the tensor cores and what its workspace holds.
//   kGatherPlan    any C / stride: producer warps build the pixel operand
//   kBoxPlan       C a whole number of slabs, stride 1: halo / pixN / pixM
//   kPointwisePlan 1x1 window: a plain GEMM [pixels][C] x [Kout][C]^T on the
//                  NHWC input itself (stride 1, TF32) or on a compacted /
//                  converted copy (stride 2, BF16), split over K when the
//                  output has too few tiles to fill the SMs
//   kIm2colPlan    C a whole number of slabs: a plain GEMM whose A rows are
//                  output pixels loaded by im2col-mode TMA (runs of 128
//                  pixels in NHW order, one tap per K-slab), filter on N
enum PlanKind : int { kGatherPlan = 0, kBoxPlan = 1, kPointwisePlan = 2, kIm2colPlan = 3 };

struct ConvPlan {
  int kind = kGatherPlan;
  bool tf32 = true;
  long long kp = 0;          // packed filter row length (elements)
  size_t filt_bytes = 0;     // packed filter
  size_t in_bytes = 0;       // converted / compacted input copy
  size_t part_bytes = 0;     // split-K partial tiles
  int cg = 2, bn = 0, splits = 1, kb_per = 0, num_kb = 0;
  TailPlan tail{};           // wave-quantisation tail (plain / pixN)
  // kBoxPlan layout
  bool halo = false, pix_on_n = false;
  BoxShape bx{};
  int imgs = 1;  // pixN: whole images per pixel tile (small planes)
  bool flat = false;  // pixN: flat-row tiles (see TcArgs::flat)
  int num_m = 0, num_n = 0;
  int narrow_cp = 0;  // narrow halo (16-byte pixels): channels after padding (4 / 8)
};

// bf16 activations in HBM (tk_exec_options.io, BF16 convs): the input needs
// no conversion pass / the epilogue writes bf16.
inline bool io_in_bf16() { return (tc_knobs().io & TK_IO_IN_BF16) != 0; }
inline bool io_out_bf16() { return (tc_knobs().io & TK_IO_OUT_BF16) != 0; }

// Split-K count from a small cost model (times in us, B200 at ~1.9 GHz):
// a unit of kb slabs costs kb * max(MMA, operand-feed) + 1 (fill + epilogue),
// units run in waves over the SM pairs, and a split adds the reduction pass
// (launch + every partial read once and the output written, ~4 TB/s).  The
// partials must stay under `cap` bytes.
// Modelled time (us) of `units` tiles split s ways over K: waves of
// (kb / s slabs + 1 us), plus the ordered reduction pass (launch + every
// partial read once and the output written at ~4 TB/s).
double split_cost_us(long long units, int num_kb, long long pairs, int cg, int bn, int s,
                     size_t out_bytes) {
  const long long waves = (units * s + pairs - 1) / pairs;
  const int kb = (num_kb + s - 1) / s;
  double t = (double)waves * (kb * slab_time_us(cg, bn) + 1.0);
  if (s > 1) t += 2.0 + (double)(s + 1) * out_bytes / (experiments().red_gbs * 1e3);
  return t;
}

int choose_splits(long long units, int num_kb, long long pairs, int bm, int bn,
                  size_t out_bytes, size_t cap) {
  const int forced = tc_knobs().split;
  if (forced == 1) return 1;
  if (forced > 1) {
    // splitk_reduce sums at most kMaxSplits partials.
    int sp = std::min(std::min(forced, kMaxSplits), std::max(1, num_kb / 2));
    while (sp > 1 && (size_t)sp * out_bytes > cap) --sp;
    return sp;
  }
  auto cost = [&](int s) { return split_cost_us(units, num_kb, pairs, bm / kRows, bn, s, out_bytes); };
  int best = 1;
  // No split leaves the balanced tail (plan_tail) to even out the last wave.
  double best_t = std::min(cost(1), plan_tail(units, num_kb, bm / kRows, bn).cost_us);
  for (int s = 2; s <= 16 && num_kb / s >= 4; ++s) {
    if ((size_t)s * out_bytes > cap) break;
    const double t = cost(s);
    if (t < best_t * 0.9) {
      best = s;
      best_t = t;
    }
  }
  return best;
}

void finish_splits(ConvPlan& c, int num_kb, int splits, size_t out_bytes, long long tiles) {
  c.num_kb = num_kb;
  c.splits = 1;
  c.kb_per = num_kb;
  if (splits > 1) {
    c.kb_per = (num_kb + splits - 1) / splits;
    c.splits = (num_kb + c.kb_per - 1) / c.kb_per;  // no empty split
  }
  (void)tiles;
  if (c.splits > 1) c.part_bytes = align256((size_t)c.splits * out_bytes);
}

// Automatic choice of the im2col plan (see plan_conv_impl).
// Measured (same-box A/B of every ResNet-50 / VGG-16 layer, tools/
// layer_times.py --mode im2col, confirmed by the tuner's DB
// profiles/r01_tune_*_knobs.ndjson):
//  * TF32 strided 1x1 layers gain from the im2col traversal (ResNet
//    res3a_branch1 33 -> 27, res4a_branch2a 19 -> 17, res5a_branch2a 24 ->
//    20, res5a_branch1 33 -> 27 us);
//  * 3x3 layers with >= 128 channels, >= 256 features on planes >= 28 x 28,
//    both precisions, once the two-half epilogue staging left the 256 x 256
//    tiles six operand stages (VGG conv4_1 99 -> 86, conv4_2 170 -> 151,
//    conv3_1 95 -> 90 us TF32; BF16 conv3_2/conv4_2 119/107 -> 112/97 us);
//    smaller planes and feature counts stay on halo / pixel boxes;
//  * BF16 stride-1 1x1 layers that expand the features (K >= 2C) or run on
//    7 x 7 planes (res2a_branch2c 40 -> 36, res5b_branch2a 29 -> 25 us).
bool prefer_im2col(const ConvGeom& g, int precision) {
  const bool tf32 = precision == TK_PREC_TF32;
  if (tf32 && g.R == 1 && g.S == 1 && g.stride == 2) return true;
  if (g.R == 3 && g.S == 3 && g.stride == 1 && g.C >= 128 && g.K >= 256 && g.OH >= 28)
    return true;
  if (!tf32 && g.R == 1 && g.S == 1 && g.stride == 1 && (g.K >= 2 * g.C || g.OH <= 7)) return true;
  return false;
}

// 3xTF32 runs one TF32 convolution over 3C channels; the operand-path rules
// that depend on the channel count judge the caller's C (measured with the
// tuner: halo tiles for VGG conv1_2 / conv2_x in 3xTF32, 1326 -> 939 us on
// conv1_2, while the 3C view had sent them to pixel boxes).
thread_local int t_split3_div = 1;
struct Split3Scope {
  Split3Scope() { t_split3_div = 3; }
  ~Split3Scope() { t_split3_div = 1; }
};

ConvPlan plan_conv_impl(const ConvGeom& g, int precision) {
  ConvPlan c;
  const long long K = (long long)g.R * g.S * g.C;
  const bool tf32 = precision == TK_PREC_TF32;
  const int esize = tf32 ? 4 : 2, ek = kSlabBytes / esize;
  const long long pix = (long long)g.N * g.OH * g.OW;
  const char* force = experiments().conv_mode.empty() ? nullptr : experiments().conv_mode.c_str();
  const int mode = tc_knobs().mode;
  // Strided 1x1 in TF32 reads the strided pixels straight through a
  // traversal-stride pixel box (no compacting pass); BF16 needs a conversion
  // pass anyway, which compacts for free.
  // (Small planes waste too much of a pixel box: 7x7 -> 8x8 boxes.)
  const bool strided_box = g.stride > 1 && tf32 && conv_boxable(g, precision) &&
                           mode != TK_TC_POINTWISE && g.OH * g.OW >= 196;
  // BF16 stride-1 1x1 layers on planes >= 14 x 14 with <= 512 features run
  // faster as one-tap halo convolutions than as the plain GEMM (same-box
  // A/B: ResNet res2b/res3b/res4b_branch2a 60/38/29 -> 45/28/24 us).
  const bool auto_sel = mode == TK_TC_AUTO && !force;
  const bool bf16_pw_halo = auto_sel && !tf32 && g.R == 1 && g.S == 1 && g.stride == 1 &&
                            g.OH >= 14 && g.K <= 512 && g.K % 32 == 0 && conv_boxable(g, precision);
  const bool pointwise = g.R == 1 && g.S == 1 && g.pad_t == 0 && g.pad_l == 0 && g.C % 8 == 0 &&
                         g.K % 4 == 0 && !(force && std::string(force) != "plain") &&
                         (mode == TK_TC_AUTO || mode == TK_TC_POINTWISE) && !strided_box &&
                         !bf16_pw_halo;
  // Pixels-on-M GEMM sizing shared by the pointwise and im2col plans: SM
  // pair tiles of 256 pixels x bn features, split over K when the tiles
  // cannot fill the pairs, the last partial wave cut into K-pieces.
  auto size_pixels_gemm = [&](ConvPlan& c) {
    c.cg = pix > kRows ? 2 : 1;
    const int step = 16 * c.cg;
    c.bn = g.K >= 256 ? 256 : (g.K + step - 1) / step * step;
    const long long pairs = sm_count() / c.cg;
    auto units = [&](int bn) {
      return ((pix + kRows * c.cg - 1) / (kRows * c.cg)) * ((g.K + bn - 1) / bn);
    };
    if (c.bn > 128 && units(c.bn) < pairs) c.bn = 128;
    // Short-K (HBM-bound) layers are epilogue-bound: a 128-wide tile keeps
    // two TMA-store staging buffers, so a tile's store overlaps the next
    // drain.
    if (c.bn > 128 && c.kp / ek <= 4) c.bn = 128;
    if (experiments().pw_bn > 0) c.bn = experiments().pw_bn;
    c.num_m = (int)((pix + kRows * c.cg - 1) / (kRows * c.cg));
    c.num_n = (g.K + c.bn - 1) / c.bn;
    const int num_kb = (int)(c.kp / ek);
    const size_t out_bytes = (size_t)pix * g.K * 4;
    finish_splits(c, num_kb,
                  choose_splits(units(c.bn), num_kb, pairs, kRows * c.cg, c.bn, out_bytes,
                                96ull << 20),
                  out_bytes, (long long)c.num_m * c.num_n);
    if (c.splits == 1) c.tail = plan_tail((long long)c.num_m * c.num_n, c.num_kb, c.cg, c.bn);
  };
  const bool im2col = conv_boxable(g, precision) && g.K % 4 == 0 &&
                      (mode == TK_TC_IM2COL || (force && std::string(force) == "im2col") ||
                       (mode == TK_TC_AUTO && !force && prefer_im2col(g, precision)));
  if (im2col) {
    c.kind = kIm2colPlan;
    c.tf32 = tf32;
    c.kp = K;
    c.filt_bytes = align256((size_t)g.K * K * esize);
    c.in_bytes = (tf32 || io_in_bf16()) ? 0 : align256((size_t)g.N * g.H * g.W * g.C * 2);
    size_pixels_gemm(c);
    return c;
  }
  if (pointwise) {
    c.kind = kPointwisePlan;
    c.tf32 = tf32;
    c.kp = (g.C + ek - 1) / ek * ek;
    c.filt_bytes = align256((size_t)g.K * c.kp * esize);
    c.in_bytes = (g.stride != 1 || (!tf32 && !io_in_bf16())) ? align256((size_t)pix * g.C * esize) : 0;
    size_pixels_gemm(c);
    return c;
  }
  if (conv_boxable(g, precision) && mode != TK_TC_GATHER) {
    c.kind = kBoxPlan;
    c.tf32 = tf32;
    c.kp = K;
    c.filt_bytes = align256((size_t)g.K * K * esize);
    c.in_bytes = (tf32 || io_in_bf16()) ? 0 : align256((size_t)g.N * g.H * g.W * g.C * 2);
    // Halo mode: small-feature stride-1 layers whose tap re-reads of the
    // input would otherwise dominate the L2->SM traffic.
    const bool halo_ok = g.stride == 1 && g.R * g.S <= 9 && g.S <= 3 && g.K % 32 == 0 &&
                         ((g.K <= 128 && g.C / t_split3_div <= 128) ||
                          (force && std::string(force).rfind("halo", 0) == 0));
    c.halo = halo_ok && !(force && std::string(force).rfind("halo", 0) != 0);
    const bool halo_geom = g.stride == 1 && g.R * g.S <= 9 && g.S <= 3 && g.K % 32 == 0;
    // Between halo and pixel boxes for >= 128 channels the deciding factor
    // is how well pixN's tiles fill the SM pairs (measured with the tuner,
    // profiles/r01_tune_*_knobs.ndjson): full waves favour pixN (VGG
    // conv2_2, 3% faster), a mostly idle last wave favours halo's 4x more,
    // narrower tiles (ResNet res4a_branch2b: 30 vs 40 us).
    if (halo_geom && g.C / t_split3_div >= 128 && g.K <= 256 && !force && mode == TK_TC_AUTO) {
      const int pcg = g.K >= 2 * kRows ? 2 : 1;
      const BoxShape pb = pick_box(g, true, pcg);
      if (pb.wb != 0) {
        const long long units = ((g.K + kRows * pcg - 1) / (kRows * pcg)) *
                                (long long)g.N * pb.tiles_w * pb.tiles_h;
        const long long pairs = sm_count() / pcg;
        const double eff = (double)units / (double)(((units + pairs - 1) / pairs) * pairs);
        // (128-wide halo tiles, K % 128 == 0, beat full-wave pixN too: VGG
        // conv2_2 185 -> 150 us)
        if (c.halo && eff >= 0.9 && g.K % 128 != 0) c.halo = false;
        if (!c.halo && eff < 0.6) c.halo = true;
      }
    }
    // BF16 on planes >= 28 x 28 with 128-multiple features: halo's one
    // input box per channel chunk halves the operand traffic of the
    // conversion-bound BF16 layers (VGG conv2_2 / conv3_1 / conv4_1 / conv4_2
    // 157/70/71/111 -> 138/67/62/107 us), and the one-tap 1x1 case above.
    if (auto_sel && !tf32 && halo_geom &&
        ((g.K % 128 == 0 && g.OH >= 28 && g.C >= 64) || bf16_pw_halo))
      c.halo = true;
    if (mode == TK_TC_HALO && halo_geom) c.halo = true;
    if (mode == TK_TC_PIXN || mode == TK_TC_PIXM) c.halo = false;
    c.num_kb = (int)(K / ek);
    c.kb_per = c.num_kb;
    if (c.halo) return c;
    c.pix_on_n = g.K >= kRows;
    if (mode == TK_TC_PIXN) c.pix_on_n = true;
    if (mode == TK_TC_PIXM && g.K % 4 == 0 && g.K <= 256) c.pix_on_n = false;  // BN <= 256
    c.cg = c.pix_on_n ? (g.K >= 2 * kRows ? 2 : 1) : 2;
    if (c.pix_on_n && (tc_knobs().cluster == 1 || tc_knobs().cluster == 2)) c.cg = tc_knobs().cluster;
    c.bx = pick_box(g, c.pix_on_n, c.cg);
    // Planes of at most 8 x 8 (ResNet res5, 7 x 7): one 8 x 8 box per image
    // wastes little and 256 / 64 = 4 images fill a 256-wide tile (instead of
    // a 64-wide tile whose N = 64 MMAs and filter re-reads dominate).
    if (c.pix_on_n && c.cg == 2 && g.OH <= 8 && g.OW <= 8 && g.N >= 4 &&
        !(force && std::string(force) == "pixn1")) {
      c.imgs = 4;
      c.bx = BoxShape{8, 8, 8, 1, 1};
    }
    // Flat rows: full-width boxes whose height divides OH tile N*OH rows
    // with no per-image row padding (28 x 28: 2 x 4 rows x 28 = 224 pixels,
    // where any per-image box pads 28 rows to 32).
    if (c.pix_on_n && c.imgs == 1 && c.bx.wb != 0 && !(force && std::string(force) == "pixn1")) {
      const double waste = (double)c.bx.tiles_w * c.bx.wb * c.bx.tiles_h * c.bx.tileH /
                           ((double)g.OW * g.OH);
      int best_bh = 0;
      for (int bh = 1; bh <= g.OH; ++bh) {
        const int P = c.cg * bh * g.OW;
        if (g.OH % bh || P > 256 || P < 64 || P % (16 * c.cg) || g.OW * g.stride > 256 ||
            bh * g.stride > 256)
          continue;
        best_bh = bh;  // the largest qualifying box
      }
      if (best_bh && waste > 1.02) {
        c.flat = true;
        c.bx = BoxShape{g.OW, c.cg * best_bh, best_bh, 1, 1};
      }
    }
    if (c.bx.wb == 0) return c;  // reported by the launcher
    const long long pix_tiles =
        c.flat ? ((long long)g.N * g.OH + c.bx.tileH - 1) / c.bx.tileH
               : ((long long)g.N + c.imgs - 1) / c.imgs * c.bx.tiles_w * c.bx.tiles_h;
    if (c.pix_on_n) {
      c.num_m = (g.K + kRows * c.cg - 1) / (kRows * c.cg);
      c.num_n = (int)pix_tiles;
      const size_t out_bytes = (size_t)g.N * g.OH * g.OW * g.K * 4;
      const bool aligned = g.K % 4 == 0;
      const long long pairs = sm_count() / c.cg;
      const int pbn = c.bx.wb * c.bx.tileH * c.imgs;
      const int sp = (aligned && !experiments().no_split)
                         ? choose_splits((long long)c.num_m * c.num_n, c.num_kb, pairs,
                                         kRows * c.cg, pbn, out_bytes, 64ull << 20)
                         : 1;
      finish_splits(c, c.num_kb, sp, out_bytes, (long long)c.num_m * c.num_n);
      if (c.splits == 1) c.tail = plan_tail((long long)c.num_m * c.num_n, c.num_kb, c.cg, pbn);
    } else {
      c.num_m = (int)pix_tiles;
      c.num_n = 1;
    }
    return c;
  }
  // Narrow pixels (C <= 4 tf32 / 8 bf16 channels, the C = 3 first layers):
  // the input padded once to 16-byte pixels feeds im2col-mode TMA, 8 taps
  // per K-slab (TcArgs::narrow_taps) -- the producer-warp gather and its
  // per-tile handshake are off the path, and BF16 stays BF16.
  const int ncp = tf32 ? 4 : 8;
  const bool narrow_ok = g.C <= ncp && (g.stride == 1 || g.stride == 2) && g.K % 32 == 0 &&
                         g.K <= 256 && (mode == TK_TC_AUTO || mode == TK_TC_HALO) &&
                         !(force && std::string(force) == "gather");
  if (narrow_ok) {
    const int taps = g.R * g.S;
    c.tf32 = tf32;
    c.narrow_cp = ncp;
    c.kp = (long long)((taps + 7) / 8) * 8 * ncp;
    c.filt_bytes = align256((size_t)g.K * c.kp * esize);
    c.in_bytes = align256((size_t)g.N * g.H * g.W * ncp * esize);
    // Halo boxes: the taps are shifted views of one box per stride phase
    // (no per-tap loads).  (Narrow im2col-mode TMA -- one 16-byte pixel per
    // box row, 8 taps per slab -- was measured slower: conv1_1 194 us.)
    if (g.S <= 2 * 16 - 2) {
      c.in_bytes = align256((size_t)g.N * g.H * g.stride *
                            (g.OW + (g.S - 1) / g.stride + 16) * ncp * esize);  // narrow_w2
      c.kind = kBoxPlan;
      c.halo = true;
      c.cg = 2;
      c.num_kb = 1;
      c.kb_per = 1;
      return c;
    }
  }
  c.narrow_cp = 0;
  c.kp = 0;
  c.kind = kGatherPlan;  // fp32 operands, kind::tf32 for every TC precision
  c.tf32 = true;
  c.kp = (K + 31) / 32 * 32;
  c.filt_bytes = align256((size_t)g.K * c.kp * 4);
  return c;
}

// The plan, with explicitly requested knobs (tk_exec_options.tc_mode /
// tc_cluster) that this shape cannot honour rejected as CapabilityError --
// a tuner then skips the candidate instead of timing a mislabeled one.
ConvPlan plan_conv(const ConvGeom& g, int precision) {
  const ConvPlan c = plan_conv_impl(g, precision);
  const int mode = tc_knobs().mode, cluster = tc_knobs().cluster;
  const bool ok = mode == TK_TC_AUTO ||
                  (mode == TK_TC_POINTWISE && c.kind == kPointwisePlan) ||
                  (mode == TK_TC_GATHER && c.kind == kGatherPlan) ||
                  (mode == TK_TC_HALO && c.kind == kBoxPlan && c.halo) ||
                  (mode == TK_TC_PIXN && c.kind == kBoxPlan && !c.halo && c.pix_on_n) ||
                  (mode == TK_TC_PIXM && c.kind == kBoxPlan && !c.halo && !c.pix_on_n) ||
                  (mode == TK_TC_IM2COL && c.kind == kIm2colPlan);
  if (!ok) fail(TK_ERR_CAPABILITY, "tc_conv: operand path " + std::to_string(mode) +
                                       " does not apply to this convolution");
  if (cluster != 0 && cluster != c.cg)  // only the pixN plan takes the cluster knob
    fail(TK_ERR_CAPABILITY, "tc_conv: cluster size " + std::to_string(cluster) +
                                " does not apply to this convolution's operand path");
  return c;
}

bool tf32_filter_rounding() { return experiments().tf32_round; }

// 1x1 convolution as a plain tensor-core GEMM (see plan_conv).
void launch_pointwise(const ConvGeom& g, const ConvPlan& c, const float* in, const float* filt,
                      float* out, char* ws, cudaStream_t st, bool prep, bool run) {
  const int esize = c.tf32 ? 4 : 2, ek = kSlabBytes / esize;
  char* cursor = ws;
  void* ft = cursor;
  cursor += c.filt_bytes;
  float* part = reinterpret_cast<float*>(ws + c.filt_bytes + c.in_bytes);
  if (prep) {
    if (c.tf32) pack_filter<float>(filt, g.C, g.K, (int)c.kp, (float*)ft, tf32_filter_rounding(), st);
    else pack_filter<__nv_bfloat16>(filt, g.C, g.K, (int)c.kp, (__nv_bfloat16*)ft, false, st);
  }
  if (!run) return;
  const long long pix = (long long)g.N * g.OH * g.OW;
  const void* a = in;
  if (c.in_bytes) {
    if (c.tf32) pointwise_gather<float>(in, g, (float*)cursor, st);
    else if (io_in_bf16())
      pointwise_gather<__nv_bfloat16>(reinterpret_cast<const __nv_bfloat16*>(in), g,
                                      (__nv_bfloat16*)cursor, st);
    else pointwise_gather<__nv_bfloat16>(in, g, (__nv_bfloat16*)cursor, st);
    a = cursor;
    cursor += c.in_bytes;
  }
  float* dst = c.splits > 1 ? part : out;
  const bool ob = io_out_bf16() && c.splits == 1;  // (split partials stay fp32)
  if (pix > 2147483647ll) fail(TK_ERR_CAPABILITY, "tc_conv: too many output pixels");
  TcArgs p{};
  p.M = (int)pix;
  p.N = g.K;
  p.K = (int)c.kp;
  p.BN = c.bn;
  p.ek = ek;
  p.num_m = c.num_m;
  p.num_n = c.num_n;
  p.batch = 1;
  p.num_kb = c.num_kb;
  p.splits = c.splits;
  p.kb_per = c.kb_per;
  p.d = out;
  p.d_sm = g.K;
  p.d_sn = 1;
  p.part = part;
  p.part_stride = pix * g.K;
  p.alpha = 1.0f;
  apply_tail(p, c.tail, reinterpret_cast<float*>(reinterpret_cast<char*>(part) + c.part_bytes));
  const CUtensorMap ma = map_rows(a, esize, g.C, pix, 1, 0, kRows);
  const CUtensorMap mb = map_rows(ft, esize, c.kp, g.K, 1, 0, c.bn / c.cg);
  const CUtensorMap md = out_map_rows(dst, ob, g.K, pix, c.splits);
  p.out_bf16 = ob;
  p.store_tma = 1;
  p.epi_bufs = 2;
  dispatch<kPlain>(ma, mb, md, p, c.cg, c.tf32, st);
  if (c.splits > 1) splitk_reduce(part, pix * g.K, c.splits, out, st, io_out_bf16());
}

}  // namespace

namespace {

// Implicit-GEMM convolution with im2col-mode TMA (see kIm2colPlan): A =
// output pixels [N*OH*OW][R*S*C] gathered by the TMA unit slab by slab (tap
// (x, y), channel chunk), B = the packed filter [Kout][R*S*C], the output
// [pixels][Kout] (NHWC) leaves through the TMA-store epilogue.
void launch_im2col_conv(const ConvGeom& g, const ConvPlan& c, const float* in, const float* filt,
                        float* out, char* ws, cudaStream_t st, bool prep, bool run) {
  const int esize = c.tf32 ? 4 : 2, ek = kSlabBytes / esize;
  const long long K = (long long)g.R * g.S * g.C;
  char* cursor = ws;
  void* ft = cursor;
  cursor += c.filt_bytes;
  float* part = reinterpret_cast<float*>(ws + c.filt_bytes + c.in_bytes);
  if (prep) {
    if (c.tf32) pack_filter<float>(filt, (int)K, g.K, (int)c.kp, (float*)ft, tf32_filter_rounding(), st);
    else pack_filter<__nv_bfloat16>(filt, (int)K, g.K, (int)c.kp, (__nv_bfloat16*)ft, false, st);
  }
  if (!run) return;
  const long long pix = (long long)g.N * g.OH * g.OW;
  const void* a = in;
  if (!c.tf32 && !io_in_bf16()) {
    to_bf16(in, (__nv_bfloat16*)cursor, (long long)g.N * g.H * g.W * g.C, st);
    a = cursor;
  }
  float* dst = c.splits > 1 ? part : out;
  const bool ob = io_out_bf16() && c.splits == 1;  // (split partials stay fp32)
  if (pix > 2147483647ll) fail(TK_ERR_CAPABILITY, "tc_conv: too many output pixels");
  TcArgs p{};
  p.M = (int)pix;
  p.N = g.K;
  p.K = (int)c.kp;
  p.BN = c.bn;
  p.ek = ek;
  p.num_m = c.num_m;
  p.num_n = c.num_n;
  p.batch = 1;
  p.num_kb = c.num_kb;
  p.splits = c.splits;
  p.kb_per = c.kb_per;
  p.d = out;
  p.d_sm = g.K;
  p.d_sn = 1;
  p.part = part;
  p.part_stride = pix * g.K;
  p.alpha = 1.0f;
  p.OH = g.OH;
  p.OW = g.OW;
  p.Kout = g.K;
  p.S = g.S;
  p.stride = g.stride;
  p.pad_t = g.pad_t;
  p.pad_l = g.pad_l;
  p.cchunks = g.C / ek;
  apply_tail(p, c.tail, reinterpret_cast<float*>(reinterpret_cast<char*>(part) + c.part_bytes));
  const CUtensorMap ma = map_nhwc_im2col(a, esize, g, kRows);
  const CUtensorMap mb = map_rows2d(ft, esize, c.kp, g.K, c.bn / c.cg);
  const CUtensorMap md = out_map_rows(dst, ob, g.K, pix, c.splits);
  p.out_bf16 = ob;
  p.store_tma = 1;
  p.epi_bufs = 2;
  dispatch<kConvIm2col>(ma, mb, md, p, c.cg, c.tf32, st);
  if (c.splits > 1) splitk_reduce(part, pix * g.K, c.splits, out, st, io_out_bf16());
}

ConvGeom tripled(const ConvGeom& g) {
  ConvGeom t = g;
  t.C = 3 * g.C;
  return t;
}
size_t split3_bytes_in(const ConvGeom& g) { return align256((size_t)g.N * g.H * g.W * g.C * 12); }
size_t split3_bytes_filt(const ConvGeom& g) { return align256((size_t)g.R * g.S * g.C * g.K * 12); }
}  // namespace

// Feature tile of the halo mode: 128 wide when the features come in 128s
// (N = 128 MMAs and half the units of N = 64: VGG conv2_1 105 -> 91 us,
// ResNet res3a/res4a_branch2b 27 -> 25 us, same-box A/B); two operand stages
// (halo 22.5 KiB + 9 filter taps x 8 KiB each) still fit.
static int halo_bn(const ConvGeom& g) {
  int bn = g.K <= 32 ? 32 : (g.K % 128 == 0 ? 128 : 64);
  const int b = experiments().halo_bn;
  if ((b == 64 || b == 128) && g.K % b == 0) bn = b;
  return bn;
}

// Halo mode keeps the CTA's filter slice resident in shared memory when it
// fits next to three halo stages and the feature blocks divide the SM pairs.
static bool halo_resident(const ConvGeom& g, int bn, int cchunks, int halo_bytes, int num_n) {
  const int cg = 2;
  const int b_bytes_h = (bn / cg) * kSlabBytes;
  const int fres = g.R * g.S * cchunks * b_bytes_h;
  const int epi = ((bn + 31) / 32) * kRows * kSlabBytes;
  const int left = 232448 - 2048 - epi - fres;
  const int units = sm_count() / cg;
  if (experiments().conv_mode == "halo_stream") return false;
  return left >= 3 * halo_bytes && units % num_n == 0;
}

// Columns per phase row of the narrow halo's phase-split input: the last
// output column's window + one spare box row of slack.
static int narrow_w2(const ConvGeom& g) { return g.OW + (g.S - 1) / g.stride + 16; }

// Narrow halo launch (TcArgs::narrow_taps + nphase): input padded to 16-byte
// pixels, filter packed in the (phase, row, column) tap order, one CTA-pair
// tile = 2 x 8 output rows of TW = 16 - (S-1)/s columns.
void launch_narrow_halo(const ConvGeom& g, const ConvPlan& c, const float* in, const float* filt,
                        float* out, char* ws, cudaStream_t st, bool prep, bool run) {
  const int esize = c.tf32 ? 4 : 2, ek = kSlabBytes / esize, cp = c.narrow_cp;
  const int s = g.stride;
  void* ft = ws;
  char* xin = ws + c.filt_bytes;
  if (prep) {
    const long long n = (long long)g.K * c.kp;
    const unsigned blocks = (unsigned)((n + 255) / 256);
    if (c.tf32)
      pack_filter_narrow_kernel<float><<<blocks, 256, 0, st>>>(
          filt, g.R, g.S, g.C, g.K, cp, (int)c.kp, s, (float*)ft, tf32_filter_rounding() ? 1 : 0);
    else
      pack_filter_narrow_kernel<__nv_bfloat16><<<blocks, 256, 0, st>>>(
          filt, g.R, g.S, g.C, g.K, cp, (int)c.kp, s, (__nv_bfloat16*)ft, 0);
    note_launch();
    TKB_CUDA(cudaGetLastError());
  }
  if (!run) return;
  const int W2 = narrow_w2(g);
  if ((long long)g.N * g.H * s > 2147483647ll) fail(TK_ERR_CAPABILITY, "narrow halo: too many rows");
  const unsigned pthreads = (unsigned)std::min(256, (W2 + 31) / 32 * 32);
  const int pblocks = (int)std::min<long long>((long long)g.N * g.H * s,
                                               (long long)sm_count() * (2048 / pthreads));
  if (c.tf32)
    launch_pdl(pad_phase_kernel<float, float>, (unsigned)pblocks, pthreads, st, in, g.N, g.H, g.W, g.C,
               s, W2, g.pad_l, cp, (float*)xin);
  else if (io_in_bf16())
    launch_pdl(pad_phase_kernel<__nv_bfloat16, __nv_bfloat16>, (unsigned)pblocks, pthreads, st,
               reinterpret_cast<const __nv_bfloat16*>(in), g.N, g.H, g.W, g.C, s, W2, g.pad_l, cp,
               (__nv_bfloat16*)xin);
  else
    launch_pdl(pad_phase_kernel<__nv_bfloat16, float>, (unsigned)pblocks, pthreads, st, in, g.N, g.H,
               g.W, g.C, s, W2, g.pad_l, cp, (__nv_bfloat16*)xin);
  const int cg = 2;
  TcArgs p{};
  p.P = kHaloPitch;
  p.TH = kRows / p.P;
  p.TW = p.P - (g.S - 1) / s;
  const int rows = p.TH + (g.R - 1) / s + 1;  // phase-box rows (one spare)
  p.nphase = s * s;
  p.phase_bytes = rows * p.P * 16;
  // The stage stride stays a multiple of 1024 bytes (every stage, the
  // resident filter and the epilogue staging behind them must keep the
  // 128-byte-swizzle atom alignment); the barrier expects halo_tx bytes.
  p.halo_tx = p.nphase * p.phase_bytes;
  p.halo_bytes = (p.halo_tx + 1023) / 1024 * 1024;
  p.narrow_taps = g.R * g.S;
  p.taps = (int)(c.kp / ek);  // filter slabs (8 taps each)
  p.K = (int)c.kp;
  p.ek = ek;
  p.cchunks = 1;
  p.num_kb = 1;
  p.BN = g.K <= 32 ? 32 : (g.K % 128 == 0 ? 128 : 64);
  p.Wb = p.TW;
  p.tileH = cg * p.TH;
  p.tiles_w = (g.OW + p.TW - 1) / p.TW;
  p.tiles_h = (g.OH + p.tileH - 1) / p.tileH;
  p.num_m = g.N * p.tiles_w * p.tiles_h;
  p.num_n = (g.K + p.BN - 1) / p.BN;
  p.M = p.num_m * kRows * cg;
  p.N = g.K;
  p.batch = 1;
  p.d = out;
  p.alpha = 1.0f;
  p.OH = g.OH;
  p.OW = g.OW;
  p.Kout = g.K;
  p.pad_t = g.pad_t;
  p.pad_l = g.pad_l;
  p.R = g.R;
  p.S = g.S;
  p.stride = s;
  p.C = cp;
  CUtensorMap ma;
  {
    // [N][H][s][W2 * cp] phase-split rows, box {16 pixels x cp, 1 phase,
    // rows (traversal s), 1}, no swizzle: one 256-byte run per box row.
    cuuint64_t dims[4] = {(cuuint64_t)W2 * cp, (cuuint64_t)s, (cuuint64_t)g.H, (cuuint64_t)g.N};
    cuuint64_t strides[3] = {(cuuint64_t)W2 * cp * esize, (cuuint64_t)s * W2 * cp * esize,
                             (cuuint64_t)g.H * s * W2 * cp * esize};
    cuuint32_t box[4] = {(cuuint32_t)(16 * cp), 1, (cuuint32_t)(rows * s), 1};
    const cuuint32_t trav[4] = {1, 1, (cuuint32_t)s, 1};
    ma = make_map(xin, esize, 4, dims, strides, box, s > 1 ? trav : nullptr,
                  CU_TENSOR_MAP_SWIZZLE_NONE);
  }
  const CUtensorMap mb = map_rows2d(ft, esize, c.kp, g.K, p.BN / cg);
  p.out_bf16 = io_out_bf16();
  const CUtensorMap md = out_map_nhwc(out, p.out_bf16, g, p.TW, p.TH);
  p.store_tma = 1;
  p.epi_bufs = 1;
  p.direct_store = p.out_bf16 ? 0 : experiments().direct_store;
  {
    const int b_bytes_h = (p.BN / cg) * kSlabBytes;
    const int fres = p.taps * b_bytes_h;
    const int epi = ((p.BN + 31) / 32) * kRows * kSlabBytes;
    const int left = 232448 - 2048 - epi - fres;
    p.resident = (left >= 3 * p.halo_bytes && (sm_count() / cg) % p.num_n == 0) ? 1 : 0;
  }
  dispatch<kConvHaloNarrow>(ma, mb, md, p, cg, c.tf32, st);
}

size_t tc_conv_workspace(const ConvGeom& g, int precision) {
  if (precision == TK_PREC_3XTF32)
  {
    Split3Scope s3;
    return split3_bytes_in(g) + split3_bytes_filt(g) + tc_conv_workspace(tripled(g), TK_PREC_TF32);
  }
  const ConvPlan c = plan_conv(g, precision);
  return c.filt_bytes + c.in_bytes + c.part_bytes + align256(c.tail.bytes);
}

void launch_tc_conv(const ConvGeom& g, const float* in, const float* filt, float* out,
                    int precision, void* ws, cudaStream_t st, int phase) {
  require_tc(precision);
  const bool prep = (phase & kConvPrepare) != 0, run = (phase & kConvRun) != 0;
  if (precision == TK_PREC_3XTF32) {
    // The same convolution over 3C channels: [x | x | x_lo] against
    // [f_hi | f_lo | f_hi], as one TF32 convolution (see split3_*).
    const ConvGeom g3 = tripled(g);
    Split3Scope s3;
    char* w = static_cast<char*>(ws);
    float* x3 = reinterpret_cast<float*>(w);
    float* f3 = reinterpret_cast<float*>(w + split3_bytes_in(g));
    void* inner = w + split3_bytes_in(g) + split3_bytes_filt(g);
    if (prep) {
      require_aligned(filt, "the filter");
      const long long n = (long long)g.R * g.S * g.C * g.K;
      const int blocks = (int)std::min<long long>((n + 255) / 256, (long long)sm_count() * 16);
      split3_filter_kernel<<<blocks, 256, 0, st>>>(filt, (long long)g.R * g.S, g.C, g.K, f3);
      note_launch();
      TKB_CUDA(cudaGetLastError());
      launch_tc_conv(g3, nullptr, f3, nullptr, TK_PREC_TF32, inner, st, kConvPrepare);
    }
    if (run) {
      const long long pix = (long long)g.N * g.H * g.W;
      const long long n = pix * g.C;
      const int blocks = (int)std::min<long long>((n + 255) / 256, (long long)sm_count() * 16);
      split3_channels_kernel<<<blocks, 256, 0, st>>>(in, pix, g.C, x3);
      note_launch();
      TKB_CUDA(cudaGetLastError());
      launch_tc_conv(g3, x3, f3, out, TK_PREC_TF32, inner, st, kConvRun);
    }
    return;
  }
  if (prep) require_aligned(filt, "the filter");
  if (run) {
    require_aligned(in, "the input");
    require_aligned(out, "the output");
  }
  const long long K = (long long)g.R * g.S * g.C;
  const ConvPlan plan = plan_conv(g, precision);
  const long long kp = plan.kp;
  char* cursor = static_cast<char*>(ws);
  if (plan.kind == kPointwisePlan) {
    launch_pointwise(g, plan, in, filt, out, cursor, st, prep, run);
    return;
  }
  if (plan.kind == kIm2colPlan) {
    launch_im2col_conv(g, plan, in, filt, out, cursor, st, prep, run);
    return;
  }
  if (plan.kind == kBoxPlan && plan.halo && plan.narrow_cp) {
    launch_narrow_halo(g, plan, in, filt, out, cursor, st, prep, run);
    return;
  }

  if (plan.kind == kGatherPlan) {
    if (tc_knobs().io != 0)
      fail(TK_ERR_CAPABILITY, "tc_conv: bf16 activations need a BF16 operand path (the gather "
                              "producers read fp32)");
    // Gather mode: the pixel operand is built in shared memory by producer
    // warps (any channel count / stride), the filter streams by TMA, the
    // output leaves through a TMA store.  fp32 operands, kind::tf32.
    float* ft = reinterpret_cast<float*>(cursor);
    if (prep) pack_filter<float>(filt, (int)K, g.K, (int)kp, ft, true, st);
    if (!run) return;
    const int pixels = g.N * g.OH * g.OW;
    // One SM per tile (cta_group::1): the gather producers then signal their
    // own CTA's barrier -- no cross-CTA release on every K-slab.
    const int cg = experiments().gather_cg;
    TcArgs p{};
    p.M = pixels;
    p.N = g.K;
    p.K = (int)kp;
    p.Kreal = (int)K;
    p.ek = 32;
    p.BN = std::min(128, (g.K + 16 * cg - 1) / (16 * cg) * (16 * cg));
    p.num_m = (pixels + kRows * cg - 1) / (kRows * cg);
    p.num_n = (g.K + p.BN - 1) / p.BN;
    p.batch = 1;
    p.num_kb = (int)(kp / 32);
    p.d = out;
    p.alpha = 1.0f;
    p.OH = g.OH;
    p.OW = g.OW;
    p.Kout = g.K;
    p.pad_t = g.pad_t;
    p.pad_l = g.pad_l;
    p.cchunks = 1;
    p.S = g.S;
    p.in = in;
    p.H = g.H;
    p.W = g.W;
    p.C = g.C;
    p.R = g.R;
    p.stride = g.stride;
    if (g.K % 4 != 0) fail(TK_ERR_CAPABILITY, "tc_conv: output features must be a multiple of 4");
    const CUtensorMap mb = map_rows2d(ft, 4, kp, g.K, p.BN / cg);
    cuuint64_t dims[3] = {(cuuint64_t)g.K, (cuuint64_t)pixels, 1};
    cuuint64_t strides[2] = {(cuuint64_t)g.K * 4, (cuuint64_t)g.K * pixels * 4};
    cuuint32_t boxd[3] = {32, (cuuint32_t)kRows, 1};
    const CUtensorMap md = make_map(out, 4, 3, dims, strides, boxd);
    p.store_tma = 1;
    p.epi_bufs = 2;
    dispatch<kConvGather>(mb, mb, md, p, cg, true, st);
    return;
  }

  const bool tf32 = precision == TK_PREC_TF32;
  const int esize = tf32 ? 4 : 2;
  const int ek = kSlabBytes / esize;
  const void* fa = nullptr;
  const void* xin = in;
  if (tf32) {
    float* ft = reinterpret_cast<float*>(cursor);
    if (prep) pack_filter<float>(filt, (int)K, g.K, (int)kp, ft, tf32_filter_rounding(), st);
    fa = ft;
  } else {
    __nv_bfloat16* ft = reinterpret_cast<__nv_bfloat16*>(cursor);
    cursor += align256((size_t)g.K * kp * 2);
    if (prep) pack_filter<__nv_bfloat16>(filt, (int)K, g.K, (int)kp, ft, false, st);
    __nv_bfloat16* xb = reinterpret_cast<__nv_bfloat16*>(cursor);
    if (run && !io_in_bf16()) to_bf16(in, xb, (long long)g.N * g.H * g.W * g.C, st);
    fa = ft;
    if (!io_in_bf16()) xin = xb;
  }

  float* part = reinterpret_cast<float*>(static_cast<char*>(ws) + plan.filt_bytes + plan.in_bytes);
  if (!run) return;
  const bool use_halo = plan.halo;
  if (use_halo) {
    const int cg = 2;
    TcArgs p{};
    p.P = kHaloPitch;
    p.TH = kRows / p.P;
    p.TW = p.P - (g.S - 1);
    p.taps = g.R * g.S;
    p.halo_bytes = (p.TH + g.R) * p.P * kSlabBytes;
    p.K = (int)K;
    p.ek = ek;
    p.cchunks = g.C / ek;
    p.num_kb = p.cchunks;
    // Feature tile: 128 wide when the features come in 128s (N = 128 MMAs
    // and half the units of N = 64: VGG conv2_1 105 -> 91 us, ResNet
    // res3a/res4a_branch2b 27 -> 25 us, same-box A/B); two operand stages
    // (halo 22.5 KiB + 9 filter taps x 8 KiB each) still fit.
    p.BN = halo_bn(g);
    p.Wb = p.TW;
    p.tileH = cg * p.TH;
    p.tiles_w = (g.OW + p.TW - 1) / p.TW;
    p.tiles_h = (g.OH + p.tileH - 1) / p.tileH;
    p.num_m = g.N * p.tiles_w * p.tiles_h;
    p.num_n = (g.K + p.BN - 1) / p.BN;
    p.M = p.num_m * kRows * cg;
    p.N = g.K;
    p.batch = 1;
    p.d = out;
    p.alpha = 1.0f;
    p.OH = g.OH;
    p.OW = g.OW;
    p.Kout = g.K;
    p.pad_t = g.pad_t;
    p.pad_l = g.pad_l;
    p.S = g.S;
    const CUtensorMap ma = map_nhwc(xin, esize, g, p.P, p.TH + g.R);
    const CUtensorMap mb = map_rows2d(fa, esize, kp, g.K, p.BN / cg);
    p.out_bf16 = io_out_bf16();
    const CUtensorMap md = out_map_nhwc(out, p.out_bf16, g, p.TW, p.TH);
    p.store_tma = 1;
    p.epi_bufs = 1;
    p.resident = halo_resident(g, p.BN, p.cchunks, p.halo_bytes, p.num_n) ? 1 : 0;
    dispatch<kConvHalo>(ma, mb, md, p, cg, tf32, st);
    return;
  }

  const bool pix_on_n = plan.pix_on_n;
  const int cg = plan.cg;
  const BoxShape bx = plan.bx;
  if (bx.wb == 0) fail(TK_ERR_CAPABILITY, "tc_conv: no pixel box fits this output plane");
  TcArgs p{};
  p.K = (int)K;
  p.ek = ek;
  p.num_kb = (int)(K / ek);
  p.batch = 1;
  p.d = out;
  p.alpha = 1.0f;
  p.OH = g.OH;
  p.OW = g.OW;
  p.Kout = g.K;
  p.Wb = bx.wb;
  p.tileH = bx.tileH;
  p.boxH = bx.boxH;
  p.tiles_w = bx.tiles_w;
  p.tiles_h = bx.tiles_h;
  p.pad_t = g.pad_t;
  p.pad_l = g.pad_l;
  p.cchunks = g.C / ek;
  p.S = g.S;
  p.stride = g.stride;
  p.imgs = plan.imgs;
  p.Nimg = g.N;
  p.flat = plan.flat ? 1 : 0;
  const int pix_tiles =
      plan.flat ? (int)(((long long)g.N * g.OH + bx.tileH - 1) / bx.tileH)
                : (g.N + plan.imgs - 1) / plan.imgs * bx.tiles_w * bx.tiles_h;
  if (pix_on_n) {
    p.BN = bx.wb * bx.tileH * plan.imgs;
    p.M = g.K;
    p.N = p.BN * pix_tiles;
    p.num_m = (g.K + kRows * cg - 1) / (kRows * cg);
    p.num_n = pix_tiles;
    p.splits = plan.splits;
    p.kb_per = plan.kb_per;
    p.part = part;
    p.part_stride = (long long)g.N * g.OH * g.OW * g.K;
    apply_tail(p, plan.tail, reinterpret_cast<float*>(reinterpret_cast<char*>(part) + plan.part_bytes));
    const CUtensorMap ma = map_rows2d(fa, esize, kp, g.K, kRows);
    const CUtensorMap mb =
        plan.imgs > 1 ? map_nhwc(xin, esize, g, bx.wb, bx.tileH, g.stride, plan.imgs / cg)
                      : map_nhwc(xin, esize, g, bx.wb, bx.boxH, g.stride);
    p.out_bf16 = io_out_bf16() && p.splits == 1;  // (split partials stay fp32)
    dispatch<kConvPixN>(ma, mb, ma, p, cg, tf32, st);
    if (p.splits > 1) splitk_reduce(part, p.part_stride, p.splits, out, st, io_out_bf16());
  } else {
    p.BN = (g.K + 16 * cg - 1) / (16 * cg) * (16 * cg);
    p.M = kRows * cg * pix_tiles;
    p.N = g.K;
    p.num_m = pix_tiles;
    p.num_n = 1;
    const CUtensorMap ma = map_nhwc(xin, esize, g, bx.wb, bx.boxH, g.stride);
    const CUtensorMap mb = map_rows2d(fa, esize, kp, g.K, p.BN / cg);
    if (g.K % 4 != 0) fail(TK_ERR_CAPABILITY, "tc_conv: output features must be a multiple of 4");
    p.out_bf16 = io_out_bf16();
    const CUtensorMap md = out_map_nhwc(out, p.out_bf16, g, bx.wb, bx.boxH);
    p.store_tma = 1;
    p.epi_bufs = 2;
    dispatch<kConvPixM>(ma, mb, md, p, cg, tf32, st);
  }
}

TcConvInfo tc_conv_info(const ConvGeom& g, int precision) {
  require_tc(precision);
  TcConvInfo r;
  if (precision == TK_PREC_3XTF32) {
    // One TF32 convolution over 3C channels ([x | x | x_lo] . [f_hi | f_lo | f_hi]).
    {
      Split3Scope s3;
      r = tc_conv_info(tripled(g), TK_PREC_TF32);
    }
    r.precision = TK_PREC_3XTF32;
    return r;
  }
  const ConvPlan c = plan_conv(g, precision);
  r.precision = c.tf32 ? TK_PREC_TF32 : TK_PREC_BF16;
  r.cta_group = c.cg;
  r.splits = c.splits;
  r.tail_pieces = c.tail.q > 1 ? c.tail.q : 0;
  switch (c.kind) {
    case kPointwisePlan:
    case kIm2colPlan:
      r.mode = c.kind == kPointwisePlan ? TK_TC_POINTWISE : TK_TC_IM2COL;
      r.tile_m = kRows * c.cg;
      r.tile_n = c.bn;
      break;
    case kGatherPlan:
      // fp32 operands built by the producer warps: kind::tf32 whatever the request.
      r.mode = TK_TC_GATHER;
      r.precision = TK_PREC_TF32;
      r.cta_group = experiments().gather_cg;
      r.tile_m = kRows * r.cta_group;
      r.tile_n = std::min(128, (g.K + 16 * r.cta_group - 1) / (16 * r.cta_group) * (16 * r.cta_group));
      r.splits = 1;
      r.tail_pieces = 0;
      break;
    default:
      if (c.halo) {
        const int ek = kSlabBytes / (c.tf32 ? 4 : 2);
        const int TH = kRows / 16, TW = 16 - (g.S - 1);
        const int bn = halo_bn(g);
        const int num_n = (g.K + bn - 1) / bn;
        r.mode = TK_TC_HALO;
        r.cta_group = 2;
        r.tile_m = kRows * 2;  // 2 x 8 rows of a pitch-16 halo (TW useful columns)
        r.tile_n = bn;
        r.box_w = TW;
        r.box_h = 2 * TH;
        r.halo_resident =
            c.narrow_cp ? 1
                        : (halo_resident(g, bn, g.C / ek, (TH + g.R) * 16 * kSlabBytes, num_n) ? 1 : 0);
        if (c.narrow_cp) {
          r.narrow = true;
          r.box_w = 16 - (g.S - 1) / g.stride;
          r.flat = 0;
        }
        r.splits = 1;
        r.tail_pieces = 0;
      } else if (c.pix_on_n) {
        r.mode = TK_TC_PIXN;
        r.tile_m = kRows * c.cg;
        r.tile_n = c.bx.wb * c.bx.tileH * c.imgs;
        r.imgs = c.imgs;
        r.flat = c.flat ? 1 : 0;
        r.box_w = c.bx.wb;
        r.box_h = c.bx.tileH;
      } else {
        r.mode = TK_TC_PIXM;
        r.tile_m = kRows * c.cg;
        r.tile_n = (g.K + 16 * c.cg - 1) / (16 * c.cg) * (16 * c.cg);
        r.box_w = c.bx.wb;
        r.box_h = c.bx.tileH;
      }
  }
  return r;
}

}  // namespace tkb

// tc_gemm.cu -- tcgen05 tensor-core GEMM and implicit-GEMM convolution.
//
// One persistent, warp-specialised kernel (192 threads, one CTA per SM):
//   warp 0      TMA producer: fills a STAGES-deep ring of 128-byte-swizzled
//               K-slabs (A: 128 rows, B: BN rows; 128 B = 32 fp32 of K each)
//   warp 1      MMA issuer: one elected thread issues 4 x tcgen05.mma
//               (kind::tf32, M=128, N=BN, K=8) per slab into a TMEM
//               accumulator; tcgen05.commit frees the slab / publishes the
//               accumulator
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> registers -> global, while the
//               MMA warp already accumulates the next tile into the second
//               TMEM buffer (2 x 256 columns)
// Operand sources:
//   plain GEMM : A [M][K], B [N][K] via 3-D TMA (K, rows, batch)
//   conv       : the filter, repacked once per call to [Kout][R*S*C], via 2-D
//                TMA; the activations via a 4-D TMA box {32 ch, Wb, Hb, 1}
//                of the NHWC input per (tap, channel chunk), shifted by the
//                tap offset.  Out-of-range rows/cols of the box are zero-
//                filled by the TMA unit, which is exactly Same padding.
// K order of the conv slabs is (x, y, c) like the reference's im2col
// (conv.hpp:286-292).
#include <cuda.h>

#include <mutex>
#include <string>

#include "common.cuh"
#include "tc_gemm.cuh"
#include "tc_ptx.cuh"

namespace tkb {

namespace {

constexpr int kBM = 128;
constexpr int kSlabBytes = 128;  // bytes of K per operand row per stage
constexpr int kThreads = 192;
constexpr int kAccCols = 256;
constexpr int kMaxStages = 8;

enum TcMode : int { kPlain = 0, kConvPixN = 1, kConvPixM = 2 };

struct TcArgs {
  int M, N, K;
  int BN;
  int num_m, num_n, batch, num_kb, stages;
  float* d;
  const float* c;
  long long d_sm, d_sn, d_batch;
  float alpha, beta;
  int read_c;
  // conv geometry
  int OH, OW, Kout, Wb, Hb, tiles_w, tiles_h, pad_t, pad_l, cchunks, S;
};

struct PixTile {
  int img, oh0, ow0;
};

__device__ __forceinline__ PixTile pix_tile(const TcArgs& p, int t) {
  PixTile r;
  const int per_img = p.tiles_w * p.tiles_h;
  r.img = t / per_img;
  const int rem = t - r.img * per_img;
  r.oh0 = (rem / p.tiles_w) * p.Hb;
  r.ow0 = (rem % p.tiles_w) * p.Wb;
  return r;
}

template <int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap map_a,
                   const __grid_constant__ CUtensorMap map_b, TcArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const int a_bytes = kBM * kSlabBytes;
  const int b_bytes = p.BN * kSlabBytes;
  const int stage_bytes = a_bytes + b_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(base + p.stages * stage_bytes);
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStages;
  uint64_t* tmem_full = bars + 2 * kMaxStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const uint32_t warp = ptx::warp_id(), lane = ptx::lane_id();
  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&map_a);
    ptx::prefetch_tmap(&map_b);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < p.stages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tmem_full[a], 1);
      ptx::mbar_init(&tmem_empty[a], 128);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<2 * kAccCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int total = p.num_m * p.num_n * p.batch;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (ptx::elect_one()) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < total; t += gridDim.x) {
        const int m_blk = t % p.num_m;
        const int rest = t / p.num_m;
        const int n_blk = rest % p.num_n;
        const int z = rest / p.num_n;
        PixTile pt{0, 0, 0};
        if constexpr (MODE == kConvPixN) pt = pix_tile(p, n_blk);
        if constexpr (MODE == kConvPixM) pt = pix_tile(p, m_blk);
        for (int kb = 0; kb < p.num_kb; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          uint8_t* sa = base + stage * stage_bytes;
          uint8_t* sb = sa + a_bytes;
          ptx::mbar_arrive_expect_tx(&full[stage], stage_bytes);
          const int k0 = kb * 32;
          int c0 = 0, dy = 0, dx = 0;
          if constexpr (MODE != kPlain) {
            const int tap = kb / p.cchunks;
            c0 = (kb - tap * p.cchunks) * 32;
            dy = tap % p.S - p.pad_l;
            dx = tap / p.S - p.pad_t;
          }
          if constexpr (MODE == kPlain) {
            ptx::tma_load_3d(sa, &map_a, &full[stage], k0, m_blk * kBM, z);
            ptx::tma_load_3d(sb, &map_b, &full[stage], k0, n_blk * p.BN, z);
          } else if constexpr (MODE == kConvPixN) {
            ptx::tma_load_2d(sa, &map_a, &full[stage], k0, m_blk * kBM);
            ptx::tma_load_4d(sb, &map_b, &full[stage], c0, pt.ow0 + dy, pt.oh0 + dx, pt.img);
          } else {
            ptx::tma_load_4d(sa, &map_a, &full[stage], c0, pt.ow0 + dy, pt.oh0 + dx, pt.img);
            ptx::tma_load_2d(sb, &map_b, &full[stage], k0, n_blk * p.BN);
          }
          if (++stage == p.stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = ptx::idesc(kBM, p.BN, true);
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      ptx::mbar_wait(&tmem_empty[acc], acc_phase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * kAccCols;
      for (int kb = 0; kb < p.num_kb; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          const uint32_t sa = ptx::smem(base + stage * stage_bytes);
          const uint32_t sb = sa + a_bytes;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            ptx::mma<true>(d_tmem, ptx::desc_sw128(sa + kk * 32), ptx::desc_sw128(sb + kk * 32),
                           idesc, (kb | kk) != 0);
          }
          ptx::mma_commit(&empty[stage]);
          if (kb == p.num_kb - 1) ptx::mma_commit(&tmem_full[acc]);
        }
        __syncwarp();
        if (++stage == p.stages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else {
    // ---------------- epilogue (warps 2..5) ----------------
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;
    int local = 0;
    for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
      const int m_blk = t % p.num_m;
      const int rest = t / p.num_m;
      const int n_blk = rest % p.num_n;
      const int z = rest / p.num_n;
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      ptx::mbar_wait(&tmem_full[acc], acc_phase);
      ptx::tc_fence_after();
      const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * kAccCols;

      if constexpr (MODE == kPlain) {
        const int m = m_blk * kBM + row;
        float* dz = p.d + (long long)z * p.d_batch;
        const float* cz = p.read_c ? p.c + (long long)z * p.d_batch : nullptr;
        for (int col = 0; col < p.BN; col += 32) {
          float v[32];
          ptx::tmem_ld32(taddr + col, v);
          if (m < p.M) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int n = n_blk * p.BN + col + j;
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
        const int m = m_blk * kBM + row;  // output feature
        const long long img_base = (long long)pt.img * p.OH;
        for (int col = 0; col < p.BN; col += 32) {
          float v[32];
          ptx::tmem_ld32(taddr + col, v);
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int n = col + j;
            const int oh = pt.oh0 + n / p.Wb, ow = pt.ow0 + n % p.Wb;
            if (n < p.BN && oh < p.OH && ow < p.OW && m < p.Kout)
              p.d[((img_base + oh) * p.OW + ow) * p.Kout + m] = v[j];
          }
        }
      } else {
        const PixTile pt = pix_tile(p, m_blk);
        const int oh = pt.oh0 + row / p.Wb, ow = pt.ow0 + row % p.Wb;
        const bool valid = oh < p.OH && ow < p.OW;
        float* dst = p.d + (((long long)pt.img * p.OH + oh) * p.OW + ow) * p.Kout;
        for (int col = 0; col < p.BN; col += 32) {
          float v[32];
          ptx::tmem_ld32(taddr + col, v);
          if (valid) {
            const int f0 = n_blk * p.BN + col;
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const int f = f0 + j;
              if (col + j + 3 < p.BN && f + 3 < p.Kout) {
                *reinterpret_cast<float4*>(dst + f) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
              } else {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  if (col + j + u < p.BN && f + u < p.Kout) dst[f + u] = v[j + u];
              }
            }
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tmem_empty[acc]);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<2 * kAccCols>(tmem_base);
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

CUtensorMap make_map(const float* base, int rank, const cuuint64_t* dims, const cuuint64_t* strides,
                     const cuuint32_t* box) {
  CUtensorMap m;
  cuuint32_t elem_strides[5] = {1, 1, 1, 1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank,
                                 const_cast<float*>(base), dims, strides, box, elem_strides,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(TK_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
  return m;
}

// [batch][rows][K] K-major operand, box {32, box_rows, 1}.
CUtensorMap map_rows(const float* base, long long K, long long rows, long long batch,
                     long long batch_stride, int box_rows) {
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)batch};
  cuuint64_t strides[2] = {(cuuint64_t)K * 4, (cuuint64_t)(batch_stride ? batch_stride : K * rows) * 4};
  cuuint32_t box[3] = {32, (cuuint32_t)box_rows, 1};
  return make_map(base, 3, dims, strides, box);
}

CUtensorMap map_rows2d(const float* base, long long K, long long rows, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)K * 4};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  return make_map(base, 2, dims, strides, box);
}

// NHWC activations, box {32 channels, Wb, Hb, 1}.
CUtensorMap map_nhwc(const float* base, const ConvGeom& g, int wb, int hb) {
  cuuint64_t dims[4] = {(cuuint64_t)g.C, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)g.N};
  cuuint64_t strides[3] = {(cuuint64_t)g.C * 4, (cuuint64_t)g.W * g.C * 4,
                           (cuuint64_t)g.H * g.W * g.C * 4};
  cuuint32_t box[4] = {32, (cuuint32_t)wb, (cuuint32_t)hb, 1};
  return make_map(base, 4, dims, strides, box);
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

template <int MODE>
void run_kernel(const CUtensorMap& ma, const CUtensorMap& mb, TcArgs p, int stages_req,
                cudaStream_t st) {
  const int stage_bytes = kBM * kSlabBytes + p.BN * kSlabBytes;
  const int budget = 232448 - 1024 - 256;
  int stages = budget / stage_bytes;
  if (stages > kMaxStages) stages = kMaxStages;
  if (stages_req > 0 && stages_req < stages) stages = stages_req;
  if (stages < 2) fail(TK_ERR_CAPABILITY, "tc_gemm: tile too large for shared memory");
  p.stages = stages;
  const size_t smem = 1024 + (size_t)stages * stage_bytes + 256;
  auto fn = tc_gemm_kernel<MODE>;
  TKB_CUDA(cudaFuncSetAttribute((const void*)fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)smem));
  const long long total = (long long)p.num_m * p.num_n * p.batch;
  const int grid = (int)(total < sm_count() ? total : sm_count());
  if (grid <= 0) return;
  fn<<<grid, kThreads, smem, st>>>(ma, mb, p);
  note_launch();
  TKB_CUDA(cudaGetLastError());
}

void require_tf32(int precision) {
  if (precision != TK_PREC_TF32)
    fail(TK_ERR_CAPABILITY, "tensor-core path: only TF32 is built in this version");
}

// ---- packing kernels ---------------------------------------------------------

// dst[r][kk] (row length kp, zero for kk >= k) = src[r*rs + kk*ks].
__global__ void __launch_bounds__(256) pack_kmajor_kernel(const float* __restrict__ src,
                                                          long long rs, long long ks, long long rows,
                                                          long long k, long long kp,
                                                          float* __restrict__ dst) {
  __shared__ float tile[32][33];
  const long long r0 = (long long)blockIdx.y * 32, k0 = (long long)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  if (ks == 1) {
    for (int i = ty; i < 32; i += 8) {
      const long long r = r0 + i, kk = k0 + tx;
      tile[i][tx] = (r < rows && kk < k) ? src[r * rs + kk] : 0.0f;
    }
  } else {
    for (int i = ty; i < 32; i += 8) {
      const long long r = r0 + tx, kk = k0 + i;
      tile[tx][i] = (r < rows && kk < k) ? src[r * rs + kk * ks] : 0.0f;
    }
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const long long r = r0 + i, kk = k0 + tx;
    if (r < rows && kk < kp) dst[r * kp + kk] = tile[i][tx];
  }
}

void pack_kmajor(const float* src, long long rs, long long ks, long long rows, long long k,
                 long long kp, float* dst, cudaStream_t st) {
  dim3 grid((unsigned)((kp + 31) / 32), (unsigned)((rows + 31) / 32));
  if (grid.y > 65535) fail(TK_ERR_CAPABILITY, "pack: too many rows");
  pack_kmajor_kernel<<<grid, dim3(32, 8), 0, st>>>(src, rs, ks, rows, k, kp, dst);
  note_launch();
  TKB_CUDA(cudaGetLastError());
}

// Row-major patch matrix [pixel][kp] (K-major, zero padded to kp), the
// explicit fallback for channel counts TMA cannot box (C % 32 != 0) and
// strides != 1.
__global__ void __launch_bounds__(256) patches_rm_kernel(ConvGeom g, const float* __restrict__ in,
                                                         long long kp, float* __restrict__ out) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long pixels = (long long)g.N * g.OH * g.OW;
  if (idx >= pixels * kp) return;
  const long long pix = idx / kp;
  const int kk = (int)(idx - pix * kp);
  const int K = g.R * g.S * g.C;
  float v = 0.0f;
  if (kk < K) {
    const int c = kk % g.C, tap = kk / g.C;
    const int y = tap % g.S, x = tap / g.S;
    const int ow = (int)(pix % g.OW);
    const long long t = pix / g.OW;
    const int oh = (int)(t % g.OH);
    const long long n = t / g.OH;
    const int ih = oh * g.stride + x - g.pad_t, iw = ow * g.stride + y - g.pad_l;
    if (ih >= 0 && iw >= 0 && ih < g.H && iw < g.W) v = __ldg(in + ((n * g.H + ih) * g.W + iw) * g.C + c);
  }
  out[idx] = v;
}

// Pixel-tile shape for the conv box: Wb * Hb pixels.
struct BoxShape {
  int wb, hb, tiles_w, tiles_h;
};

BoxShape pick_box(const ConvGeom& g, bool pix_on_n) {
  BoxShape best{0, 0, 0, 0};
  double best_score = 1e30;
  for (int wb = 1; wb <= 256; ++wb) {
    for (int hb = 1; wb * hb <= 256; ++hb) {
      const int P = wb * hb;
      if (pix_on_n ? (P % 16 != 0 || P < 64) : (P != kBM)) continue;
      if (wb > 2 * g.OW + 16 || hb > 2 * g.OH + 16) continue;
      const int tw = (g.OW + wb - 1) / wb, th = (g.OH + hb - 1) / hb;
      const double waste = (double)tw * wb * th * hb / ((double)g.OW * g.OH);
      const double score = waste * (1.0 + 24.0 / P);
      if (score < best_score - 1e-9) {
        best_score = score;
        best = BoxShape{wb, hb, tw, th};
      }
    }
  }
  return best;
}

}  // namespace

void launch_tc_gemm(const TcGemm& g, cudaStream_t st) {
  require_tf32(g.precision);
  if (g.K % 4 != 0) fail(TK_ERR_CAPABILITY, "tc_gemm: K must be a multiple of 4 (pack first)");
  int bn = g.tile_n > 0 ? g.tile_n : (g.N >= 256 ? 256 : ((g.N + 15) / 16) * 16);
  if (bn > 256) bn = 256;
  if (bn < 16) bn = 16;
  bn = (bn + 15) / 16 * 16;
  TcArgs p{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.BN = bn;
  p.num_m = (g.M + kBM - 1) / kBM;
  p.num_n = (g.N + bn - 1) / bn;
  p.batch = g.batch;
  p.num_kb = (g.K + 31) / 32;
  p.d = g.d;
  p.c = g.c;
  p.d_sm = g.d_sm;
  p.d_sn = g.d_sn;
  p.d_batch = g.d_batch;
  p.alpha = g.alpha;
  p.beta = g.beta;
  p.read_c = g.c != nullptr && g.beta != 0.0f;
  const CUtensorMap ma = map_rows(g.a, g.K, g.M, g.batch, g.a_batch, kBM);
  const CUtensorMap mb = map_rows(g.b, g.K, g.N, g.batch, g.b_batch, bn);
  run_kernel<kPlain>(ma, mb, p, 0, st);
}

void launch_tc_colmajor_gemm(size_t m, size_t n, size_t k, float alpha, float beta, bool ta,
                             bool tb, const float* a, const float* b, const float* c, float* d,
                             int precision, int tile_n, cudaStream_t st) {
  require_tf32(precision);
  const long long kp = (long long)((k + 3) / 4 * 4);
  // A as [m][k]: stored k x m (transposed) is already K-major.
  const bool a_ok = ta && kp == (long long)k;
  const bool b_ok = !tb && kp == (long long)k;
  float* pa = nullptr;
  float* pb = nullptr;
  if (!a_ok) TKB_CUDA(cudaMallocAsync(&pa, (size_t)m * kp * 4, st));
  if (!b_ok) TKB_CUDA(cudaMallocAsync(&pb, (size_t)n * kp * 4, st));
  if (!a_ok) {
    if (ta) pack_kmajor(a, (long long)k, 1, (long long)m, (long long)k, kp, pa, st);
    else pack_kmajor(a, 1, (long long)m, (long long)m, (long long)k, kp, pa, st);
  }
  if (!b_ok) {
    if (tb) pack_kmajor(b, 1, (long long)n, (long long)n, (long long)k, kp, pb, st);
    else pack_kmajor(b, (long long)k, 1, (long long)n, (long long)k, kp, pb, st);
  }
  TcGemm g;
  g.M = (int)m;
  g.N = (int)n;
  g.K = (int)kp;
  g.a = a_ok ? a : pa;
  g.b = b_ok ? b : pb;
  g.d = d;
  g.c = c;
  g.d_sm = 1;
  g.d_sn = (long long)m;
  g.alpha = alpha;
  g.beta = beta;
  g.precision = precision;
  g.tile_n = tile_n;
  launch_tc_gemm(g, st);
  if (pa) cudaFreeAsync(pa, st);
  if (pb) cudaFreeAsync(pb, st);
}

namespace {

bool conv_boxable(const ConvGeom& g) { return g.C % 32 == 0 && g.stride == 1; }

long long conv_kp(const ConvGeom& g) {
  const long long K = (long long)g.R * g.S * g.C;
  return conv_boxable(g) ? K : (K + 31) / 32 * 32;
}

}  // namespace

size_t tc_conv_workspace(const ConvGeom& g, int precision) {
  (void)precision;
  const long long kp = conv_kp(g);
  size_t bytes = ((size_t)g.K * kp * 4 + 255) / 256 * 256;
  if (!conv_boxable(g)) bytes += (size_t)g.N * g.OH * g.OW * kp * 4;
  return bytes;
}

void launch_tc_conv(const ConvGeom& g, const float* in, const float* filt, float* out,
                    int precision, void* ws, cudaStream_t st) {
  require_tf32(precision);
  const long long K = (long long)g.R * g.S * g.C;
  const long long kp = conv_kp(g);
  float* ft = static_cast<float*>(ws);
  // Filter HWCK = [K][Kout] -> [Kout][kp] (K-major, zero padded).
  pack_kmajor(filt, 1, g.K, g.K, K, kp, ft, st);

  if (!conv_boxable(g)) {
    // Explicit patch matrix + plain GEMM: D(feature, pixel) -> NHWC.
    float* patches = reinterpret_cast<float*>(static_cast<char*>(ws) +
                                              ((size_t)g.K * kp * 4 + 255) / 256 * 256);
    const long long pixels = (long long)g.N * g.OH * g.OW;
    const long long n = pixels * kp;
    patches_rm_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(g, in, kp, patches);
    note_launch();
    TKB_CUDA(cudaGetLastError());
    TcGemm t;
    t.M = g.K;
    t.N = (int)pixels;
    t.K = (int)kp;
    t.a = ft;
    t.b = patches;
    t.d = out;
    t.d_sm = 1;
    t.d_sn = g.K;
    t.precision = precision;
    launch_tc_gemm(t, st);
    return;
  }

  const bool pix_on_n = g.K >= kBM;
  const BoxShape box = pick_box(g, pix_on_n);
  if (box.wb == 0) fail(TK_ERR_CAPABILITY, "tc_conv: no pixel box fits this output plane");
  TcArgs p{};
  p.K = (int)K;
  p.num_kb = (int)(K / 32);
  p.batch = 1;
  p.d = out;
  p.alpha = 1.0f;
  p.OH = g.OH;
  p.OW = g.OW;
  p.Kout = g.K;
  p.Wb = box.wb;
  p.Hb = box.hb;
  p.tiles_w = box.tiles_w;
  p.tiles_h = box.tiles_h;
  p.pad_t = g.pad_t;
  p.pad_l = g.pad_l;
  p.cchunks = g.C / 32;
  p.S = g.S;
  const int pix_tiles = g.N * box.tiles_w * box.tiles_h;
  if (pix_on_n) {
    p.BN = box.wb * box.hb;
    p.M = g.K;
    p.N = p.BN * pix_tiles;
    p.num_m = (g.K + kBM - 1) / kBM;
    p.num_n = pix_tiles;
    const CUtensorMap ma = map_rows2d(ft, kp, g.K, kBM);
    const CUtensorMap mb = map_nhwc(in, g, box.wb, box.hb);
    run_kernel<kConvPixN>(ma, mb, p, 0, st);
  } else {
    p.BN = (g.K + 15) / 16 * 16;
    p.M = kBM * pix_tiles;
    p.N = g.K;
    p.num_m = pix_tiles;
    p.num_n = 1;
    const CUtensorMap ma = map_nhwc(in, g, box.wb, box.hb);
    const CUtensorMap mb = map_rows2d(ft, kp, g.K, p.BN);
    run_kernel<kConvPixM>(ma, mb, p, 0, st);
  }
}

}  // namespace tkb

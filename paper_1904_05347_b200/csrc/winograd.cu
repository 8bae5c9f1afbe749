// winograd.cu -- Cook-Toom F(2x2,3x3) / F(4x4,3x3) transform kernels.
//
// Reference: conv2d_winograd (winograd.hpp:169-301) with transform_tile
// (winograd.hpp:125-147) and the plans of winograd_plan (winograd.hpp:50-119).
//
// Each transform reproduces transform_tile's arithmetic exactly: pass 1
// tmp = T*src, pass 2 dst = tmp*T^T, every sum started at +0 and updated
// with separately rounded multiply and add in ascending k.  Terms whose
// coefficient is exactly 0 are skipped: for finite data they add a signed
// zero to a running sum that can never be -0, which leaves the bits
// unchanged.  The batched GEMM between the transforms runs on the exact
// SIMT kernel (or the tensor-core kernel for TF32), so the FP32 path is
// bit-identical to the reference.
//
// Transform-domain layouts are chosen for coalescing on B200 (the reference
// layout is internal to conv2d_winograd and not observable):
//   V[spot][tile][C]   input transform output   (C contiguous)
//   U[spot][C][K]      filter transform output  (K contiguous, exact path)
//   Ut[spot][K][C]     filter transform output  (C contiguous, tensor cores)
//   P[spot][tile][K]   batched GEMM output      (K contiguous)
// Every kernel is HBM-bound; its roofline is bytes moved / HBM bandwidth.
#include "common.cuh"
#include "winograd.cuh"

namespace tkb {

namespace {

// Plans, row-major, the reference's float constants (winograd.hpp:62-107).
struct F2 {
  static constexpr int M = 2, T = 4;
  static __device__ __forceinline__ constexpr float bt(int i) {
    constexpr float v[] = {1, 0, -1, 0, 0, 1, 1, 0, 0, -1, 1, 0, 0, 1, 0, -1};
    return v[i];
  }
  static __device__ __forceinline__ constexpr float g(int i) {
    constexpr float v[] = {1, 0, 0, 0.5f, 0.5f, 0.5f, 0.5f, -0.5f, 0.5f, 0, 0, 1};
    return v[i];
  }
  static __device__ __forceinline__ constexpr float at(int i) {
    constexpr float v[] = {1, 1, 1, 0, 0, 1, -1, -1};
    return v[i];
  }
};
struct F4 {
  static constexpr int M = 4, T = 6;
  static __device__ __forceinline__ constexpr float bt(int i) {
    constexpr float v[] = {4, 0, -5, 0,  1, 0, 0, -4, -4, 1,  1, 0,
                                   0, 4, -4, -1, 1, 0, 0, -2, -1, 2,  1, 0,
                                   0, 2, -1, -2, 1, 0, 0, 4,  0,  -5, 0, 1};
    return v[i];
  }
  static __device__ __forceinline__ constexpr float g(int i) {
    constexpr float v[] = {1.0f / 4,  0,          0,         -1.0f / 6, -1.0f / 6, -1.0f / 6,
                                  -1.0f / 6, 1.0f / 6,   -1.0f / 6, 1.0f / 24, 1.0f / 12, 1.0f / 6,
                                  1.0f / 24, -1.0f / 12, 1.0f / 6,  0,         0,         1};
    return v[i];
  }
  static __device__ __forceinline__ constexpr float at(int i) {
    constexpr float v[] = {1, 1, 1, 1, 1, 0, 0, 1, -1, 2, -2, 0,
                                   0, 1, 1, 4, 4, 0, 0, 1, -1, 8, -8, 1};
    return v[i];
  }
};

// dst (P x P) = T (P x Q) * src (Q x Q) * T^T, transform_tile's two passes.
template <int P, int Q, typename CoefFn>
__device__ __forceinline__ void transform(CoefFn t, const float* src, float* dst) {
  float tmp[P * Q];
#pragma unroll
  for (int i = 0; i < P; ++i)
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      float sum = 0.0f;
#pragma unroll
      for (int k = 0; k < Q; ++k)
        if (t(i, k) != 0.0f) sum = __fadd_rn(sum, __fmul_rn(t(i, k), src[k * Q + j]));
      tmp[i * Q + j] = sum;
    }
#pragma unroll
  for (int i = 0; i < P; ++i)
#pragma unroll
    for (int j = 0; j < P; ++j) {
      float sum = 0.0f;
#pragma unroll
      for (int k = 0; k < Q; ++k)
        if (t(j, k) != 0.0f) sum = __fadd_rn(sum, __fmul_rn(tmp[i * Q + k], t(j, k)));
      dst[i * P + j] = sum;
    }
}

// Stage 1 (winograd.hpp:197-237): one thread per (tile, channel), channel
// fastest so both the NHWC reads and the V writes coalesce.
template <class Plan>
__global__ void __launch_bounds__(256) wino_input_kernel(WinoGeom g, const float* __restrict__ in,
                                                         float* __restrict__ v) {
  constexpr int T = Plan::T, M = Plan::M;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)g.tiles * g.C;
  if (idx >= total) return;
  const int c = (int)(idx % g.C);
  const int tile = (int)(idx / g.C);
  const int tj = tile % g.tiles_c;
  const int ti = (tile / g.tiles_c) % g.tiles_r;
  const int b = tile / (g.tiles_c * g.tiles_r);
  const int r0 = ti * M - g.pad_t, c0 = tj * M - g.pad_l;
  float patch[T * T];
#pragma unroll
  for (int i = 0; i < T; ++i) {
    const int ih = r0 + i;
#pragma unroll
    for (int j = 0; j < T; ++j) {
      const int iw = c0 + j;
      const bool inside = ih >= 0 && iw >= 0 && ih < g.H && iw < g.W;
      patch[i * T + j] = inside ? __ldg(in + (((long long)b * g.H + ih) * g.W + iw) * g.C + c) : 0.0f;
    }
  }
  float out[T * T];
  transform<T, T>([](int i, int k) { return Plan::bt(i * T + k); }, patch, out);
  const long long plane = (long long)g.tiles * g.C;
#pragma unroll
  for (int s = 0; s < T * T; ++s) v[s * plane + (long long)tile * g.C + c] = out[s];
}

// Stage 2 (winograd.hpp:239-259): one thread per (channel, feature).
// k_major = 0 writes U[s][c][k]; 1 writes Ut[s][k][c].  The index order
// follows the written layout (feature fastest for U, channel fastest for
// Ut): the T^2 = 16 / 36 stores per thread coalesce, the 9 filter reads are
// the strided side.
template <class Plan>
__global__ void __launch_bounds__(256) wino_filter_kernel(WinoGeom g, const float* __restrict__ filt,
                                                          float* __restrict__ u, int k_major) {
  constexpr int T = Plan::T;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)g.C * g.K) return;
  const int k = k_major ? (int)(idx / g.C) : (int)(idx % g.K);
  const int c = k_major ? (int)(idx % g.C) : (int)(idx / g.K);
  float w[9];
#pragma unroll
  for (int x = 0; x < 3; ++x)
#pragma unroll
    for (int y = 0; y < 3; ++y) w[x * 3 + y] = __ldg(filt + ((long long)(x * 3 + y) * g.C + c) * g.K + k);
  float out[T * T];
  transform<T, 3>([](int i, int kk) { return Plan::g(i * 3 + kk); }, w, out);
  const long long plane = (long long)g.C * g.K;
  const long long off = k_major ? (long long)k * g.C + c : (long long)c * g.K + k;
#pragma unroll
  for (int s = 0; s < T * T; ++s) u[s * plane + off] = out[s];
}

// Stage 4 (winograd.hpp:267-294): one thread per (tile, feature), feature
// fastest; gathers the T*T products, applies A^T M A, writes the clipped
// M x M block of NHWC output.
template <class Plan>
__global__ void __launch_bounds__(256) wino_output_kernel(WinoGeom g, const float* __restrict__ prod,
                                                          float* __restrict__ out) {
  constexpr int T = Plan::T, M = Plan::M;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)g.tiles * g.K) return;
  const int k = (int)(idx % g.K);
  const int tile = (int)(idx / g.K);
  const int tj = tile % g.tiles_c;
  const int ti = (tile / g.tiles_c) % g.tiles_r;
  const int b = tile / (g.tiles_c * g.tiles_r);
  const long long plane = (long long)g.tiles * g.K;
  float gathered[T * T];
#pragma unroll
  for (int s = 0; s < T * T; ++s) gathered[s] = __ldg(prod + s * plane + (long long)tile * g.K + k);
  float res[M * M];
  transform<M, T>([](int i, int kk) { return Plan::at(i * T + kk); }, gathered, res);
  const int rh = min(M, g.OH - ti * M), cw = min(M, g.OW - tj * M);
#pragma unroll
  for (int i = 0; i < M; ++i) {
    if (i >= rh) break;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      if (j >= cw) break;
      out[(((long long)b * g.OH + ti * M + i) * g.OW + tj * M + j) * g.K + k] = res[i * M + j];
    }
  }
}

// Vectorised stage 1 / stage 4: V channels (V = 4 for F(2x2), 2 for
// F(4x4): 16 x float4 / 36 x float2 patches stay in registers) per thread,
// 16- / 8-byte loads and stores along C (input) or K (output).  Same
// per-element arithmetic as the scalar kernels (transform_tile's two
// passes, lane by lane), so the bits are the same.
template <int V>
struct VecT;
template <>
struct VecT<4> {
  using type = float4;
  static __device__ __forceinline__ float get(const float4& v, int i) {
    return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w;
  }
  static __device__ __forceinline__ void set(float4& v, int i, float x) {
    if (i == 0) v.x = x;
    else if (i == 1) v.y = x;
    else if (i == 2) v.z = x;
    else v.w = x;
  }
};
template <>
struct VecT<2> {
  using type = float2;
  static __device__ __forceinline__ float get(const float2& v, int i) { return i == 0 ? v.x : v.y; }
  static __device__ __forceinline__ void set(float2& v, int i, float x) {
    if (i == 0) v.x = x;
    else v.y = x;
  }
};

template <class Plan, int V>
__global__ void __launch_bounds__(256) wino_input_vec_kernel(WinoGeom g, const float* __restrict__ in,
                                                             float* __restrict__ v) {
  using VT = typename VecT<V>::type;
  constexpr int T = Plan::T, M = Plan::M;
  const int cv = g.C / V;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)g.tiles * cv) return;
  const int c = (int)(idx % cv) * V;
  const int tile = (int)(idx / cv);
  const int tj = tile % g.tiles_c;
  const int ti = (tile / g.tiles_c) % g.tiles_r;
  const int b = tile / (g.tiles_c * g.tiles_r);
  const int r0 = ti * M - g.pad_t, c0 = tj * M - g.pad_l;
  VT patch[T * T];
#pragma unroll
  for (int i = 0; i < T; ++i) {
    const int ih = r0 + i;
#pragma unroll
    for (int j = 0; j < T; ++j) {
      const int iw = c0 + j;
      const bool inside = ih >= 0 && iw >= 0 && ih < g.H && iw < g.W;
      VT z{};
      patch[i * T + j] =
          inside ? __ldg(reinterpret_cast<const VT*>(in + (((long long)b * g.H + ih) * g.W + iw) * g.C + c))
                 : z;
    }
  }
  const long long plane = (long long)g.tiles * g.C;
  VT res[T * T];
#pragma unroll
  for (int lane = 0; lane < V; ++lane) {
    float src[T * T], out[T * T];
#pragma unroll
    for (int q = 0; q < T * T; ++q) src[q] = VecT<V>::get(patch[q], lane);
    transform<T, T>([](int i, int k) { return Plan::bt(i * T + k); }, src, out);
#pragma unroll
    for (int q = 0; q < T * T; ++q) VecT<V>::set(res[q], lane, out[q]);
  }
#pragma unroll
  for (int q = 0; q < T * T; ++q)
    __stcs(reinterpret_cast<VT*>(v + q * plane + (long long)tile * g.C + c), res[q]);
}

template <class Plan, int V>
__global__ void __launch_bounds__(256) wino_output_vec_kernel(WinoGeom g, const float* __restrict__ prod,
                                                              float* __restrict__ out) {
  using VT = typename VecT<V>::type;
  constexpr int T = Plan::T, M = Plan::M;
  const int kv = g.K / V;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long long)g.tiles * kv) return;
  const int k = (int)(idx % kv) * V;
  const int tile = (int)(idx / kv);
  const int tj = tile % g.tiles_c;
  const int ti = (tile / g.tiles_c) % g.tiles_r;
  const int b = tile / (g.tiles_c * g.tiles_r);
  const long long plane = (long long)g.tiles * g.K;
  VT gathered[T * T];
#pragma unroll
  for (int q = 0; q < T * T; ++q)
    gathered[q] = __ldcs(reinterpret_cast<const VT*>(prod + q * plane + (long long)tile * g.K + k));
  VT res[M * M];
#pragma unroll
  for (int lane = 0; lane < V; ++lane) {
    float src[T * T], o[M * M];
#pragma unroll
    for (int q = 0; q < T * T; ++q) src[q] = VecT<V>::get(gathered[q], lane);
    transform<M, T>([](int i, int kk) { return Plan::at(i * T + kk); }, src, o);
#pragma unroll
    for (int q = 0; q < M * M; ++q) VecT<V>::set(res[q], lane, o[q]);
  }
  const int rh = min(M, g.OH - ti * M), cw = min(M, g.OW - tj * M);
#pragma unroll
  for (int i = 0; i < M; ++i) {
    if (i >= rh) break;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      if (j >= cw) break;
      *reinterpret_cast<VT*>(out + (((long long)b * g.OH + ti * M + i) * g.OW + tj * M + j) * g.K + k) =
          res[i * M + j];
    }
  }
}

inline unsigned blocks_for(long long n, int threads) { return (unsigned)((n + threads - 1) / threads); }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

void wino_input_transform(const WinoGeom& g, const float* d_in, float* d_v, cudaStream_t st) {
  const long long n = (long long)g.tiles * g.C;
  const bool vec = aligned16(d_in) && aligned16(d_v);
  if (g.m == 2 && vec && g.C % 4 == 0)
    wino_input_vec_kernel<F2, 4><<<blocks_for(n / 4, 256), 256, 0, st>>>(g, d_in, d_v);
  else if (g.m == 4 && vec && g.C % 2 == 0)
    wino_input_vec_kernel<F4, 2><<<blocks_for(n / 2, 256), 256, 0, st>>>(g, d_in, d_v);
  else if (g.m == 2) wino_input_kernel<F2><<<blocks_for(n, 256), 256, 0, st>>>(g, d_in, d_v);
  else wino_input_kernel<F4><<<blocks_for(n, 256), 256, 0, st>>>(g, d_in, d_v);
  note_launch();
  TKB_CUDA(cudaGetLastError());
}

void wino_filter_transform(const WinoGeom& g, const float* d_filt, float* d_u, bool k_major,
                           cudaStream_t st) {
  const long long n = (long long)g.C * g.K;
  if (g.m == 2) wino_filter_kernel<F2><<<blocks_for(n, 256), 256, 0, st>>>(g, d_filt, d_u, k_major);
  else wino_filter_kernel<F4><<<blocks_for(n, 256), 256, 0, st>>>(g, d_filt, d_u, k_major);
  note_launch();
  TKB_CUDA(cudaGetLastError());
}

void wino_output_transform(const WinoGeom& g, const float* d_prod, float* d_out, cudaStream_t st) {
  const long long n = (long long)g.tiles * g.K;
  const bool vec = aligned16(d_prod) && aligned16(d_out);
  if (g.m == 2 && vec && g.K % 4 == 0)
    wino_output_vec_kernel<F2, 4><<<blocks_for(n / 4, 256), 256, 0, st>>>(g, d_prod, d_out);
  else if (g.m == 4 && vec && g.K % 2 == 0)
    wino_output_vec_kernel<F4, 2><<<blocks_for(n / 2, 256), 256, 0, st>>>(g, d_prod, d_out);
  else if (g.m == 2) wino_output_kernel<F2><<<blocks_for(n, 256), 256, 0, st>>>(g, d_prod, d_out);
  else wino_output_kernel<F4><<<blocks_for(n, 256), 256, 0, st>>>(g, d_prod, d_out);
  note_launch();
  TKB_CUDA(cudaGetLastError());
}

}  // namespace tkb

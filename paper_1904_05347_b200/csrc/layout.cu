// layout.cu -- HBM-bound layout kernels: explicit im2col, filter_matrix and
// the operand transposes that feed the tensor-core GEMM.
//
// im2col (conv.hpp:255-300) writes the column-major patch matrix
// (N*OH*OW) x (R*S*C): row (n*OH+oh)*OW+ow, column (x*S+y)*C+c, zero outside
// the input.  Reads run along columns (channels of one tap are contiguous
// in NHWC), writes along rows (column-major), so each 32x32 tile goes
// through a padded shared-memory transpose and both sides coalesce.
#include "common.cuh"
#include "layout.cuh"

namespace tkb {

namespace {

__global__ void __launch_bounds__(256) im2col_kernel(ConvGeom g, const float* __restrict__ in,
                                                     float* __restrict__ out, long long rows,
                                                     int cols) {
  __shared__ float tile[32][33];
  const long long r0 = (long long)blockIdx.x * 32;
  const int c0 = blockIdx.y * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  // Load: tx runs along columns (k), ty along rows (pixels).
  const int k = c0 + tx;
  int x = 0, y = 0, c = 0;
  if (k < cols) {
    c = k % g.C;
    const int tap = k / g.C;
    y = tap % g.S;
    x = tap / g.S;
  }
  for (int i = ty; i < 32; i += 8) {
    const long long row = r0 + i;
    float v = 0.0f;
    if (row < rows && k < cols) {
      const int ow = (int)(row % g.OW);
      const long long t = row / g.OW;
      const int oh = (int)(t % g.OH);
      const long long n = t / g.OH;
      const int ih = oh * g.stride + x - g.pad_t;
      const int iw = ow * g.stride + y - g.pad_l;
      if (ih >= 0 && iw >= 0 && ih < g.H && iw < g.W)
        v = __ldg(in + ((n * g.H + ih) * g.W + iw) * g.C + c);
    }
    tile[i][tx] = v;
  }
  __syncthreads();
  // Store: tx runs along rows (contiguous in column-major), ty along columns.
  const long long row = r0 + tx;
  for (int j = ty; j < 32; j += 8) {
    const int col = c0 + j;
    if (row < rows && col < cols) out[row + (long long)col * rows] = tile[tx][j];
  }
}

// Generic 2-D transpose: dst[j*ld_dst + i] = src[i*ld_src + j], i < rows,
// j < cols (filter_matrix is the HWCK (rows = R*S*C, cols = K) instance).
__global__ void __launch_bounds__(256) transpose_kernel(const float* __restrict__ src,
                                                        float* __restrict__ dst, long long rows,
                                                        long long cols) {
  __shared__ float tile[32][33];
  const long long i0 = (long long)blockIdx.y * 32, j0 = (long long)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int r = ty; r < 32; r += 8) {
    const long long i = i0 + r, j = j0 + tx;
    tile[r][tx] = (i < rows && j < cols) ? __ldg(src + i * cols + j) : 0.0f;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const long long j = j0 + r, i = i0 + tx;
    if (i < rows && j < cols) dst[j * rows + i] = tile[tx][r];
  }
}

}  // namespace

void launch_im2col(const ConvGeom& g, const float* d_in, float* d_patches, cudaStream_t st) {
  const long long rows = (long long)g.N * g.OH * g.OW;
  const int cols = g.R * g.S * g.C;
  dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((cols + 31) / 32));
  if (grid.y > 65535) fail(TK_ERR_CAPABILITY, "im2col: too many patch columns");
  im2col_kernel<<<grid, dim3(32, 8), 0, st>>>(g, d_in, d_patches, rows, cols);
  note_launch();
  TKB_CUDA(cudaGetLastError());
}

void launch_transpose(const float* d_src, float* d_dst, long long rows, long long cols,
                      cudaStream_t st) {
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  if (grid.y > 65535) fail(TK_ERR_CAPABILITY, "transpose: matrix too tall");
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(d_src, d_dst, rows, cols);
  note_launch();
  TKB_CUDA(cudaGetLastError());
}

}  // namespace tkb

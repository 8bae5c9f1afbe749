// layout.cuh -- conv geometry + layout kernel launchers.
#pragma once

#include <cuda_runtime.h>

namespace tkb {

// Resolved geometry of one ConvShape (config.hpp:137-195).
struct ConvGeom {
  int N, H, W, C, K;   // batch, input rows/cols, channels, features
  int R, S, stride;    // window, stride
  int OH, OW;          // output plane
  int pad_t, pad_l;    // signed Same-padding offsets (smaller half first)
};

void launch_im2col(const ConvGeom& g, const float* d_in, float* d_patches, cudaStream_t st);
// dst = src^T for a row-major rows x cols src.
void launch_transpose(const float* d_src, float* d_dst, long long rows, long long cols,
                      cudaStream_t st);

}  // namespace tkb

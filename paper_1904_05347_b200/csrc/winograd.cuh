// winograd.cuh -- geometry + launchers of the Winograd transform kernels.
#pragma once

#include <cuda_runtime.h>

namespace tkb {

// Tile geometry of one conv2d_winograd call (winograd.hpp:181-195).
struct WinoGeom {
  int m, t;                  // output tile M, input tile T = M + 2
  int N, H, W, C, K;         // batch, input plane, channels, features
  int OH, OW;                // output plane
  int tiles_r, tiles_c;      // ceil(OH/M), ceil(OW/M)
  int tiles;                 // N * tiles_r * tiles_c
  int pad_t, pad_l;          // Same-padding origin offsets
};

void wino_input_transform(const WinoGeom& g, const float* d_in, float* d_v, cudaStream_t st);
void wino_filter_transform(const WinoGeom& g, const float* d_filt, float* d_u, bool k_major,
                           cudaStream_t st);
void wino_output_transform(const WinoGeom& g, const float* d_prod, float* d_out, cudaStream_t st);

}  // namespace tkb

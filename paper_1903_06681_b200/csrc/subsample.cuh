// subsample.cuh -- 1x1 stride-2 convolutions as plain GEMMs over the pixels
// they read (Eq. 1 with K = 1, S = 2, P = 0: y(n, i, j) = W x(n, 2i, 2j),
// PAPER.md:61; capi.cu dc_conv_fwd). The strided pixels are gathered into a
// dense buffer that the flattened 1x1 GEMM reads like a stride-1 input.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dc {

// xs[s][i][j][:] = x[s][oh + 2 i][ow + 2 j][:] for s < n, i < ho, j < wo:
// x a margined buffer [n][hb][wb] of pix_bytes per pixel (a multiple of 16),
// xs dense [n][ho][wo]. Device pointers, 16-byte aligned.
void launch_subsample2(const void *x, int64_t n, int64_t hb, int64_t wb, int pix_bytes, int oh, int ow,
                       int64_t ho, int64_t wo, void *xs, cudaStream_t st);

// The backward of the gather (dx of a 1x1 stride-2 convolution, Eq. 3 with
// K = 1, S = 2: only the read pixels receive a gradient): dx dense [n][h][w]
// of pix_bytes per pixel, dx[s][oh + 2 i][ow + 2 j] = xs[s][i][j] for
// i < ho, j < wo, every other pixel zero.
void launch_scatter2(const void *xs, int64_t n, int64_t ho, int64_t wo, int pix_bytes, int oh, int ow, int64_t h,
                     int64_t w, void *dx, cudaStream_t st);

}  // namespace dc

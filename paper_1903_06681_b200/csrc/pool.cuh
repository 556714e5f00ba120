// pool.cuh -- max pooling on the decomposition ("Pooling layers
// are parallelized similarly", "halo exchanges before ...
// pooling"; capi.cu dc_pool_*).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dc {

// One rank's view: the owned outputs (n, oh0 + i, ow0 + j), i < oh, j < ow,
// read from a margined input buffer whose element (n, r, c) is the global
// input (n, xr0 + r, xc0 + c), r < xhb, c < xwb; positions outside the global
// H x W are not part of any window (max over the in-range positions).
struct PoolGeom {
    int K, S, P;
    int H, W;              // global input extent
    int n;                 // local samples
    int cpad;              // channels per pixel (multiple of 8)
    // input buffer (margined x)
    int xr0, xc0, xhb, xwb;
    // owned outputs
    int oh0, ow0, oh, ow;
    // backward: owned inputs (gi0 + r, gj0 + c), r < ih, c < iw, written dense;
    // the dy buffer holds global outputs (dr0 + r, dc0 + c), r < dhb, c < dwb
    int gi0, gj0, ih, iw;
    int dr0, dc0, dhb, dwb;
    int Ho, Wo;            // global output extent
};

// y[n][i][j][c] = max over the in-range window of x (first maximum in (a, b)
// order, bf16 values copied exactly); y dense [n][oh][ow][cpad].
void launch_maxpool_fwd(const PoolGeom &g, const void *x, void *y, cudaStream_t st);
// dx[n][r][c][ch] (dense, owned inputs) = sum over the windows that contain
// the input and whose first maximum (recomputed from x) is it, of dy, in
// (oh, ow) order, fp32, rounded to bf16 once.
void launch_maxpool_bwd(const PoolGeom &g, const void *x, const void *dy, void *dx, cudaStream_t st);

}  // namespace dc

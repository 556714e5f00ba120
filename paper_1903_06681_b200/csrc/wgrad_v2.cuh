// wgrad_v2.cuh -- tile-reuse backward-filter kernel (see wgrad_v2.cu).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace dc {

struct WgradV2Params {
    int s_in, origin_h, origin_w;  // x coord of output pixel (0,0) at tap offset 0
    int kh, kw, T;                 // tap grid (T = kh * kw)
    int cgw, ncg, mode;            // channel-group width (16/32/64), groups, M-tile mode (see .cu)
    int PH;                        // x tile rows = s_in * 7 + kh (+ phantom rows, mode 1)
    int bw;                        // pixel block = 8 output rows x bw (8 or 16) columns
    int pitch;                     // pixels per tile row (per parity plane)
    int x_plane_bytes;             // PH * pitch * cgw * 2 B, rounded up to 1 KB
    int x_stage_bytes, dy_stage_bytes, stages;
    int bn, bn_cols;               // N tile (filters) and its TMEM column stride
    int n_mtiles, G;               // M = 128 tiles (atoms stacked), M tiles per CTA
    int tiles_h, tiles_w, nblocks; // 8 x bw output-pixel blocks per sample, total
    int splits;
    float *ws;                     // [splits][F][T][C] fp32 (or dW itself: one split / atomic_out)
    int atomic_out;                // splits add their partials into a zeroed dW (RED.ADD.F32)
    long long ws_split;            // elements per split (a multiple of 4)
    int F, Fp, cp, C;              // filters, padded filters, padded / logical input channels
    long long pixels_hint;         // host: output pixels of this launch (N tile width choice)
    // 3xTF32 (kind = 1): fp32 operands (esz = 4), 32-channel MN
    // atoms (128-byte rows, descriptor layout SW128_BASE32B), 8 x 8 pixel blocks
    // of eight K = 8 steps; the K range is `passes` copies of the pixel blocks,
    // pass 0 = x_hi . dy_hi, 1 = x_hi . dy_lo (dy channels + dy_lo), 2 = x_lo .
    // dy_hi (x channels + x_lo): the 3xTF32 product as one accumulation.
    int kind, esz, passes, nblocks_pix, x_lo, dy_lo;
};

bool wgrad_v2_configure(WgradV2Params &p, int smem_limit);
size_t wgrad_v2_smem_bytes(const WgradV2Params &p);
int wgrad_v2_mgroups(const WgradV2Params &p);  // grid.x
// xmap: 4D over the x buffer, box {cgw, pitch * s_in, PH, 1}, element strides
// {1, s_in, 1, 1}, swizzle cgw * 2 bytes. dymap: 4D over the OWNED dy block, box
// {64, 8, 8, 1}, 128B swizzle.
void launch_wgrad_v2(const CUtensorMap &xmap, const CUtensorMap &dymap, const WgradV2Params &p,
                     cudaStream_t st);

}  // namespace dc

// wgrad_v2.cuh -- tile-reuse backward-filter kernel (see wgrad_v2.cu).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace dc {

struct WgradV2Params {
    int s_in, origin_h, origin_w;  // x coord of output pixel (0,0) at tap offset 0
    int kh, kw, T;                 // tap grid (T = kh * kw)
    int PH;                        // x tile rows = s_in * 7 + kh (8 output rows per block)
    int x_plane_bytes;             // PH * 16 px * 128 B
    int x_stage_bytes, dy_stage_bytes, stages;
    int bn, bn_cols;               // N tile (filters) and its TMEM column stride
    int natoms, n_mtiles, G;       // (cp/64)*T atoms of 64 channels; M tiles = atom pairs; per CTA
    int tiles_h, tiles_w, nblocks; // 8x8 output-pixel blocks per sample, total
    int splits;
    float *ws;                     // [splits][F][T][cp] fp32
    long long ws_split;
    int F, Fp, cp;
};

bool wgrad_v2_configure(WgradV2Params &p, int smem_limit);
size_t wgrad_v2_smem_bytes(const WgradV2Params &p);
// xmap: 4D over the x buffer, box {64, 16 * s_in, PH, 1}, element strides
// {1, s_in, 1, 1}, 128B swizzle. dymap: 4D over the OWNED dy block, box
// {64, 8, 8, 1}, 128B swizzle.
void launch_wgrad_v2(const CUtensorMap &xmap, const CUtensorMap &dymap, const WgradV2Params &p,
                     cudaStream_t st);

}  // namespace dc

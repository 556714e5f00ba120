// conv_tc.cuh -- host-visible parameter blocks and launchers of the sm_100a
// implicit-GEMM convolution kernels (conv_tc.cu).
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <vector>

namespace dc {

constexpr int kMaxTaps = 64;
constexpr int kMaxRects = 5;

// A rectangle of GEMM output pixels (local coordinates of the launch's
// output pixel grid), tiled by TH x TW tiles.
struct OutRect {
    int h0, w0, nh, nw;
};

// Parameters of the forward / backward-data implicit GEMM
//   D[pixel, o] = sum_{tap t} sum_{c} A_t[pixel, c] * B[o, t, c]
// A_t[pixel (i,j), c] = in[n, s_in*i + origin_h + tap_h[t], s_in*j + origin_w + tap_w[t], c]
// (TMA zero-fills coordinates outside the input buffer = the padding).
struct ConvGemmParams {
    int T;          // taps
    int kc;         // channel chunks per tap (cin_p / bkc)
    int bkc;        // channels per chunk (16, 32, 64) -> swizzle 32/64/128 B
    int bn;         // GEMM N tile (output channels per CTA): 16..256, multiple of 16
    int stages;
    int s_in, origin_h, origin_w;
    int8_t tap_h[kMaxTaps], tap_w[kMaxTaps];
    int nrect;
    OutRect rect[kMaxRects];
    int rect_twl[kMaxRects];  // per rect: tile = (128 >> twl) rows x (1 << twl) cols
    int rect_tiles_w[kMaxRects];
    int rect_start[kMaxRects + 1];
    // output: pixel (i, j) of the GEMM grid -> out[n][out_h0 + out_dh*i][out_w0 + out_dw*j][o]
    __nv_bfloat16 *out;
    long long out_sn, out_sh, out_sw;
    int out_h0, out_w0, out_dh, out_dw;
    int nout_p;     // channels written (padded, multiple of 16)
};

// Parameters of the backward-filter implicit GEMM (both operands MN-major)
//   D[(t, c), f] = sum_{pixels} X_t[pixel, c] * DY[pixel, f]
struct WgradParams {
    int T, kc, bkc;      // taps, channel chunks per tap, channels per chunk
    int pairs_total;     // T * kc  ("pairs" = (tap, chunk) = 128/bkc per M tile)
    int bf;              // dy channels per TMA box (16/32/64)
    int bn;              // GEMM N tile (filters per CTA)
    int stages;
    int s_in, origin_h, origin_w;
    int8_t tap_h[kMaxTaps], tap_w[kMaxTaps];
    int tw_log2;         // pixel block = (64 >> tw_log2) x (1 << tw_log2)
    int tiles_h, tiles_w, nblocks;  // pixel blocks per sample, total over samples
    int splits;
    float *ws;           // [splits][F][T][C] (dW itself when splits == 1)
    long long ws_split;  // elements per split (>= F * T * C, a multiple of 4)
    int F, cp, C;        // filters, padded / logical input channels
};

// ---- host helpers ----
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
void make_tmap(CUtensorMap *m, const void *ptr, int rank, const uint64_t *dims,
               const uint64_t *strides_bytes /* rank-1 */, const uint32_t *box,
               const uint32_t *estrides, int swizzle_bytes);

// The same with an explicit element type and swizzle mode (e.g. fp32 with
// CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B for MN-major tf32 operands).
void make_tmap_ex(CUtensorMap *m, const void *ptr, int rank, const uint64_t *dims, const uint64_t *strides_bytes,
                  const uint32_t *box, const uint32_t *estrides, CUtensorMapDataType dt, CUtensorMapSwizzle sw);

void launch_conv_gemm(const CUtensorMap &amap, const CUtensorMap &bmap, const ConvGemmParams &p,
                      int nsamples, int nout_tiles, cudaStream_t st);
void launch_wgrad(const CUtensorMap &amap, const CUtensorMap &bmap, const WgradParams &p,
                  int m_tiles, int n_tiles, cudaStream_t st);
void launch_splitk_reduce(const float *ws, int splits, long long n, long long split_stride, float *dw,
                          cudaStream_t st);
// W'[c][t][f] = w[f][ka[t]][kb[t]][c] for the backward-data taps (zero if c >= C or f >= F)
// All stride phases at once: tap j (of ntaps) reads w tap (ka[j], kb[j]) and
// writes index t[j] of its phase's [Cp][T[j]][Fp] block at wt_base + off[j].
void launch_weight_transform_multi(const __nv_bfloat16 *w, __nv_bfloat16 *wt_base, int F, int Fp, int C, int Cp,
                                   int K, int ntaps, const int8_t *ka, const int8_t *kb, const int *T,
                                   const int *t, const long long *off, cudaStream_t st);
// Sub-pixel backward-data weights for stride 2 (see conv_tc.cu): [4 Cp][D*D][Fp].
void launch_subpix_weights(const __nv_bfloat16 *w, __nv_bfloat16 *wt, int F, int Fp, int C, int Cp, int K, int P,
                           int dmin, int D, cudaStream_t st);
void launch_weight_transform(const __nv_bfloat16 *w, __nv_bfloat16 *wt, int F, int Fp, int C,
                             int Cp, int K, int T, const int8_t *ka, const int8_t *kb,
                             cudaStream_t st);

size_t conv_gemm_smem_bytes(int bkc, int bn, int stages);
size_t wgrad_smem_bytes(int bkc, int bf, int bn, int stages);

}  // namespace dc

// conv_v2.cuh -- persistent tile-reuse implicit-GEMM convolution (forward and
// backward-data) for sm_100a.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "conv_tc.cuh"
#include "halo.cuh"

namespace dc {

// Output tile: TH x TW = 16 x 8 GEMM pixels (M = 128). The input tile that
// all taps of the tile read (the "halo'd tile") is loaded ONCE per channel
// group into shared memory as 16-byte "core-matrix planes"
//   plane[(chunk8 * s_in + parity)][PH rows][PWs cols][8 channels]
// (parity = input column mod s_in), so the UMMA operand of every tap is the
// same smem buffer at a shifted start address (SWIZZLE_NONE K-major: core
// matrix = 8 consecutive output pixels x 16 bytes, SBO = next output row,
// LBO = next 8-channel chunk).
constexpr int kV2TH = 16, kV2TW = 8;
// dynamic shared memory budget (227 KB per block minus the static tap table)
constexpr int kV2SmemLimit = 227 * 1024 - 1024;

// Two A layouts:
//   a_swz == 0   : the core-matrix planes above (any cin_p multiple of 16, any s_in)
//   a_swz == 128 : cin_p % 64 == 0 and s_in == 1: the halo'd tile as 128-byte
//                  rows (64 channels, 128B swizzle), row pitch padded to 16
//                  pixels so every output row starts at a 1024-byte boundary
//                  and a tap shift (th, tw) only changes the start address and
//                  the swizzle phase (tw mod 8) of the descriptor.
struct ConvV2Params {
    int a_swz;                 // 0 or 128 (see above)
    // Measured: the 128B swizzle is a function of the absolute smem address, so
    // the phase of a shifted start address must NOT be put in the descriptor's
    // base-offset field (doing so breaks parity).
    // Taps always form the grid th in [0,kh) x tw in [0,kw) (tap t = th*kw + tw);
    // the A operand of tap (th, tw) starts at (16-byte units)
    //   th*a_row16 + (tw >> s_shift)*a_col16 + (tw & (s_in-1))*a_par16
    int kh, kw, s_shift;
    uint32_t a_row16, a_col16, a_par16;
    int tpw;                       // tiles per work item (1, or 2 stacked 16 x 8 tiles sharing
                                   // each streamed weight stage; set by conv_v2_configure)
    int tw_log2;                   // GEMM tile: (128 >> tw_log2) rows x (1 << tw_log2) cols:
                                   // 3 -> 16 x 8 (default), 7 -> 1 x 128 (thin boundary strips)
    uint32_t a_sbo;                // A descriptor SBO: byte distance between 8-pixel groups
    uint32_t a_kstep16;            // A descriptor delta between 16-channel K slices
    // Fused BN statistics of the stored y: per CTA, fp64 sum and
    // sum of squares of every channel over the CTA's tiles, written to
    // bn_part[blockIdx.x][2][nout_p] (needs ksplit == 1 and nout_tiles == 1)
    int bn_stats;
    int epi2;                  // device: 8 epilogue warps (two groups split the 16-column chunks)
    double *bn_part;
    int s_in;                  // A element stride (conv stride for fwd, 1 for bwd-data)
    int origin_h, origin_w;    // input coord of GEMM pixel (0,0) at tap offset 0
    int T;                     // taps
    int8_t tap_h[kMaxTaps], tap_w[kMaxTaps];  // tap offsets (>= 0)
    int cin_p;                 // input channels (multiple of 16)
    int cg;                    // channels per A stage (16, 32 or 64; divides cin_p)
    int ncg;                   // cin_p / cg
    int PH, PWs;               // halo'd tile rows / cols per parity plane
    int plane_bytes;           // PH * PWs * 16 rounded up to 128
    int a_stage_bytes;         // (cg / 8) * s_in * plane_bytes
    int a_stages;
    int bn;                    // GEMM N tile (multiple of 16, <= 256)
    int b_resident;            // 1: the whole [T][cin_p] x bn weight tile stays in smem
    int b_slot_bytes;          // bn * cg * 2 rounded up to 1024
    int b_stages;              // ring depth when not resident
    int nrect;
    OutRect rect[kMaxRects];
    int rect_tiles_w[kMaxRects];
    int rect_start[kMaxRects + 1];
    int nsamples, nout_tiles, total_tiles;
    // split-K over channel groups (small-spatial, many-channel layers): CTA b
    // takes split b % ksplit; partial sums (fp32) go to ws[split][n][ws_h][ws_w][nout_p]
    // and conv_v2_reduce sums them in split order. ksplit depends only on the
    // global layer shape, so partitioned results stay bitwise equal to 1 GPU.
    int ksplit;
    int work_hint;             // work items of THIS launch at tpw = 1 (x ksplit): pairing only when plentiful
    int max_ctas;              // host: persistent grid cap (0: SM count)
    int cluster;               // 2: CTA pairs share (multicast) every streamed weight stage; 1: none
    int allow_cg32;            // stride 2: may narrow 64-channel stages to 32 for tile pairs (changes the
                               // summation order: decided from the GLOBAL layer, see capi.cu)
    float *ws;
    int ws_h, ws_w;
    __nv_bfloat16 *out;
    long long out_sn, out_sh, out_sw;
    int out_h0, out_w0, out_dh, out_dw;
    // sub-pixel backward-data (stride 2, small C): output column n = phase *
    // sub_cp + c goes to pixel (out_h0 + 2 i + phase/2, out_w0 + 2 j + phase%2),
    // kept only inside [0, out_hmax) x [0, out_wmax)
    int subpix, sub_cp, out_hmax, out_wmax;
    int nout_p;
    // 3xTF32 (DC_FP32_3XTF32): kind = 1 runs kind::tf32 MMAs on
    // fp32 data seen as pairs of 16-bit "channels" (a 32-byte K step is 8 fp32
    // = 16 bf16, so every smem / TMA / descriptor geometry is unchanged);
    // a_seg > 0 maps weight K channels >= a_seg (in 16-bit units) a_seg lower
    // in the input (x_hi x_hi x_lo against w_hi w_lo w_hi); out_f32 stores fp32.
    int kind, a_seg, out_f32;
    // fp32 output scattered by output-channel block (channel / filter
    // parallelism, capi.cu dc_cconv_*): column o goes to scat[o / scat_seg] at
    // channel o % scat_seg of a tensor with channel pitch scat_seg (out_s*
    // strides in that pitch); scat_seg = 0: plain out
    float *scat[8];
    int scat_seg;
};

size_t conv_v2_smem_bytes(const ConvV2Params &p);
// Fills the derived fields (PH, PWs, stage sizes, residency, stages) from the
// taps / stride / channels / bn / tw_log2 already set; returns false if it
// cannot fit (e.g. a 1 x 128 strip with stride 2).
bool conv_v2_configure(ConvV2Params &p, int smem_limit);
// amap: 4D map over the input buffer with box {8, PWs * s_in, PH, 1} and
// element strides {1, s_in, 1, 1}, no swizzle. bmap: [N rows][T * cin_p]
// weights with box {cg, bn}, swizzle cg * 2 bytes.
// returns the grid size (number of CTAs, = BN partial slots used)
int launch_conv_v2(const CUtensorMap &amap, const CUtensorMap &bmap, const ConvV2Params &p,
                    cudaStream_t st);
// Fixed-order sum of the split-K partials -> bf16 output (rects / out mapping of p).
void launch_conv_v2_reduce(const ConvV2Params &p, cudaStream_t st);
int device_sm_count();

}  // namespace dc

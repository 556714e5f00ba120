// tf32.cuh -- the fp32 (DC_FP32_3XTF32) side kernels: operand splitting for
// 3xTF32, tensor import into margined buffers, fp32 BN partial sums.
//
// 3xTF32 (reading R18): an fp32 value is split exactly as
//   x = x_hi + x_lo,  x_hi = x with its low 13 mantissa bits cleared (a tf32
//   value), x_lo = x - x_hi (exact in fp32);
// the tensor core reads tf32 operands by truncation (tools/tf32_probe.cu), and
//   x.w ~ x_hi.w_hi + x_hi.w_lo + x_lo.w_hi
// with a relative error ~2^-21 per product (the dropped x_lo.w_lo and the
// truncation of x_lo, w_lo). The conv kernels compute the three products as
// ONE accumulation over a K dimension three times as long (weights laid out
// [w_hi | w_lo | w_hi] per tap against the input's [x_hi | x_hi | x_lo]).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "conv_tc.cuh"

namespace dc {

// src: dense NHWC block [n][h][w][C] (the owned block, logical channels),
// fp32 (or bf16 when src_bf16, for bf16 plans: a plain copy).
// dst: the margined buffer [n][hb][wb][cb] at rows/cols offset (r0, c0):
//   split == 0: bf16, cb = cp channels (rounded to nearest, zeros past C);
//   split == 1: fp32, cb = 2 cp: [x_hi (cp) | x_lo (cp)], zeros past C.
void launch_import(const void *src, bool src_bf16, void *dst, int n, int h, int w, int C, int cp, int hb, int wb,
                   int r0, int c0, int split, cudaStream_t st);

// Forward weights for 3xTF32: w fp32 [F][T][cp] -> ws fp32 [F][T][3 cp] =
// per tap [w_hi | w_lo | w_hi] (channels >= C zero).
void launch_weight_split(const float *w, float *ws, int F, int T, int C, int cp, cudaStream_t st);

// Backward-data weights for 3xTF32 (phase decomposition of Eq. 3): for each
// listed tap j, wt[off_j + ((c * T_j + t_j) * 3 + seg) * fp + f] =
// {hi, lo, hi}[seg] of w[f][ka_j][kb_j][c] (zeros past F / C).
void launch_weight_transform_tf32(const float *w, float *wt_base, int F, int fp, int C, int cp, int K, int ntaps,
                                  const int8_t *ka, const int8_t *kb, const int *T, const int *t,
                                  const long long *off, cudaStream_t st);

// Per-block fp64 sums / sums of squares of a dense NHWC fp32 tensor
// [npix][cpad] -> partials [blocks][2][cpad] (reduced by launch_bn_reduce).
int bn_partial_blocks_f32(long long npix, int cpad);
void launch_bn_partials_f32(const float *t, long long npix, int cpad, double *partials, cudaStream_t st);

}  // namespace dc

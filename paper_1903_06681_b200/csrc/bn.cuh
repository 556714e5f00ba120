// bn.cuh -- batch-norm apply / backward on the decomposition (bn.cu).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dc {

// One elementwise pass over a shard: y (and res, dout) dense NHWC [npix][cpad]
// (bf16: esz 2, fp32: esz 4); per-channel coefficients coef[4][cpad] =
// {gamma/sd, beta - gamma mean/sd, 1/sd, mean}; output pixel p = (n, i, j) of
// the n x h x w block goes to dst pixel (n, r0 + i, c0 + j) of a buffer
// [.][hb][wb][dcp] (bf16, or fp32 [hi | lo] halves of dcp/2 when split).
struct BnArgs {
    const void *y, *res, *dout;
    const float *coef;
    int esz, relu;
    long long npix;
    int cpad, c;
    void *dst;
    int n, h, w, hb, wb, r0, c0, dcp, split;
};

void launch_bn_coeff(const double *mean, const double *var, const float *gamma, const float *beta, double eps,
                     int c, int cpad, float *coef, cudaStream_t st);
void launch_bn_apply(const BnArgs &a, cudaStream_t st);
int bn_bwd_blocks(const BnArgs &a);  // grid of the backward partials (one block per SM at most)
// partials [blocks][2][cpad]: sum g, sum g y_hat (fp64; reduce with launch_bn_reduce)
void launch_bn_bwd_partials(const BnArgs &a, double *partials, int blocks, cudaStream_t st);
// sums[2][cpad] = the group's sum g, sum g y_hat; count = the group's pixels
// BN statistics of a dense bf16 NHWC tensor [npix][cpad]: partials
// [blocks][2][cpad] = per-block sum y, sum y^2 (fp64; reduce with launch_bn_reduce)
int bn_stats_blocks(long long npix, int cpad);
void launch_bn_stats(const void *y, long long npix, int cpad, double *partials, int blocks, cudaStream_t st);
void launch_bn_bwd_apply(const BnArgs &a, const double *sums, double count, const float *gamma, float *dgamma,
                         float *dbeta, void *dres, cudaStream_t st);

}  // namespace dc

// bn.cu -- the layers between the convolutions on the same decomposition
// (PAPER.md:149, 234-236): batch-norm apply with the
// spatially aggregated statistics (+ residual add, ReLU), written straight
// into the next layer's margined input, and its backward, whose per-channel
// sums sum(g), sum(g y_hat) are aggregated over the spatial group like the
// forward statistics. Memory-bound elementwise / reduction
// kernels: 16-byte vector loads, one thread per 8 channels of a pixel.
#include <cuda_bf16.h>

#include "bn.cuh"
#include "common.hpp"
#include "launch.cuh"

namespace dc {

namespace {
__device__ __forceinline__ float hi_tf32(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// 8 channels of pixel p of a dense NHWC tensor (bf16 or fp32) as fp32
__device__ __forceinline__ void load8(const void *t, int esz, long long p, int cpad, int c8, float (&v)[8]) {
    if (esz == 2) {
        const uint4 r = reinterpret_cast<const uint4 *>(t)[(p * cpad) / 8 + c8];
        const __nv_bfloat16 *h = reinterpret_cast<const __nv_bfloat16 *>(&r);
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = __bfloat162float(h[e]);
    } else {
        const float4 *f = reinterpret_cast<const float4 *>(t) + (p * cpad) / 4 + 2 * c8;
        const float4 a = f[0], b = f[1];
        v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
    }
}

// 8 channels into a (margined) buffer pixel q: bf16, or the fp32 [hi | lo] split
__device__ __forceinline__ void store8(void *dst, int esz, int split, long long q, int dcp, int c8,
                                       const float (&v)[8]) {
    if (esz == 2) {
        uint4 r;
        __nv_bfloat16 *h = reinterpret_cast<__nv_bfloat16 *>(&r);
#pragma unroll
        for (int e = 0; e < 8; ++e) h[e] = __float2bfloat16_rn(v[e]);
        reinterpret_cast<uint4 *>(dst)[(q * dcp) / 8 + c8] = r;
    } else {
        float *d = reinterpret_cast<float *>(dst) + q * dcp + c8 * 8;
        if (split) {
            const int half = dcp / 2;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const float hv = hi_tf32(v[e]);
                d[e] = hv;
                d[half + e] = v[e] - hv;
            }
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e) d[e] = v[e];
        }
    }
}

__device__ __forceinline__ long long dst_pixel(const BnArgs &a, long long p) {
    const int j = (int)(p % a.w);
    const long long r = p / a.w;
    const int i = (int)(r % a.h), n = (int)(r / a.h);
    return ((long long)n * a.hb + a.r0 + i) * a.wb + a.c0 + j;
}
}  // namespace

// per channel: scale = gamma / sqrt(var + eps), shift = beta - scale * mean,
// inv_sd = 1 / sqrt(var + eps) (fp64, rounded once); zero past c
__global__ void bn_coeff_kernel(const double *mean, const double *var, const float *gamma, const float *beta,
                                double eps, int c, int cpad, float *coef) {
    pdl_wait();  // (launch.cuh: PDL)
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < cpad; k += gridDim.x * blockDim.x) {
        double s = 0, sh = 0, inv = 0, mu = 0;
        if (k < c) {
            inv = 1.0 / sqrt(var[k] + eps);
            s = (double)gamma[k] * inv;
            sh = (double)beta[k] - s * mean[k];
            mu = mean[k];
        }
        coef[k] = (float)s;
        coef[cpad + k] = (float)sh;
        coef[2 * cpad + k] = (float)inv;
        coef[3 * cpad + k] = (float)mu;
    }
}

__global__ void bn_apply_kernel(const __grid_constant__ BnArgs a) {
    pdl_wait();  // (launch.cuh: PDL)
    const int c8n = a.cpad / 8;
    const long long total = a.npix * c8n;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c8 = (int)(i % c8n);
        const long long p = i / c8n;
        float v[8], r[8];
        load8(a.y, a.esz, p, a.cpad, c8, v);
        if (a.res) load8(a.res, a.esz, p, a.cpad, c8, r);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int k = c8 * 8 + e;
            float z = fmaf(a.coef[k], v[e], a.coef[a.cpad + k]);
            if (a.res) z += r[e];
            v[e] = (a.relu && z < 0.f) ? 0.f : z;
        }
        store8(a.dst, a.esz, a.split, dst_pixel(a, p), a.dcp, c8, v);
    }
}

// backward partials: per block fp64 sums of g and g * y_hat per channel, g the
// output gradient through the ReLU mask (recomputed from y) -> [blocks][2][cpad]
__global__ void __launch_bounds__(256) bn_bwd_partials_kernel(const __grid_constant__ BnArgs a, double *partials) {
    pdl_wait();  // (launch.cuh: PDL)
    extern __shared__ double sh[];
    const int c8n = a.cpad / 8;
    const int lanes = max(1, 256 / c8n);
    const int c8 = threadIdx.x % c8n, pl = threadIdx.x / c8n;
    if (pl < lanes) {
        double sg[8], sgy[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) sg[e] = sgy[e] = 0.0;
        for (long long p = (long long)blockIdx.x * lanes + pl; p < a.npix; p += (long long)gridDim.x * lanes) {
            float v[8], d[8], r[8];
            load8(a.y, a.esz, p, a.cpad, c8, v);
            load8(a.dout, a.esz, p, a.cpad, c8, d);
            if (a.res) load8(a.res, a.esz, p, a.cpad, c8, r);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int k = c8 * 8 + e;
                float z = fmaf(a.coef[k], v[e], a.coef[a.cpad + k]);
                if (a.res) z += r[e];
                const float g = (a.relu && z <= 0.f) ? 0.f : d[e];
                const float yh = (v[e] - a.coef[3 * a.cpad + k]) * a.coef[2 * a.cpad + k];
                sg[e] += (double)g;
                sgy[e] += (double)g * (double)yh;
            }
        }
        double *row = sh + (long long)pl * 2 * a.cpad;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            row[c8 * 8 + e] = sg[e];
            row[a.cpad + c8 * 8 + e] = sgy[e];
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < 2 * a.cpad; k += blockDim.x) {
        double acc = 0.0;
        for (int l = 0; l < lanes; ++l) acc += sh[(long long)l * 2 * a.cpad + k];
        partials[(long long)blockIdx.x * 2 * a.cpad + k] = acc;
    }
}

// dy = gamma inv_sd (g - sum g / M - y_hat sum(g y_hat) / M) into the margined dy
// buffer; dgamma = sum(g y_hat), dbeta = sum(g) (block 0); dres = g (dense)
__global__ void bn_bwd_apply_kernel(const __grid_constant__ BnArgs a, const double *sums, double count,
                                    const float *gamma, float *dgamma, float *dbeta, void *dres) {
    pdl_wait();  // (launch.cuh: PDL)
    if (blockIdx.x == 0)
        for (int k = threadIdx.x; k < a.c; k += blockDim.x) {
            if (dgamma) dgamma[k] = (float)sums[a.cpad + k];
            if (dbeta) dbeta[k] = (float)sums[k];
        }
    const int c8n = a.cpad / 8;
    const long long total = a.npix * c8n;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c8 = (int)(i % c8n);
        const long long p = i / c8n;
        float v[8], d[8], r[8], o[8];
        load8(a.y, a.esz, p, a.cpad, c8, v);
        load8(a.dout, a.esz, p, a.cpad, c8, d);
        if (a.res) load8(a.res, a.esz, p, a.cpad, c8, r);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int k = c8 * 8 + e;
            float z = fmaf(a.coef[k], v[e], a.coef[a.cpad + k]);
            if (a.res) z += r[e];
            const float g = (a.relu && z <= 0.f) ? 0.f : d[e];
            d[e] = g;
            if (k < a.c) {
                const float inv = a.coef[2 * a.cpad + k];
                const float yh = (v[e] - a.coef[3 * a.cpad + k]) * inv;
                const float m1 = (float)(sums[k] / count), m2 = (float)(sums[a.cpad + k] / count);
                o[e] = gamma[k] * inv * (g - m1 - yh * m2);
            } else {
                o[e] = 0.f;
            }
        }
        store8(a.dst, a.esz, a.split, dst_pixel(a, p), a.dcp, c8, o);
        if (dres) store8(dres, a.esz, 0, p, a.cpad, c8, d);
    }
}

int bn_bwd_blocks(long long npix, int cpad) {
    const int lanes = std::max(1, 256 / (cpad / 8));
    const long long iters = (npix + lanes - 1) / lanes;
    return (int)std::max<long long>(1, std::min<long long>((iters + 15) / 16, 148 * 2));
}

void launch_bn_coeff(const double *mean, const double *var, const float *gamma, const float *beta, double eps,
                     int c, int cpad, float *coef, cudaStream_t st) {
    launch_k(bn_coeff_kernel, dim3((cpad + 255) / 256), dim3(256), 0, st, 1, "bn coeff", mean, var, gamma, beta,
             eps, c, cpad, coef);
}

void launch_bn_apply(const BnArgs &a, cudaStream_t st) {
    DC_REQUIRE(a.cpad % 8 == 0 && a.dcp % 8 == 0, DC_ERR_UNSUPPORTED, "BN apply: channels must be multiples of 8");
    const long long total = a.npix * (a.cpad / 8);
    if (total == 0) return;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
    launch_k(bn_apply_kernel, dim3(blocks), dim3(256), 0, st, 1, "bn apply", a);
}

void launch_bn_bwd_partials(const BnArgs &a, double *partials, int blocks, cudaStream_t st) {
    DC_REQUIRE(a.cpad % 8 == 0 && a.cpad / 8 <= 256, DC_ERR_UNSUPPORTED, "BN backward: channels");
    const int lanes = std::max(1, 256 / (a.cpad / 8));
    launch_k(bn_bwd_partials_kernel, dim3(blocks), dim3(256), (size_t)lanes * 2 * a.cpad * sizeof(double), st, 1,
             "bn bwd partials", a, partials);
}

void launch_bn_bwd_apply(const BnArgs &a, const double *sums, double count, const float *gamma, float *dgamma,
                         float *dbeta, void *dres, cudaStream_t st) {
    const long long total = a.npix * (a.cpad / 8);
    const int blocks = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, 148 * 16));
    launch_k(bn_bwd_apply_kernel, dim3(blocks), dim3(256), 0, st, 1, "bn bwd apply", a, sums, count, gamma, dgamma,
             dbeta, dres);
}

// Loads this file's kernels (see preload_conv_v2)
void preload_bn() {
    cudaFuncAttributes at;
    cudaFuncGetAttributes(&at, reinterpret_cast<const void *>(bn_coeff_kernel));
    cudaFuncGetAttributes(&at, reinterpret_cast<const void *>(bn_apply_kernel));
    cudaFuncGetAttributes(&at, reinterpret_cast<const void *>(bn_bwd_partials_kernel));
    cudaFuncGetAttributes(&at, reinterpret_cast<const void *>(bn_bwd_apply_kernel));
}

}  // namespace dc

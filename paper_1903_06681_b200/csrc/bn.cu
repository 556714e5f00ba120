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

// Thread -> (pixel lane, 8-channel group) mapping of the elementwise / reduction
// kernels: a thread keeps ONE channel group (its per-channel constants live in
// registers) and walks the pixels; cb = min(c8n, 256) groups per pass,
// lanes = 256 / cb pixel lanes per block, further passes for cpad > 2048.
struct Lanes {
    int cb, lanes, pl, c8;
};
__device__ __forceinline__ Lanes lanes_of(int cpad) {
    Lanes l;
    const int c8n = cpad / 8;
    l.cb = c8n < 256 ? c8n : 256;
    l.lanes = 256 / l.cb;
    l.pl = threadIdx.x / l.cb;
    l.c8 = threadIdx.x % l.cb;
    return l;
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

__global__ void __launch_bounds__(256) bn_apply_kernel(const __grid_constant__ BnArgs a) {
    pdl_wait();  // (launch.cuh: PDL)
    const Lanes L = lanes_of(a.cpad);
    if (L.pl >= L.lanes) return;
    for (int c8 = L.c8; c8 < a.cpad / 8; c8 += L.cb) {
        float sc[8], sh[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) sc[e] = a.coef[c8 * 8 + e], sh[e] = a.coef[a.cpad + c8 * 8 + e];
        for (long long p = (long long)blockIdx.x * L.lanes + L.pl; p < a.npix; p += (long long)gridDim.x * L.lanes) {
            float v[8], r[8];
            load8(a.y, a.esz, p, a.cpad, c8, v);
            if (a.res) load8(a.res, a.esz, p, a.cpad, c8, r);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                float z = fmaf(sc[e], v[e], sh[e]);
                if (a.res) z += r[e];
                v[e] = (a.relu && z < 0.f) ? 0.f : z;
            }
            store8(a.dst, a.esz, a.split, dst_pixel(a, p), a.dcp, c8, v);
        }
    }
}

// backward partials: per block fp64 sums of g and g * y_hat per channel, g the
// output gradient through the ReLU mask (recomputed from y) -> [blocks][2][cpad]
__global__ void __launch_bounds__(256) bn_bwd_partials_kernel(const __grid_constant__ BnArgs a, double *partials) {
    pdl_wait();  // (launch.cuh: PDL)
    extern __shared__ double sh[];
    const Lanes L = lanes_of(a.cpad);
    for (int c8 = L.c8; c8 < a.cpad / 8; c8 += L.cb) {
        if (L.pl < L.lanes) {
            float sc[8], sf[8], inv[8], mu[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const int k = c8 * 8 + e;
                sc[e] = a.coef[k], sf[e] = a.coef[a.cpad + k], inv[e] = a.coef[2 * a.cpad + k];
                mu[e] = a.coef[3 * a.cpad + k];
            }
            double sg[8], sgy[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) sg[e] = sgy[e] = 0.0;
            const long long step = (long long)gridDim.x * L.lanes;
            long long p = (long long)blockIdx.x * L.lanes + L.pl;
            // two pixels per trip: twice the loads in flight
            for (; p + step < a.npix; p += 2 * step) {
                float v[8], d[8], v2[8], d2[8], r[8], r2[8];
                load8(a.y, a.esz, p, a.cpad, c8, v);
                load8(a.dout, a.esz, p, a.cpad, c8, d);
                load8(a.y, a.esz, p + step, a.cpad, c8, v2);
                load8(a.dout, a.esz, p + step, a.cpad, c8, d2);
                if (a.res) {
                    load8(a.res, a.esz, p, a.cpad, c8, r);
                    load8(a.res, a.esz, p + step, a.cpad, c8, r2);
                }
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    float z = fmaf(sc[e], v[e], sf[e]), z2 = fmaf(sc[e], v2[e], sf[e]);
                    if (a.res) z += r[e], z2 += r2[e];
                    const float g = (a.relu && z <= 0.f) ? 0.f : d[e];
                    const float g2 = (a.relu && z2 <= 0.f) ? 0.f : d2[e];
                    const float yh = (v[e] - mu[e]) * inv[e], yh2 = (v2[e] - mu[e]) * inv[e];
                    sg[e] += (double)g;
                    sgy[e] += (double)g * (double)yh;
                    sg[e] += (double)g2;
                    sgy[e] += (double)g2 * (double)yh2;
                }
            }
            if (p < a.npix) {
                float v[8], d[8], r[8];
                load8(a.y, a.esz, p, a.cpad, c8, v);
                load8(a.dout, a.esz, p, a.cpad, c8, d);
                if (a.res) load8(a.res, a.esz, p, a.cpad, c8, r);
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    float z = fmaf(sc[e], v[e], sf[e]);
                    if (a.res) z += r[e];
                    const float g = (a.relu && z <= 0.f) ? 0.f : d[e];
                    sg[e] += (double)g;
                    sgy[e] += (double)g * (double)((v[e] - mu[e]) * inv[e]);
                }
            }
            double *row = sh + (long long)L.pl * 2 * a.cpad;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                row[c8 * 8 + e] = sg[e];
                row[a.cpad + c8 * 8 + e] = sgy[e];
            }
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < 2 * a.cpad; k += blockDim.x) {
        double acc = 0.0;
        for (int l = 0; l < L.lanes; ++l) acc += sh[(long long)l * 2 * a.cpad + k];
        partials[(long long)blockIdx.x * 2 * a.cpad + k] = acc;
    }
}

// dy = gamma inv_sd (g - sum g / M - y_hat sum(g y_hat) / M) into the margined dy
// buffer; dgamma = sum(g y_hat), dbeta = sum(g) (block 0); dres = g (dense)
__global__ void __launch_bounds__(256) bn_bwd_apply_kernel(const __grid_constant__ BnArgs a, const double *sums,
                                                           double count, const float *gamma, float *dgamma,
                                                           float *dbeta, void *dres) {
    pdl_wait();  // (launch.cuh: PDL)
    if (blockIdx.x == 0)
        for (int k = threadIdx.x; k < a.c; k += blockDim.x) {
            if (dgamma) dgamma[k] = (float)sums[a.cpad + k];
            if (dbeta) dbeta[k] = (float)sums[k];
        }
    const Lanes L = lanes_of(a.cpad);
    if (L.pl >= L.lanes) return;
    for (int c8 = L.c8; c8 < a.cpad / 8; c8 += L.cb) {
        // per-channel constants of this thread's 8 channels, once
        float sc[8], sf[8], inv[8], mu[8], k1[8], m1[8], m2[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int k = c8 * 8 + e;
            sc[e] = a.coef[k], sf[e] = a.coef[a.cpad + k], inv[e] = a.coef[2 * a.cpad + k];
            mu[e] = a.coef[3 * a.cpad + k];
            const bool live = k < a.c;
            k1[e] = live ? gamma[k] * inv[e] : 0.f;
            m1[e] = live ? (float)(sums[k] / count) : 0.f;
            m2[e] = live ? (float)(sums[a.cpad + k] / count) : 0.f;
        }
        for (long long p = (long long)blockIdx.x * L.lanes + L.pl; p < a.npix; p += (long long)gridDim.x * L.lanes) {
            float v[8], d[8], r[8], o[8];
            load8(a.y, a.esz, p, a.cpad, c8, v);
            load8(a.dout, a.esz, p, a.cpad, c8, d);
            if (a.res) load8(a.res, a.esz, p, a.cpad, c8, r);
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                float z = fmaf(sc[e], v[e], sf[e]);
                if (a.res) z += r[e];
                const float g = (a.relu && z <= 0.f) ? 0.f : d[e];
                d[e] = g;
                const float yh = (v[e] - mu[e]) * inv[e];
                o[e] = k1[e] * (g - m1[e] - yh * m2[e]);
            }
            store8(a.dst, a.esz, a.split, dst_pixel(a, p), a.dcp, c8, o);
            if (dres) store8(dres, a.esz, 0, p, a.cpad, c8, d);
        }
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

// bn.cu -- the layers between the convolutions on the same decomposition
// (PAPER.md:149, 234-236): batch-norm apply with the
// spatially aggregated statistics (+ residual add, ReLU), written straight
// into the next layer's margined input, and its backward, whose per-channel
// sums sum(g), sum(g y_hat) are aggregated over the spatial group like the
// forward statistics. Memory-bound elementwise / reduction
// kernels: 16-byte vector loads, one thread per 8 channels of a pixel.
#include <cuda_bf16.h>

#include <mutex>

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

// 2 channels (pair c2) of pixel p of a dense NHWC tensor as fp32
__device__ __forceinline__ void load2(const void *t, int esz, long long p, int cpad, int c2, float &x0, float &x1) {
    if (esz == 2) {
        const uint32_t r = reinterpret_cast<const uint32_t *>(t)[(p * cpad) / 2 + c2];
        x0 = __uint_as_float(r << 16), x1 = __uint_as_float(r & 0xffff0000u);
    } else {
        const float2 f = reinterpret_cast<const float2 *>(t)[(p * cpad) / 2 + c2];
        x0 = f.x, x1 = f.y;
    }
}

// 2 channels into a (margined) buffer pixel q: bf16, or the fp32 [hi | lo] split
__device__ __forceinline__ void store2(void *dst, int esz, int split, long long q, int dcp, int c2, float x0,
                                       float x1) {
    if (esz == 2) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(x0, x1);
        reinterpret_cast<__nv_bfloat162 *>(dst)[(q * dcp) / 2 + c2] = h;
    } else if (split) {
        float *d = reinterpret_cast<float *>(dst) + q * dcp + 2 * c2;
        const float h0 = hi_tf32(x0), h1 = hi_tf32(x1);
        d[0] = h0, d[1] = h1;
        d[dcp / 2] = x0 - h0, d[dcp / 2 + 1] = x1 - h1;
    } else {
        reinterpret_cast<float2 *>(dst)[(q * dcp) / 2 + c2] = make_float2(x0, x1);
    }
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
// Backward kernels: a thread keeps ONE channel pair (4-byte loads; a warp
// covers 64 channels of a pixel, coalesced) and four pixels in flight per trip,
// with few registers, so enough warps stay resident to keep HBM busy
// (the 8-channel version with fp64 accumulators ran at 164 registers, one
// block per SM and 16% of DRAM bandwidth).
constexpr int kBnPix = 4;

__global__ void __launch_bounds__(256) bn_bwd_partials_kernel(const __grid_constant__ BnArgs a, double *partials) {
    pdl_wait();  // (launch.cuh: PDL)
    extern __shared__ double sh[];
    const int c2n = a.cpad / 2;
    const int cb = c2n < 256 ? c2n : 256, lanes = 256 / cb;
    const int pl = threadIdx.x / cb, c2 = threadIdx.x % cb;
    for (int k = threadIdx.x; k < lanes * 2 * a.cpad; k += blockDim.x) sh[k] = 0.0;
    __syncthreads();
    if (pl < lanes) {
        for (int cc = c2; cc < c2n; cc += cb) {
            const int k0 = 2 * cc;
            const float sc0 = a.coef[k0], sc1 = a.coef[k0 + 1], sf0 = a.coef[a.cpad + k0], sf1 = a.coef[a.cpad + k0 + 1];
            const float in0 = a.coef[2 * a.cpad + k0], in1 = a.coef[2 * a.cpad + k0 + 1];
            const float mu0 = a.coef[3 * a.cpad + k0], mu1 = a.coef[3 * a.cpad + k0 + 1];
            double sg0 = 0, sg1 = 0, sy0 = 0, sy1 = 0;
            const long long step = (long long)gridDim.x * lanes;
            for (long long p0 = (long long)blockIdx.x * lanes + pl; p0 < a.npix; p0 += kBnPix * step) {
                float v[kBnPix][2], d[kBnPix][2], r[kBnPix][2];
#pragma unroll
                for (int u = 0; u < kBnPix; ++u) {
                    const long long p = p0 + u * step;
                    v[u][0] = v[u][1] = d[u][0] = d[u][1] = r[u][0] = r[u][1] = 0.f;
                    if (p < a.npix) {
                        load2(a.y, a.esz, p, a.cpad, cc, v[u][0], v[u][1]);
                        load2(a.dout, a.esz, p, a.cpad, cc, d[u][0], d[u][1]);
                        if (a.res) load2(a.res, a.esz, p, a.cpad, cc, r[u][0], r[u][1]);
                    }
                }
                // fp32 sums of the trip's <= 4 pixels, then one fp64 add per
                // trip (fp64 arithmetic per element ran the kernel at 1.6 ms
                // for 2.1 GB; error <= (3 + 1) u sum|term|)
                float tg0 = 0.f, tg1 = 0.f, ty0 = 0.f, ty1 = 0.f;
#pragma unroll
                for (int u = 0; u < kBnPix; ++u) {
                    const float z0 = fmaf(sc0, v[u][0], sf0) + r[u][0], z1 = fmaf(sc1, v[u][1], sf1) + r[u][1];
                    const float g0 = (a.relu && z0 <= 0.f) ? 0.f : d[u][0];   // (padding pixels: d = 0)
                    const float g1 = (a.relu && z1 <= 0.f) ? 0.f : d[u][1];
                    tg0 += g0, tg1 += g1;
                    ty0 = fmaf(g0, (v[u][0] - mu0) * in0, ty0);
                    ty1 = fmaf(g1, (v[u][1] - mu1) * in1, ty1);
                }
                sg0 += (double)tg0, sg1 += (double)tg1, sy0 += (double)ty0, sy1 += (double)ty1;
            }
            double *row = sh + (long long)pl * 2 * a.cpad;
            row[k0] = sg0, row[k0 + 1] = sg1, row[a.cpad + k0] = sy0, row[a.cpad + k0 + 1] = sy1;
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
__global__ void __launch_bounds__(256) bn_bwd_apply_kernel(const __grid_constant__ BnArgs a, const double *sums,
                                                           double count, const float *gamma, float *dgamma,
                                                           float *dbeta, void *dres) {
    pdl_wait();  // (launch.cuh: PDL)
    if (blockIdx.x == 0)
        for (int k = threadIdx.x; k < a.c; k += blockDim.x) {
            if (dgamma) dgamma[k] = (float)sums[a.cpad + k];
            if (dbeta) dbeta[k] = (float)sums[k];
        }
    const int c2n = a.cpad / 2;
    const int cb = c2n < 256 ? c2n : 256, lanes = 256 / cb;
    const int pl = threadIdx.x / cb, c2 = threadIdx.x % cb;
    if (pl >= lanes) return;
    for (int cc = c2; cc < c2n; cc += cb) {
        // the pair's constants, once
        float sc[2], sf[2], inv[2], mu[2], k1[2], m1[2], m2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const int k = 2 * cc + e;
            sc[e] = a.coef[k], sf[e] = a.coef[a.cpad + k], inv[e] = a.coef[2 * a.cpad + k];
            mu[e] = a.coef[3 * a.cpad + k];
            const bool live = k < a.c;
            k1[e] = live ? gamma[k] * inv[e] : 0.f;
            m1[e] = live ? (float)(sums[k] / count) : 0.f;
            m2[e] = live ? (float)(sums[a.cpad + k] / count) : 0.f;
        }
        const long long step = (long long)gridDim.x * lanes;
        for (long long p0 = (long long)blockIdx.x * lanes + pl; p0 < a.npix; p0 += kBnPix * step) {
            float v[kBnPix][2], d[kBnPix][2], r[kBnPix][2];
#pragma unroll
            for (int u = 0; u < kBnPix; ++u) {
                const long long p = p0 + u * step;
                v[u][0] = v[u][1] = d[u][0] = d[u][1] = r[u][0] = r[u][1] = 0.f;
                if (p < a.npix) {
                    load2(a.y, a.esz, p, a.cpad, cc, v[u][0], v[u][1]);
                    load2(a.dout, a.esz, p, a.cpad, cc, d[u][0], d[u][1]);
                    if (a.res) load2(a.res, a.esz, p, a.cpad, cc, r[u][0], r[u][1]);
                }
            }
#pragma unroll
            for (int u = 0; u < kBnPix; ++u) {
                const long long p = p0 + u * step;
                if (p >= a.npix) break;
                float o[2], g[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const float z = fmaf(sc[e], v[u][e], sf[e]) + r[u][e];
                    g[e] = (a.relu && z <= 0.f) ? 0.f : d[u][e];
                    const float yh = (v[u][e] - mu[e]) * inv[e];
                    o[e] = k1[e] * (g[e] - m1[e] - yh * m2[e]);
                }
                store2(a.dst, a.esz, a.split, dst_pixel(a, p), a.dcp, cc, o[0], o[1]);
                if (dres) store2(dres, a.esz, 0, p, a.cpad, cc, g[0], g[1]);
            }
        }
    }
}

int bn_bwd_blocks(long long npix, int cpad) {
    const int c2n = cpad / 2, lanes = std::max(1, 256 / std::min(c2n, 256));
    const long long trips = (npix + lanes - 1) / lanes;
    return (int)std::max<long long>(1, std::min<long long>((trips + 4 * kBnPix - 1) / (4 * kBnPix), 148 * 8));
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
    DC_REQUIRE(a.cpad % 8 == 0 && a.cpad <= 4096, DC_ERR_UNSUPPORTED, "BN backward: channels");
    const int lanes = std::max(1, 256 / std::min(a.cpad / 2, 256));
    const size_t smem = (size_t)lanes * 2 * a.cpad * sizeof(double);
    static std::once_flag once;
    std::call_once(once, [] {
        cudaFuncSetAttribute(bn_bwd_partials_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    });
    launch_k(bn_bwd_partials_kernel, dim3(blocks), dim3(256), smem, st, 1, "bn bwd partials", a, partials);
}

void launch_bn_bwd_apply(const BnArgs &a, const double *sums, double count, const float *gamma, float *dgamma,
                         float *dbeta, void *dres, cudaStream_t st) {
    launch_k(bn_bwd_apply_kernel, dim3(bn_bwd_blocks(a.npix, a.cpad)), dim3(256), 0, st, 1, "bn bwd apply", a, sums,
             count, gamma, dgamma, dbeta, dres);
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

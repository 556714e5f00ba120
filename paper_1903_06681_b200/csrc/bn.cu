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

// 4 channels (quad c4) of pixel p of a dense NHWC tensor as fp32
__device__ __forceinline__ void load4(const void *t, int esz, long long p, int cpad, int c4, float (&x)[4]) {
    if (esz == 2) {
        const uint2 r = reinterpret_cast<const uint2 *>(t)[(p * cpad) / 4 + c4];
        x[0] = __uint_as_float(r.x << 16), x[1] = __uint_as_float(r.x & 0xffff0000u);
        x[2] = __uint_as_float(r.y << 16), x[3] = __uint_as_float(r.y & 0xffff0000u);
    } else {
        const float4 f = reinterpret_cast<const float4 *>(t)[(p * cpad) / 4 + c4];
        x[0] = f.x, x[1] = f.y, x[2] = f.z, x[3] = f.w;
    }
}

// 4 channels into a (margined) buffer pixel q: bf16, or the fp32 [hi | lo] split
__device__ __forceinline__ void store4(void *dst, int esz, int split, long long q, int dcp, int c4,
                                       const float (&x)[4]) {
    if (esz == 2) {
        const __nv_bfloat162 h0 = __floats2bfloat162_rn(x[0], x[1]), h1 = __floats2bfloat162_rn(x[2], x[3]);
        uint2 r;
        r.x = *reinterpret_cast<const uint32_t *>(&h0), r.y = *reinterpret_cast<const uint32_t *>(&h1);
        reinterpret_cast<uint2 *>(dst)[(q * dcp) / 4 + c4] = r;
    } else if (split) {
        float *d = reinterpret_cast<float *>(dst) + q * dcp + 4 * c4;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float h = hi_tf32(x[e]);
            d[e] = h, d[dcp / 2 + e] = x[e] - h;
        }
    } else {
        reinterpret_cast<float4 *>(dst)[(q * dcp) / 4 + c4] = make_float4(x[0], x[1], x[2], x[3]);
    }
}

// Pixel p = (n, i, j) of an n x h x w block walked with a fixed stride: the
// margined-buffer position without a division per step.
struct PixWalk {
    int n, i, j, sn, si, sj;
    __device__ __forceinline__ void init(const BnArgs &a, long long p, long long step) {
        j = (int)(p % a.w), i = (int)((p / a.w) % a.h), n = (int)(p / ((long long)a.w * a.h));
        sj = (int)(step % a.w), si = (int)((step / a.w) % a.h), sn = (int)(step / ((long long)a.w * a.h));
    }
    __device__ __forceinline__ void next(const BnArgs &a) {
        j += sj, i += si, n += sn;
        if (j >= a.w) j -= a.w, ++i;
        if (i >= a.h) i -= a.h, ++n;
    }
    __device__ __forceinline__ long long pos(const BnArgs &a) const {
        return ((long long)n * a.hb + a.r0 + i) * a.wb + a.c0 + j;
    }
};

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
// Backward kernels: a thread keeps ONE quad of channels (8-byte loads; a
// warp covers 128 channels of a pixel, coalesced) with its per-channel
// constants in registers, and two pixels in flight per trip; the margined
// output position is walked, not divided out. (The 8-channel version with
// fp64 accumulators ran at 164 registers and 16% of DRAM bandwidth; a
// 2-channel one at 4-byte loads and a 64-bit division per pixel at 19%.)
constexpr int kBnPix = 2;

__global__ void __launch_bounds__(256, 3) bn_bwd_partials_kernel(const __grid_constant__ BnArgs a, double *partials) {
    pdl_wait();  // (launch.cuh: PDL)
    extern __shared__ double sh[];
    const int c4n = a.cpad / 4;
    const int cb = c4n < 256 ? c4n : 256, lanes = 256 / cb;
    const int pl = threadIdx.x / cb, c4 = threadIdx.x % cb;
    for (int k = threadIdx.x; k < lanes * 2 * a.cpad; k += blockDim.x) sh[k] = 0.0;
    __syncthreads();
    if (pl < lanes) {
        for (int cc = c4; cc < c4n; cc += cb) {
            float sc[4], sf[4], inv[4], mu[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int k = 4 * cc + e;
                sc[e] = a.coef[k], sf[e] = a.coef[a.cpad + k], inv[e] = a.coef[2 * a.cpad + k];
                mu[e] = a.coef[3 * a.cpad + k];
            }
            double sg[4] = {0, 0, 0, 0}, sy[4] = {0, 0, 0, 0};
            const long long step = (long long)gridDim.x * lanes;
            for (long long p0 = (long long)blockIdx.x * lanes + pl; p0 < a.npix; p0 += kBnPix * step) {
                float v[kBnPix][4], d[kBnPix][4], r[kBnPix][4];
#pragma unroll
                for (int u = 0; u < kBnPix; ++u) {
                    const long long p = p0 + u * step;
#pragma unroll
                    for (int e = 0; e < 4; ++e) v[u][e] = d[u][e] = r[u][e] = 0.f;
                    if (p < a.npix) {
                        load4(a.y, a.esz, p, a.cpad, cc, v[u]);
                        load4(a.dout, a.esz, p, a.cpad, cc, d[u]);
                        if (a.res) load4(a.res, a.esz, p, a.cpad, cc, r[u]);
                    }
                }
                // fp32 sums of the trip's pixels, then one fp64 add per trip
                // (fp64 per element was slow; error bound: DESIGN.md §7)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    float tg = 0.f, ty = 0.f;
#pragma unroll
                    for (int u = 0; u < kBnPix; ++u) {
                        const float z = fmaf(sc[e], v[u][e], sf[e]) + r[u][e];
                        const float g = (a.relu && z <= 0.f) ? 0.f : d[u][e];  // (padding pixels: d = 0)
                        tg += g;
                        ty = fmaf(g, (v[u][e] - mu[e]) * inv[e], ty);
                    }
                    sg[e] += (double)tg, sy[e] += (double)ty;
                }
            }
            double *row = sh + (long long)pl * 2 * a.cpad;
#pragma unroll
            for (int e = 0; e < 4; ++e) row[4 * cc + e] = sg[e], row[a.cpad + 4 * cc + e] = sy[e];
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
__global__ void __launch_bounds__(256, 3) bn_bwd_apply_kernel(const __grid_constant__ BnArgs a, const double *sums,
                                                           double count, const float *gamma, float *dgamma,
                                                           float *dbeta, void *dres) {
    pdl_wait();  // (launch.cuh: PDL)
    if (blockIdx.x == 0)
        for (int k = threadIdx.x; k < a.c; k += blockDim.x) {
            if (dgamma) dgamma[k] = (float)sums[a.cpad + k];
            if (dbeta) dbeta[k] = (float)sums[k];
        }
    const int c4n = a.cpad / 4;
    const int cb = c4n < 256 ? c4n : 256, lanes = 256 / cb;
    const int pl = threadIdx.x / cb, c4 = threadIdx.x % cb;
    if (pl >= lanes) return;
    for (int cc = c4; cc < c4n; cc += cb) {
        // the quad's constants, once
        float sc[4], sf[4], inv[4], mu[4], k1[4], m1[4], m2[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int k = 4 * cc + e;
            sc[e] = a.coef[k], sf[e] = a.coef[a.cpad + k], inv[e] = a.coef[2 * a.cpad + k];
            mu[e] = a.coef[3 * a.cpad + k];
            const bool live = k < a.c;
            k1[e] = live ? gamma[k] * inv[e] : 0.f;
            m1[e] = live ? (float)(sums[k] / count) : 0.f;
            m2[e] = live ? (float)(sums[a.cpad + k] / count) : 0.f;
        }
        const long long step = (long long)gridDim.x * lanes;
        long long p = (long long)blockIdx.x * lanes + pl;
        if (p >= a.npix) continue;
        PixWalk q;
        q.init(a, p, step);
        while (p < a.npix) {
            float v[kBnPix][4], d[kBnPix][4], r[kBnPix][4];
#pragma unroll
            for (int u = 0; u < kBnPix; ++u) {
                const long long pu = p + u * step;
#pragma unroll
                for (int e = 0; e < 4; ++e) v[u][e] = d[u][e] = r[u][e] = 0.f;
                if (pu < a.npix) {
                    load4(a.y, a.esz, pu, a.cpad, cc, v[u]);
                    load4(a.dout, a.esz, pu, a.cpad, cc, d[u]);
                    if (a.res) load4(a.res, a.esz, pu, a.cpad, cc, r[u]);
                }
            }
#pragma unroll
            for (int u = 0; u < kBnPix; ++u) {
                if (p >= a.npix) break;
                float o[4], g[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const float z = fmaf(sc[e], v[u][e], sf[e]) + r[u][e];
                    g[e] = (a.relu && z <= 0.f) ? 0.f : d[u][e];
                    const float yh = (v[u][e] - mu[e]) * inv[e];
                    o[e] = k1[e] * (g[e] - m1[e] - yh * m2[e]);
                }
                store4(a.dst, a.esz, a.split, q.pos(a), a.dcp, cc, o);
                if (dres) store4(dres, a.esz, 0, p, a.cpad, cc, g);
                p += step;
                q.next(a);
            }
        }
    }
}

int bn_bwd_blocks(long long npix, int cpad) {
    const int c4n = cpad / 4, lanes = std::max(1, 256 / std::min(c4n, 256));
    const long long trips = (npix + lanes - 1) / lanes;
    return (int)std::max<long long>(1, std::min<long long>((trips + 8 * kBnPix - 1) / (8 * kBnPix), 148 * 8));
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
    const int lanes = std::max(1, 256 / std::min(a.cpad / 4, 256));
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

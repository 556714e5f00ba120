// bn.cu -- the layers between the convolutions on the same decomposition
// (PAPER.md:149, 234-236): batch-norm apply with the
// spatially aggregated statistics (+ residual add, ReLU), written straight
// into the next layer's margined input, and its backward, whose per-channel
// sums sum(g), sum(g y_hat) are aggregated over the spatial group like the
// forward statistics, and the statistics pass itself.
// Memory-bound elementwise / reduction kernels: the inputs stream through a
// ring of shared-memory stages filled by bulk copies (bn_staged_kernel), one
// consumer thread per 8 channels of a pixel.
#include <cuda_bf16.h>

#include <mutex>

#include "bn.cuh"
#include "common.hpp"
#include "launch.cuh"
#include "sm100.cuh"

namespace dc {

namespace {
__device__ __forceinline__ float hi_tf32(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }

// 8 channels into a (margined) buffer pixel q: bf16, or the fp32 [hi | lo] split
__device__ __forceinline__ void store8(void *dst, int esz, int split, long long q, int dcp, int c8,
                                       const float (&v)[8]) {
    if (esz == 2) {
        uint4 r;
        __nv_bfloat16 *h = reinterpret_cast<__nv_bfloat16 *>(&r);
#pragma unroll
        for (int e = 0; e < 8; ++e) h[e] = __float2bfloat16_rn(v[e]);
        reinterpret_cast<uint4 *>(dst)[(unsigned long long)q * dcp / 8 + c8] = r;
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

// 8 channels at byte offset `off` of a staged chunk (bf16 or fp32) as fp32
template <int ESZ>
__device__ __forceinline__ void lds8(const unsigned char *chunk, uint32_t off, float (&v)[8]) {
    if (ESZ == 2) {
        const uint4 r = *reinterpret_cast<const uint4 *>(chunk + off);
        const uint32_t w[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) v[2 * e] = __uint_as_float(w[e] << 16), v[2 * e + 1] = __uint_as_float(w[e] & 0xffff0000u);
    } else {
        const float4 *f = reinterpret_cast<const float4 *>(chunk + off);
        const float4 x = f[0], y = f[1];
        v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w, v[4] = y.x, v[5] = y.y, v[6] = y.z, v[7] = y.w;
    }
}

// n / d for 32-bit n by a multiply-high (Granlund-Montgomery; d >= 1)
struct FastDiv {
    uint32_t m, l;
    __device__ __forceinline__ void init(uint32_t d) {
        l = d > 1 ? 32 - __clz(d - 1) : 0;  // ceil(log2 d)
        m = (uint32_t)((((1ull << l) - d) << 32) / d + 1);
    }
    __device__ __forceinline__ uint32_t div(uint32_t n) const {
        if (l == 0) return n;
        const uint32_t t = __umulhi(m, n);
        return (t + ((n - t) >> 1)) >> (l - 1);
    }
};

// pixel p = (n, i, j) of the n x h x w block -> its pixel in the margined dst
struct DstMap {
    FastDiv fw, fh;
    __device__ __forceinline__ void init(const BnArgs &a) { fw.init(a.w), fh.init(a.h); }
    __device__ __forceinline__ long long pos(const BnArgs &a, uint32_t p) const {
        const uint32_t r = fw.div(p), j = p - r * a.w, n = fh.div(r), i = r - n * a.h;
        return ((long long)n * a.hb + a.r0 + i) * a.wb + a.c0 + j;
    }
};
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

// The three passes over a shard (forward apply; backward partial sums;
// backward apply) stream their dense inputs -- y, dout, the residual --
// through shared memory: a producer warp issues one bulk copy per tensor per
// chunk of P whole pixels (TMA, cp.async.bulk) into a ring of stages, 16
// consumer warps evaluate it. The copies in flight do not depend on the
// consumers' registers, which hold one 8-channel group's constants: thread t
// keeps channel group c8 = t % (cpad / 8) for the whole launch and takes pixel
// lanes t / (cpad / 8), t / (cpad / 8) + lanes, ... of every chunk. (The
// register-staged kernels before this -- 4 or 8 channels, 1-4 pixels in
// flight per thread -- ran the backward at 1.3-1.9 TB/s, bound by the loads a
// thread could keep in flight next to its constants.)
constexpr int kBnWarps = 12, kBnThreads = 32 * kBnWarps, kBnMaxStages = 8;
constexpr size_t kBnRingBytes = 192 * 1024;

struct BnRing {
    long long nchunks;
    int P, stages;
};

enum { kBnFwdApply = 0, kBnBwdPartials = 1, kBnBwdApply = 2, kBnStats = 3 };

template <int MODE, int ESZ, bool RES, bool RELU>
__global__ void __launch_bounds__(kBnThreads + 32, 1)
    bn_staged_kernel(const __grid_constant__ BnArgs a, const __grid_constant__ BnRing r, double *partials,
                     const double *sums, double count, const float *gamma, float *dgamma, float *dbeta, void *dres) {
    constexpr int T = (MODE == kBnFwdApply || MODE == kBnStats ? 1 : 2) + (RES ? 1 : 0);  // y, dout, res
    constexpr int PPT = (ESZ == 2 ? 2 : 1) * (MODE == kBnStats ? 2 : 1);  // pixels per thread per chunk
    extern __shared__ __align__(128) unsigned char ring[];
    __shared__ uint64_t full[kBnMaxStages], empty[kBnMaxStages];
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rowb = (uint32_t)a.cpad * ESZ, chunkb = (uint32_t)r.P * rowb;
    if (threadIdx.x == 0) {
        for (int s = 0; s < r.stages; ++s) sm100::mbar_init(&full[s], 1), sm100::mbar_init(&empty[s], kBnWarps);
        sm100::fence_mbar_init();
    }
    __syncthreads();
    pdl_wait();  // (launch.cuh: PDL)

    const int c8n = a.cpad / 8, lanes = kBnThreads / c8n;
    const int c8 = threadIdx.x % c8n, pl = threadIdx.x / c8n;
    const bool active = warp < kBnWarps && pl < lanes;
    double sg[8], sy[8];  // (kBnBwdPartials, kBnStats)
#pragma unroll
    for (int e = 0; e < 8; ++e) sg[e] = sy[e] = 0.0;

    if (warp == kBnWarps) {  // producer
        if (lane == 0) {
            const unsigned char *src[3] = {static_cast<const unsigned char *>(a.y),
                                           static_cast<const unsigned char *>(MODE == kBnFwdApply ? a.res : a.dout),
                                           static_cast<const unsigned char *>(a.res)};
            int s = 0;
            uint32_t ph = 0;
            for (long long k = blockIdx.x; k < r.nchunks; k += gridDim.x) {
                sm100::mbar_wait(&empty[s], ph ^ 1);
                const long long p0 = k * r.P;
                const uint32_t bytes = (uint32_t)(a.npix - p0 < r.P ? a.npix - p0 : (long long)r.P) * rowb;
                sm100::mbar_arrive_expect_tx(&full[s], T * bytes);
                unsigned char *dst = ring + (size_t)s * T * chunkb;
#pragma unroll
                for (int j = 0; j < T; ++j)
                    sm100::bulk_load_1d(dst + j * chunkb, src[j] + (size_t)p0 * rowb, bytes, &full[s]);
                if (++s == r.stages) s = 0, ph ^= 1;
            }
        }
        __syncwarp();
    } else {
        // the channel group's constants (kBnBwdApply: dy = k1 (g - m1 - y_hat m2))
        float sc[8], sf[8], mu[8], inv[8], k1[8], m1[8], m2[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const int k = 8 * c8 + e;
            sc[e] = sf[e] = mu[e] = inv[e] = k1[e] = m1[e] = m2[e] = 0.f;
            if (MODE != kBnStats) sc[e] = a.coef[k], sf[e] = a.coef[a.cpad + k];
            if (MODE == kBnBwdPartials || MODE == kBnBwdApply) inv[e] = a.coef[2 * a.cpad + k], mu[e] = a.coef[3 * a.cpad + k];
            if (MODE == kBnBwdApply && k < a.c) {
                k1[e] = gamma[k] * inv[e];
                m1[e] = (float)(sums[k] / count);
                m2[e] = (float)(sums[a.cpad + k] / count);
            }
        }
        DstMap dm;
        if (MODE == kBnFwdApply || MODE == kBnBwdApply) dm.init(a);
        unsigned char *const dst = static_cast<unsigned char *>(a.dst);
        const uint32_t c8b = (uint32_t)c8 * 8 * ESZ;
        int s = 0;
        uint32_t ph = 0;
        for (long long k = blockIdx.x; k < r.nchunks; k += gridDim.x) {
            sm100::mbar_wait(&full[s], ph);
            const unsigned char *yc = ring + (size_t)s * T * chunkb;
            const long long p0 = k * r.P;
            const int np = (int)(a.npix - p0 < r.P ? a.npix - p0 : (long long)r.P);
            float tg[8], ty[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) tg[e] = ty[e] = 0.f;
#pragma unroll
            for (int u = 0; u < PPT; ++u) {
                const int pp = pl + u * lanes;
                if (!active || pp >= np) break;
                const uint32_t off = (uint32_t)pp * rowb + c8b;
                float v[8], d[8], rr[8];
                lds8<ESZ>(yc, off, v);
                if (MODE == kBnBwdPartials || MODE == kBnBwdApply) lds8<ESZ>(yc + chunkb, off, d);
                if (RES) lds8<ESZ>(yc + (T - 1) * chunkb, off, rr);
                if (MODE == kBnStats) {
                    // sum y, sum y^2 (y^2 of a bf16 is exact in fp32)
#pragma unroll
                    for (int e = 0; e < 8; ++e) tg[e] += v[e], ty[e] = fmaf(v[e], v[e], ty[e]);
                } else if (MODE == kBnFwdApply) {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        float z = fmaf(sc[e], v[e], sf[e]);
                        if (RES) z += rr[e];
                        v[e] = (RELU && z < 0.f) ? 0.f : z;
                    }
                    store8(dst, ESZ, a.split, dm.pos(a, (uint32_t)(p0 + pp)), a.dcp, c8, v);
                } else {
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                        float z = fmaf(sc[e], v[e], sf[e]);
                        if (RES) z += rr[e];
                        d[e] = (RELU && z <= 0.f) ? 0.f : d[e];  // g
                    }
                    if (MODE == kBnBwdPartials) {
                        // fp32 sums of this chunk's <= 2 pixels, then one fp64 add
                        // per chunk (error bound: DESIGN.md §7)
#pragma unroll
                        for (int e = 0; e < 8; ++e) tg[e] += d[e], ty[e] = fmaf(d[e], (v[e] - mu[e]) * inv[e], ty[e]);
                    } else {
                        float o[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) o[e] = k1[e] * (d[e] - m1[e] - (v[e] - mu[e]) * inv[e] * m2[e]);
                        store8(dst, ESZ, a.split, dm.pos(a, (uint32_t)(p0 + pp)), a.dcp, c8, o);
                        if (RES && dres) store8(dres, ESZ, 0, p0 + pp, a.cpad, c8, d);
                    }
                }
            }
            if (MODE == kBnBwdPartials || MODE == kBnStats) {
#pragma unroll
                for (int e = 0; e < 8; ++e) sg[e] += (double)tg[e], sy[e] += (double)ty[e];
            }
            __syncwarp();
            if (lane == 0) sm100::mbar_arrive(&empty[s]);
            if (++s == r.stages) s = 0, ph ^= 1;
        }
    }
    if (MODE == kBnBwdPartials || MODE == kBnStats) {  // the block's sums per channel -> partials[block][2][cpad]
        __syncthreads();           // (every chunk consumed: the ring is free)
        double *red = reinterpret_cast<double *>(ring);
        if (active) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                red[(size_t)pl * 2 * a.cpad + 8 * c8 + e] = sg[e];
                red[(size_t)pl * 2 * a.cpad + a.cpad + 8 * c8 + e] = sy[e];
            }
        }
        __syncthreads();
        for (int k = threadIdx.x; k < 2 * a.cpad; k += blockDim.x) {
            double acc = 0.0;
            for (int l = 0; l < lanes; ++l) acc += red[(size_t)l * 2 * a.cpad + k];
            partials[(size_t)blockIdx.x * 2 * a.cpad + k] = acc;
        }
    }
    if (MODE == kBnBwdApply && blockIdx.x == 0)
        for (int k = threadIdx.x; k < a.c; k += blockDim.x) {
            if (dgamma) dgamma[k] = (float)sums[a.cpad + k];
            if (dbeta) dbeta[k] = (float)sums[k];
        }
}

using BnKernel = void (*)(BnArgs, BnRing, double *, const double *, double, const float *, float *, float *, void *);

template <int MODE>
BnKernel staged_kernel(int esz, bool res, bool relu) {
    if (esz == 2)
        return res ? (relu ? bn_staged_kernel<MODE, 2, true, true> : bn_staged_kernel<MODE, 2, true, false>)
                   : (relu ? bn_staged_kernel<MODE, 2, false, true> : bn_staged_kernel<MODE, 2, false, false>);
    return res ? (relu ? bn_staged_kernel<MODE, 4, true, true> : bn_staged_kernel<MODE, 4, true, false>)
               : (relu ? bn_staged_kernel<MODE, 4, false, true> : bn_staged_kernel<MODE, 4, false, false>);
}

template <typename F>
void for_each_staged(F &&f) {
    for (int esz : {2, 4})
        for (int res = 0; res < 2; ++res)
            for (int relu = 0; relu < 2; ++relu) {
                f(staged_kernel<kBnFwdApply>(esz, res, relu));
                f(staged_kernel<kBnBwdPartials>(esz, res, relu));
                f(staged_kernel<kBnBwdApply>(esz, res, relu));
            }
    f(bn_staged_kernel<kBnStats, 2, false, false>);
}

void launch_bn_coeff(const double *mean, const double *var, const float *gamma, const float *beta, double eps,
                     int c, int cpad, float *coef, cudaStream_t st) {
    launch_k(bn_coeff_kernel, dim3((cpad + 255) / 256), dim3(256), 0, st, 1, "bn coeff", mean, var, gamma, beta,
             eps, c, cpad, coef);
}

namespace {
BnRing bn_ring(const BnArgs &a, int tensors, bool stats) {
    DC_REQUIRE(a.cpad % 8 == 0 && a.cpad <= 8 * kBnThreads && a.dcp % 8 == 0, DC_ERR_UNSUPPORTED,
               "BN: channels must be multiples of 8, at most %d", 8 * kBnThreads);
    DC_REQUIRE(a.npix < (1ll << 31), DC_ERR_UNSUPPORTED, "BN: more than 2^31 pixels per shard");
    for (const void *t : {a.y, a.dout, a.res})
        DC_REQUIRE(reinterpret_cast<uintptr_t>(t) % 16 == 0, DC_ERR_ARG, "BN: tensors must be 16-byte aligned");
    BnRing r;
    const int lanes = kBnThreads / (a.cpad / 8);
    r.P = (a.esz == 2 ? 2 : 1) * (stats ? 2 : 1) * lanes;  // 12 KB per tensor (statistics: 24 KB)
    r.nchunks = (a.npix + r.P - 1) / r.P;
    const size_t stage = (size_t)tensors * r.P * a.cpad * a.esz;
    r.stages = (int)std::min<size_t>(kBnMaxStages, kBnRingBytes / stage);
    return r;
}

size_t bn_smem(const BnArgs &a, const BnRing &r, int tensors) {
    const size_t ring = (size_t)r.stages * tensors * r.P * a.cpad * a.esz;
    const size_t red = (size_t)(kBnThreads / (a.cpad / 8)) * 2 * a.cpad * sizeof(double);
    return std::max(ring, red);
}

template <int MODE>
void launch_staged(const BnArgs &a, int blocks, double *partials, const double *sums, double count,
                   const float *gamma, float *dgamma, float *dbeta, void *dres, cudaStream_t st, const char *what) {
    DC_REQUIRE(a.esz == 2 || a.esz == 4, DC_ERR_ARG, "BN: element size %d", a.esz);
    const int tensors = (MODE == kBnFwdApply || MODE == kBnStats ? 1 : 2) + (a.res ? 1 : 0);
    const BnRing r = bn_ring(a, tensors, MODE == kBnStats);
    static std::once_flag once;
    std::call_once(once, [] {
        for_each_staged([](BnKernel k) {
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBnRingBytes);
        });
    });
    BnKernel k;
    if constexpr (MODE == kBnStats)
        k = bn_staged_kernel<kBnStats, 2, false, false>;
    else
        k = staged_kernel<MODE>(a.esz, a.res != nullptr, a.relu != 0);
    launch_k(k, dim3(blocks), dim3(kBnThreads + 32),
             bn_smem(a, r, tensors), st, 1, what, a, r, partials, sums, count, gamma, dgamma, dbeta, dres);
}
}  // namespace

int bn_bwd_blocks(const BnArgs &a) {
    const int lanes = kBnThreads / std::max(1, a.cpad / 8);
    const long long P = (a.esz == 2 ? 2 : 1) * lanes;
    return (int)std::max<long long>(1, std::min<long long>((a.npix + P - 1) / P, 148));
}

void launch_bn_apply(const BnArgs &a, cudaStream_t st) {
    if (a.npix == 0) return;
    launch_staged<kBnFwdApply>(a, bn_bwd_blocks(a), nullptr, nullptr, 0.0, nullptr, nullptr, nullptr, nullptr, st,
                               "bn apply");
}

void launch_bn_bwd_partials(const BnArgs &a, double *partials, int blocks, cudaStream_t st) {
    launch_staged<kBnBwdPartials>(a, blocks, partials, nullptr, 0.0, nullptr, nullptr, nullptr, nullptr, st,
                                  "bn bwd partials");
}

void launch_bn_bwd_apply(const BnArgs &a, const double *sums, double count, const float *gamma, float *dgamma,
                         float *dbeta, void *dres, cudaStream_t st) {
    launch_staged<kBnBwdApply>(a, bn_bwd_blocks(a), nullptr, sums, count, gamma, dgamma, dbeta, dres, st,
                               "bn bwd apply");
}

int bn_stats_blocks(long long npix, int cpad) {
    BnArgs a{};
    a.npix = npix, a.cpad = cpad, a.esz = 2;
    return bn_bwd_blocks(a);
}

void launch_bn_stats(const void *y, long long npix, int cpad, double *partials, int blocks, cudaStream_t st) {
    if (npix == 0) return;
    BnArgs a{};
    a.y = y, a.npix = npix, a.cpad = cpad, a.c = cpad, a.esz = 2, a.dcp = cpad;
    launch_staged<kBnStats>(a, blocks, partials, nullptr, 0.0, nullptr, nullptr, nullptr, nullptr, st, "bn stats");
}

// Loads this file's kernels (see preload_conv_v2)
void preload_bn() {
    cudaFuncAttributes at;
    cudaFuncGetAttributes(&at, reinterpret_cast<const void *>(bn_coeff_kernel));
    for_each_staged([&](BnKernel k) {
        cudaFuncGetAttributes(&at, reinterpret_cast<const void *>(k));
        // (set here, at communicator creation, so that no first launch inside
        // a stream capture has to change a function attribute)
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kBnRingBytes);
    });
}

}  // namespace dc

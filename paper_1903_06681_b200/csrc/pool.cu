// pool.cu -- max pooling forward / backward on a rank's shard (pool.cuh).
// Memory-bound: one thread per (pixel, 8-channel vector), 16-byte loads and
// stores along the contiguous channel run; the window reads of neighbouring
// threads hit the same lines in L1 / L2.
#include <cuda_bf16.h>

#include "common.hpp"
#include "launch.cuh"
#include "pool.cuh"

namespace dc {

namespace {

__device__ __forceinline__ void unpack8(const uint4 &v, float (&f)[8]) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        f[2 * k] = __uint_as_float(w[k] << 16);
        f[2 * k + 1] = __uint_as_float(w[k] & 0xffff0000u);
    }
}

__device__ __forceinline__ uint32_t pack2_rn(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t *>(&v);
}

__global__ void __launch_bounds__(256) maxpool_fwd_kernel(const __grid_constant__ PoolGeom g,
                                                          const uint4 *__restrict__ x, uint4 *__restrict__ y) {
    pdl_wait();  // (launch.cuh: PDL)
    const int vecs = g.cpad / 8;
    const long long total = (long long)g.n * g.oh * g.ow * vecs;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int v = (int)(idx % vecs);
        long long p = idx / vecs;
        const int j = (int)(p % g.ow);
        p /= g.ow;
        const int i = (int)(p % g.oh);
        const int n = (int)(p / g.oh);
        const int r0 = g.S * (g.oh0 + i) - g.P, c0 = g.S * (g.ow0 + j) - g.P;
        uint4 best = make_uint4(0, 0, 0, 0);
        float bf[8];
        bool any = false;
        for (int a = 0; a < g.K; ++a) {
            const int r = r0 + a;
            if (r < 0 || r >= g.H) continue;
            for (int b = 0; b < g.K; ++b) {
                const int c = c0 + b;
                if (c < 0 || c >= g.W) continue;
                const uint4 val = x[(((long long)n * g.xhb + (r - g.xr0)) * g.xwb + (c - g.xc0)) * vecs + v];
                float f[8];
                unpack8(val, f);
                if (!any) {
                    best = val;
#pragma unroll
                    for (int e = 0; e < 8; ++e) bf[e] = f[e];
                    any = true;
                    continue;
                }
                uint32_t w[4] = {best.x, best.y, best.z, best.w};
                const uint32_t vw[4] = {val.x, val.y, val.z, val.w};
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    if (f[e] > bf[e]) {  // strictly greater: the first maximum stays
                        bf[e] = f[e];
                        const int k = e >> 1;
                        const uint32_t m = (e & 1) ? 0xffff0000u : 0x0000ffffu;
                        w[k] = (w[k] & ~m) | (vw[k] & m);
                    }
                best = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
        y[(((long long)n * g.oh + i) * g.ow + j) * vecs + v] = best;
    }
}

__global__ void __launch_bounds__(256) maxpool_bwd_kernel(const __grid_constant__ PoolGeom g,
                                                          const uint4 *__restrict__ x, const uint4 *__restrict__ dy,
                                                          uint4 *__restrict__ dx) {
    pdl_wait();  // (launch.cuh: PDL)
    const int vecs = g.cpad / 8;
    const long long total = (long long)g.n * g.ih * g.iw * vecs;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const int v = (int)(idx % vecs);
        long long p = idx / vecs;
        const int cc = (int)(p % g.iw);
        p /= g.iw;
        const int rr = (int)(p % g.ih);
        const int n = (int)(p / g.ih);
        const int gi = g.gi0 + rr, gj = g.gj0 + cc;
        float acc[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = 0.f;
        // windows (oh, ow) that contain (gi, gj): S oh - P <= gi <= S oh - P + K - 1
        const int oh_lo = max(0, (gi + g.P - g.K + 1 + g.S - 1 + g.S * g.K) / g.S - g.K);
        const int oh_hi = min(g.Ho - 1, (gi + g.P) / g.S);
        const int ow_lo = max(0, (gj + g.P - g.K + 1 + g.S - 1 + g.S * g.K) / g.S - g.K);
        const int ow_hi = min(g.Wo - 1, (gj + g.P) / g.S);
        for (int oh = oh_lo; oh <= oh_hi; ++oh)
            for (int ow = ow_lo; ow <= ow_hi; ++ow) {
                // first maximum of the window, per channel
                float bf[8];
                int br[8], bc[8];
                bool any = false;
                const int r0 = g.S * oh - g.P, c0 = g.S * ow - g.P;
                for (int a = 0; a < g.K; ++a) {
                    const int r = r0 + a;
                    if (r < 0 || r >= g.H) continue;
                    for (int b = 0; b < g.K; ++b) {
                        const int c = c0 + b;
                        if (c < 0 || c >= g.W) continue;
                        float f[8];
                        unpack8(x[(((long long)n * g.xhb + (r - g.xr0)) * g.xwb + (c - g.xc0)) * vecs + v], f);
#pragma unroll
                        for (int e = 0; e < 8; ++e)
                            if (!any || f[e] > bf[e]) bf[e] = f[e], br[e] = r, bc[e] = c;
                        any = true;
                    }
                }
                float d[8];
                unpack8(dy[(((long long)n * g.dhb + (oh - g.dr0)) * g.dwb + (ow - g.dc0)) * vecs + v], d);
#pragma unroll
                for (int e = 0; e < 8; ++e)
                    if (br[e] == gi && bc[e] == gj) acc[e] += d[e];
            }
        uint4 o;
        o.x = pack2_rn(acc[0], acc[1]), o.y = pack2_rn(acc[2], acc[3]);
        o.z = pack2_rn(acc[4], acc[5]), o.w = pack2_rn(acc[6], acc[7]);
        dx[(((long long)n * g.ih + rr) * g.iw + cc) * vecs + v] = o;
    }
}

int blocks_for(long long work) {
    return (int)std::max<long long>(1, std::min<long long>((work + 255) / 256, 148 * 16));
}

}  // namespace

void launch_maxpool_fwd(const PoolGeom &g, const void *x, void *y, cudaStream_t st) {
    const long long work = (long long)g.n * g.oh * g.ow * (g.cpad / 8);
    if (work == 0) return;
    launch_k(maxpool_fwd_kernel, dim3(blocks_for(work)), dim3(256), 0, st, 1, "maxpool fwd", g,
             reinterpret_cast<const uint4 *>(x), reinterpret_cast<uint4 *>(y));
}

void launch_maxpool_bwd(const PoolGeom &g, const void *x, const void *dy, void *dx, cudaStream_t st) {
    const long long work = (long long)g.n * g.ih * g.iw * (g.cpad / 8);
    if (work == 0) return;
    launch_k(maxpool_bwd_kernel, dim3(blocks_for(work)), dim3(256), 0, st, 1, "maxpool bwd", g,
             reinterpret_cast<const uint4 *>(x), reinterpret_cast<const uint4 *>(dy), reinterpret_cast<uint4 *>(dx));
}

// (CUDA lazy loading: see preload_halo)
void preload_pool() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(maxpool_fwd_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(maxpool_bwd_kernel));
}

}  // namespace dc

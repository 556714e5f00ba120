// cfpar.cu -- channel / filter parallelism: handshake, wait and the rank-order
// reduce of the fp32 partial sums (cfpar.cuh).
#include <cuda_bf16.h>

#include "cfpar.cuh"
#include "common.hpp"
#include "launch.cuh"

namespace dc {

namespace {

__global__ void __launch_bounds__(32) cf_handshake_kernel(const __grid_constant__ CfFlags f) {
    pdl_wait();  // (launch.cuh: PDL)
    const uint32_t e = *reinterpret_cast<const volatile uint32_t *>(f.epoch) + 1;
    const int n_in = f.n_in > 0 ? f.n_in : f.n;
    if ((int)threadIdx.x < f.n) {
        __threadfence_system();
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(f.out[threadIdx.x]), "r"(e) : "memory");
    }
    if ((int)threadIdx.x < n_in) spin_until_geq(f.in[threadIdx.x], e);
    __syncwarp();
    __threadfence_system();
}

__global__ void __launch_bounds__(32) cf_wait_kernel(const __grid_constant__ CfFlags f) {
    pdl_wait();  // (launch.cuh: PDL)
    const uint32_t e = *reinterpret_cast<const volatile uint32_t *>(f.epoch) + 1;
    const int n_in = f.n_in > 0 ? f.n_in : f.n;
    if ((int)threadIdx.x < n_in) spin_until_geq(f.in[threadIdx.x], e);
    __syncwarp();
    __threadfence_system();
    if (f.publish && threadIdx.x == 0) *reinterpret_cast<volatile uint32_t *>(f.epoch) = e;
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<const uint32_t *>(&v);
}

__global__ void __launch_bounds__(256) cf_reduce_kernel(const float *__restrict__ slots, int n, long long slot,
                                                        long long npix, int seg, __nv_bfloat16 *__restrict__ out,
                                                        int out_pitch, uint32_t *epoch) {
    pdl_wait();  // (launch.cuh: PDL)
    const int vecs = seg / 8;
    const long long total = npix * vecs;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < total;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long pix = idx / vecs;
        const int v = (int)(idx - pix * vecs);
        const float *src = slots + pix * seg + v * 8;
        // (the senders wrote these over the system fabric: uncached loads)
        float4 a = __ldcv(reinterpret_cast<const float4 *>(src)), b = __ldcv(reinterpret_cast<const float4 *>(src) + 1);
        for (int s = 1; s < n; ++s) {
            const float4 c = __ldcv(reinterpret_cast<const float4 *>(src + s * slot));
            const float4 d = __ldcv(reinterpret_cast<const float4 *>(src + s * slot) + 1);
            a.x += c.x, a.y += c.y, a.z += c.z, a.w += c.w;
            b.x += d.x, b.y += d.y, b.z += d.z, b.w += d.w;
        }
        uint4 o;
        o.x = pack_bf16x2(a.x, a.y), o.y = pack_bf16x2(a.z, a.w);
        o.z = pack_bf16x2(b.x, b.y), o.w = pack_bf16x2(b.z, b.w);
        *reinterpret_cast<uint4 *>(out + pix * out_pitch + v * 8) = o;
    }
    __syncthreads();
    if (threadIdx.x == 0) {  // the last block publishes the epoch and resets the count
        const uint32_t prev = atomicAdd(epoch + 1, 1u);
        if (prev == gridDim.x - 1) {
            epoch[1] = 0;
            __threadfence();
            *reinterpret_cast<volatile uint32_t *>(epoch) = epoch[0] + 1;
        }
    }
}

}  // namespace

void launch_cf_handshake(const CfFlags &f, cudaStream_t st) {
    DC_REQUIRE(f.n >= 0 && f.n <= kCfMaxGroup && f.n_in >= 0 && f.n_in <= kCfMaxGroup, DC_ERR_ARG,
               "flag group of %d / %d", f.n, f.n_in);
    launch_k(cf_handshake_kernel, dim3(1), dim3(32), 0, st, 1, "cf handshake", f);
}

void launch_cf_wait(const CfFlags &f, cudaStream_t st) {
    DC_REQUIRE(f.n >= 0 && f.n <= kCfMaxGroup && f.n_in >= 0 && f.n_in <= kCfMaxGroup, DC_ERR_ARG,
               "flag group of %d / %d", f.n, f.n_in);
    launch_k(cf_wait_kernel, dim3(1), dim3(32), 0, st, 1, "cf wait", f);
}

void launch_cf_reduce(const float *slots, int n, long long slot_stride, long long npix, int seg, void *out,
                      int out_pitch, uint32_t *epoch, cudaStream_t st) {
    DC_REQUIRE(seg % 8 == 0 && out_pitch % 8 == 0, DC_ERR_ARG, "cf reduce: channel blocks of 8");
    const long long work = npix * (seg / 8);
    const int blocks = (int)std::max<long long>(1, std::min<long long>((work + 255) / 256, 148 * 8));
    launch_k(cf_reduce_kernel, dim3(blocks), dim3(256), 0, st, 1, "cf reduce", slots, n, slot_stride, npix, seg,
             reinterpret_cast<__nv_bfloat16 *>(out), out_pitch, epoch);
}

// (CUDA lazy loading: see preload_halo)
void preload_cfpar() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(cf_handshake_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(cf_wait_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(cf_reduce_kernel));
}

}  // namespace dc

// tf32.cu -- fp32 (DC_FP32_3XTF32) side kernels (tf32.cuh). All of them move
// or split operands; the convolution arithmetic stays in conv_v2 / wgrad_v2.
#include <cuda_bf16.h>

#include "common.hpp"
#include "launch.cuh"
#include "tf32.cuh"

namespace dc {

namespace {
__device__ __forceinline__ float hi_of(float x) { return __uint_as_float(__float_as_uint(x) & 0xffffe000u); }
}  // namespace

__global__ void import_kernel(const void *__restrict__ src, int src_bf16, void *__restrict__ dst, int n, int h,
                              int w, int C, int cp, int hb, int wb, int r0, int c0, int split) {
    pdl_wait();  // (launch.cuh: PDL)
    const long long total = (long long)n * h * w * cp;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % cp);
        const long long pix = i / cp;
        const int j = (int)(pix % w);
        const long long r = pix / w;
        const int row = (int)(r % h), s = (int)(r / h);
        const long long q = ((long long)s * hb + r0 + row) * wb + c0 + j;
        if (src_bf16) {  // bf16 plan, bf16 source: a copy into the margined layout
            const __nv_bfloat16 z = __float2bfloat16_rn(0.f);
            reinterpret_cast<__nv_bfloat16 *>(dst)[q * cp + c] =
                c < C ? reinterpret_cast<const __nv_bfloat16 *>(src)[pix * C + c] : z;
            continue;
        }
        const float v = c < C ? reinterpret_cast<const float *>(src)[pix * C + c] : 0.f;
        if (split) {
            float *d = reinterpret_cast<float *>(dst) + q * 2 * cp;
            const float hv = hi_of(v);
            d[c] = hv;
            d[cp + c] = v - hv;
        } else {
            reinterpret_cast<__nv_bfloat16 *>(dst)[q * cp + c] = __float2bfloat16_rn(v);
        }
    }
}

void launch_import(const void *src, bool src_bf16, void *dst, int n, int h, int w, int C, int cp, int hb, int wb,
                   int r0, int c0, int split, cudaStream_t st) {
    const long long total = (long long)n * h * w * cp;
    if (total == 0) return;
    const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 16);
    launch_k(import_kernel, dim3(blocks), dim3(256), 0, st, 1, "import", src, (int)src_bf16, dst, n, h, w, C, cp, hb,
             wb, r0, c0, split);
}

__global__ void weight_split_kernel(const float *__restrict__ w, float *__restrict__ ws, int F, int T, int C,
                                    int cp) {
    pdl_wait();  // (launch.cuh: PDL)
    const long long total = (long long)F * T * cp;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % cp);
        const long long ft = i / cp;
        const float v = c < C ? w[i] : 0.f;
        const float hv = hi_of(v);
        float *d = ws + ft * 3 * cp;
        d[c] = hv;
        d[cp + c] = v - hv;
        d[2 * cp + c] = hv;
    }
}

void launch_weight_split(const float *w, float *ws, int F, int T, int C, int cp, cudaStream_t st) {
    const long long total = (long long)F * T * cp;
    const int blocks = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, 148 * 8));
    launch_k(weight_split_kernel, dim3(blocks), dim3(256), 0, st, 1, "weight split", w, ws, F, T, C, cp);
}

struct TapTableF {
    int8_t a[kMaxTaps], b[kMaxTaps];
    int T[kMaxTaps], t[kMaxTaps];
    long long off[kMaxTaps];
};

// grid.y = listed tap j; threads over (c, f): f fastest, so the writes of
// wt[..][f] are coalesced (the reads of w[f][a][b][c] are strided: weights are
// small and read once per backward-data call)
__global__ void weight_transform_tf32_kernel(const float *__restrict__ w, float *__restrict__ wt_base, int F, int fp,
                                             int C, int cp, int K, const __grid_constant__ TapTableF tt) {
    pdl_wait();  // (launch.cuh: PDL)
    const int j = blockIdx.y;
    const int T = tt.T[j], t = tt.t[j];
    float *wt = wt_base + tt.off[j];
    const long long tap_off = ((long long)tt.a[j] * K + tt.b[j]) * cp;
    const long long total = (long long)cp * fp;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
         i += (long long)gridDim.x * blockDim.x) {
        const int f = (int)(i % fp), c = (int)(i / fp);
        const float v = (f < F && c < C) ? w[(long long)f * K * K * cp + tap_off + c] : 0.f;
        const float hv = hi_of(v);
        float *d = wt + ((long long)c * T + t) * 3 * fp;
        d[f] = hv;
        d[fp + f] = v - hv;
        d[2 * fp + f] = hv;
    }
}

void launch_weight_transform_tf32(const float *w, float *wt_base, int F, int fp, int C, int cp, int K, int ntaps,
                                  const int8_t *ka, const int8_t *kb, const int *T, const int *t,
                                  const long long *off, cudaStream_t st) {
    if (ntaps == 0) return;
    DC_REQUIRE(ntaps <= kMaxTaps, DC_ERR_ARG, "too many taps");
    TapTableF tt{};
    for (int j = 0; j < ntaps; ++j) {
        tt.a[j] = ka[j], tt.b[j] = kb[j], tt.T[j] = T[j], tt.t[j] = t[j], tt.off[j] = off[j];
    }
    const long long total = (long long)cp * fp;
    const int bx = (int)std::max<long long>(1, std::min<long long>((total + 255) / 256, 64));
    launch_k(weight_transform_tf32_kernel, dim3(bx, ntaps), dim3(256), 0, st, 1, "weight transform (tf32)", w,
             wt_base, F, fp, C, cp, K, tt);
}

// BN partial sums of an fp32 tensor: thread = (pixel lane, 4-channel vector),
// fp64 accumulation (the bf16 kernel's exact-x^2-in-fp32 grouping does not
// apply to fp32 values), then a fixed-order per-block reduction in shared
// memory (deterministic).
constexpr int kBnF32Threads = 256;

int bn_partial_blocks_f32(long long npix, int cpad) {
    const int vecs = cpad / 4;
    const int lanes = std::max(1, kBnF32Threads / vecs);
    const long long iters = (npix + lanes - 1) / lanes;
    return (int)std::max<long long>(1, std::min<long long>((iters + 15) / 16, 148 * 2));
}

__global__ void __launch_bounds__(kBnF32Threads) bn_partials_f32_kernel(const float4 *__restrict__ t, long long npix,
                                                                        int cpad, double *__restrict__ partials) {
    pdl_wait();  // (launch.cuh: PDL)
    extern __shared__ double sh[];
    const int vecs = cpad / 4;
    const int lanes = max(1, kBnF32Threads / vecs);
    const int v = threadIdx.x % vecs, pl = threadIdx.x / vecs;
    if (pl < lanes) {
        double s[4] = {0, 0, 0, 0}, q[4] = {0, 0, 0, 0};
        for (long long p = (long long)blockIdx.x * lanes + pl; p < npix; p += (long long)gridDim.x * lanes) {
            const float4 x = __ldg(&t[p * vecs + v]);
            const float e[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                s[k] += (double)e[k];
                q[k] += (double)e[k] * (double)e[k];
            }
        }
        double *row = sh + (long long)pl * 2 * cpad;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            row[v * 4 + k] = s[k];
            row[cpad + v * 4 + k] = q[k];
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * cpad; i += blockDim.x) {
        double acc = 0.0;
        for (int l = 0; l < lanes; ++l) acc += sh[(long long)l * 2 * cpad + i];
        partials[(long long)blockIdx.x * 2 * cpad + i] = acc;
    }
}

void launch_bn_partials_f32(const float *t, long long npix, int cpad, double *partials, cudaStream_t st) {
    DC_REQUIRE(cpad % 4 == 0 && cpad / 4 <= kBnF32Threads, DC_ERR_UNSUPPORTED,
               "fp32 BN stats: channels must be a multiple of 4 and <= 1024");
    const int vecs = cpad / 4, lanes = std::max(1, kBnF32Threads / vecs);
    const size_t smem = (size_t)lanes * 2 * cpad * sizeof(double);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(bn_partials_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        attr = true;
    }
    launch_k(bn_partials_f32_kernel, dim3(bn_partial_blocks_f32(npix, cpad)), dim3(kBnF32Threads), smem, st, 1,
             "bn partials (fp32)", reinterpret_cast<const float4 *>(t), npix, cpad, partials);
}


// Loads this file's kernels now (CUDA lazy loading would otherwise load a
// kernel at its first launch, which waits for the device: with the spinning
// halo / BN protocol kernels of a loopback group in flight, that wait never
// ends).
void preload_tf32() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(import_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(weight_split_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(weight_transform_tf32_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(bn_partials_f32_kernel));
}

}  // namespace dc

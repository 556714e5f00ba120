// subsample.cu -- the stride-2 pixel gather of 1x1 stride-2 convolutions
// (subsample.cuh). Memory-bound copy: a block per output row, 16-byte
// vectors across the row.
#include "common.hpp"
#include "launch.cuh"
#include "subsample.cuh"

namespace dc {

namespace {
__global__ void __launch_bounds__(256) subsample2_kernel(const uint4 *__restrict__ x, int hb, int wb, int vecs,
                                                         int oh, int ow, int ho, int wo, long long rows,
                                                         uint4 *__restrict__ xs) {
    pdl_wait();  // (launch.cuh: PDL)
    const int per_row = wo * vecs;
    for (long long r = blockIdx.x; r < rows; r += gridDim.x) {  // r = s ho + i
        const long long s = r / ho;
        const int i = (int)(r - s * ho);
        const uint4 *src = x + ((s * hb + oh + 2 * i) * wb + ow) * vecs;
        uint4 *dst = xs + r * per_row;
        for (int k = threadIdx.x; k < per_row; k += blockDim.x) {
            const int j = k / vecs, v = k - j * vecs;
            dst[k] = src[2 * j * vecs + v];
        }
    }
}
__global__ void __launch_bounds__(256) scatter2_kernel(const uint4 *__restrict__ xs, int vecs, int ho, int wo,
                                                       int oh, int ow, int h, int w, long long rows,
                                                       uint4 *__restrict__ dx) {
    pdl_wait();  // (launch.cuh: PDL)
    const int per_row = w * vecs;
    for (long long r = blockIdx.x; r < rows; r += gridDim.x) {  // r = s h + i
        const long long s = r / h;
        const int ii = (int)(r - s * h) - oh;
        const bool row_ok = ii >= 0 && (ii & 1) == 0 && (ii >> 1) < ho;
        const uint4 *src = xs + (s * ho + (ii >> 1)) * wo * vecs;
        uint4 *dst = dx + r * per_row;
        for (int k = threadIdx.x; k < per_row; k += blockDim.x) {
            const int j = k / vecs, v = k - j * vecs, jj = j - ow;
            uint4 val = make_uint4(0, 0, 0, 0);
            if (row_ok && jj >= 0 && (jj & 1) == 0 && (jj >> 1) < wo) val = src[(jj >> 1) * vecs + v];
            dst[k] = val;
        }
    }
}
}  // namespace

void launch_scatter2(const void *xs, int64_t n, int64_t ho, int64_t wo, int pix_bytes, int oh, int ow, int64_t h,
                     int64_t w, void *dx, cudaStream_t st) {
    DC_REQUIRE(pix_bytes % 16 == 0 && reinterpret_cast<uintptr_t>(xs) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(dx) % 16 == 0,
               DC_ERR_ARG, "scatter2: 16-byte pixels and buffers");
    const long long rows = n * h;
    if (rows == 0 || w == 0) return;
    const int blocks = (int)std::min<long long>(rows, 148 * 16);
    launch_k(scatter2_kernel, dim3(blocks), dim3(256), 0, st, 1, "scatter2", reinterpret_cast<const uint4 *>(xs),
             pix_bytes / 16, (int)ho, (int)wo, oh, ow, (int)h, (int)w, rows, reinterpret_cast<uint4 *>(dx));
}

void launch_subsample2(const void *x, int64_t n, int64_t hb, int64_t wb, int pix_bytes, int oh, int ow,
                       int64_t ho, int64_t wo, void *xs, cudaStream_t st) {
    DC_REQUIRE(pix_bytes % 16 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(xs) % 16 == 0,
               DC_ERR_ARG, "subsample: 16-byte pixels and buffers");
    DC_REQUIRE(oh >= 0 && ow >= 0 && oh + 2 * (ho - 1) < hb && ow + 2 * (wo - 1) < wb, DC_ERR_ARG,
               "subsample: window outside the input buffer");
    const long long rows = n * ho;
    if (rows == 0 || wo == 0) return;
    const int blocks = (int)std::min<long long>(rows, 148 * 16);
    launch_k(subsample2_kernel, dim3(blocks), dim3(256), 0, st, 1, "subsample2", reinterpret_cast<const uint4 *>(x),
             (int)hb, (int)wb, pix_bytes / 16, oh, ow, (int)ho, (int)wo, rows, reinterpret_cast<uint4 *>(xs));
}

// (CUDA lazy loading: see preload_halo)
void preload_subsample() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(subsample2_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(scatter2_kernel));
}

}  // namespace dc

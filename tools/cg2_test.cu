// cg2_test.cu -- standalone check of the 2-SM MMA conventions (tcgen05
// cta_group::2) before using them in conv_v2: a CTA pair computes
// D[256 x N] = A[256 x 64] * B[N x 64]^T with CTA r holding A rows 128r..128r+127
// and B rows (N) N/2*r .. at the same smem offsets (K-major, 128B swizzle);
// the leader issues M = 256 MMAs; each CTA reads its 128 rows of D from TMEM.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -I../paper_1903_06681_b200/csrc cg2_test.cu -o cg2_test
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_bf16.h>
#include "sm100.cuh"
using namespace dc::sm100;

constexpr int N = 64, K = 64;

__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t chunk16) {  // byte offset in a K-major SW128 tile
    return row * 128 + ((chunk16 ^ (row & 7)) << 4);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    cg2_kernel(const __nv_bfloat16 *A, const __nv_bfloat16 *B, float *D) {
    __shared__ __align__(1024) uint8_t sA[128 * 128];
    __shared__ __align__(1024) uint8_t sB[(N / 2) * 128];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const uint32_t cr = cluster_ctarank();
    const int tid = threadIdx.x, warp = tid >> 5;
    // fill: A rows 128*cr.., B rows (N/2)*cr..
    for (int i = tid; i < 128 * 8; i += blockDim.x) {
        const int r = i / 8, c = i % 8;
        const uint4 v = reinterpret_cast<const uint4 *>(A + (size_t)(128 * cr + r) * K)[c];
        *reinterpret_cast<uint4 *>(sA + sw128(r, c)) = v;
    }
    for (int i = tid; i < (N / 2) * 8; i += blockDim.x) {
        const int r = i / 8, c = i % 8;
        const uint4 v = reinterpret_cast<const uint4 *>(B + (size_t)((N / 2) * cr + r) * K)[c];
        *reinterpret_cast<uint4 *>(sB + sw128(r, c)) = v;
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                     "r"(64u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (cr == 0 && warp == 0) {
        if (elect_one()) {
            const uint64_t ad = smem_desc(smem_u32(sA), 16, 1024, 2);
            const uint64_t bd = smem_desc(smem_u32(sB), 16, 1024, 2);
            const uint32_t idesc = idesc_bf16(256, N, 0, 0);
            for (int k = 0; k < K / 16; ++k)
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                    "l"(ad + 2 * k), "l"(bd + 2 * k), "r"(idesc), "r"(k));
            asm volatile(
                "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                    smem_u32(&bar)),
                "h"((uint16_t)3)
                : "memory");
        }
        __syncwarp();
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    // each warp reads its 32 lanes (rows) x N columns
    for (int c16 = 0; c16 < N / 16; ++c16) {
        uint32_t v[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + c16 * 16, v);
        tmem_ld_wait();
        const int row = 128 * cr + warp * 32 + (tid & 31);
        for (int e = 0; e < 16; ++e) D[(size_t)row * N + c16 * 16 + e] = __uint_as_float(v[e]);
    }
    tc_fence_before();
    cluster_sync();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64u));
}

int main() {
    std::vector<__nv_bfloat16> hA(256 * K), hB(N * K);
    std::vector<float> fA(256 * K), fB(N * K);
    srand(7);
    for (int i = 0; i < 256 * K; ++i) fA[i] = (float)((rand() % 17) - 8) / 8.f, hA[i] = __float2bfloat16(fA[i]);
    for (int i = 0; i < N * K; ++i) fB[i] = (float)((rand() % 13) - 6) / 8.f, hB[i] = __float2bfloat16(fB[i]);
    __nv_bfloat16 *dA, *dB;
    float *dD;
    cudaMalloc(&dA, hA.size() * 2);
    cudaMalloc(&dB, hB.size() * 2);
    cudaMalloc(&dD, 256 * N * 4);
    cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0xff, 256 * N * 4);
    cg2_kernel<<<2, 128>>>(dA, dB, dD);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> hD(256 * N);
    cudaMemcpy(hD.data(), dD, hD.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < 256; ++m)
        for (int n = 0; n < N; ++n) {
            double r = 0;
            for (int k = 0; k < K; ++k) r += (double)fA[m * K + k] * fB[n * K + k];
            maxerr = std::max(maxerr, std::fabs(r - hD[m * N + n]));
        }
    printf("cg2 M=256 N=%d K=%d: max abs err %.3g (%s)\n", N, K, maxerr, maxerr < 1e-3 ? "OK" : "FAIL");
    return maxerr < 1e-3 ? 0 : 2;
}

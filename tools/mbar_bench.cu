// Microbenchmark of the sm_100a synchronisation primitives the conv kernels
// rely on (cycles via clock64): mbarrier ping-pong between two warps (with
// and without a try_wait suspend-time hint), tcgen05.commit -> mbarrier
// latency, and tcgen05.mma latency / throughput for M=128, N=64/256, K=16.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1903_06681_b200/csrc tools/mbar_bench.cu -o /tmp/mbar_bench
#include <cstdio>
#include <cstdint>
#include "sm100.cuh"

using namespace dc::sm100;

__device__ __forceinline__ void wait_hint(uint64_t *bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "W_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra W_%=;\n}" ::"r"(a), "r"(parity), "r"(0x989680)
        : "memory");
}
__device__ __forceinline__ void wait_test(uint64_t *bar, uint32_t parity) {
    const uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "W_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra W_%=;\n}" ::"r"(a), "r"(parity)
        : "memory");
}

__global__ void bench(long long *out, int mode) {
    __shared__ __align__(1024) uint8_t sm[40960];
    __shared__ uint64_t bar[4];
    __shared__ uint32_t tslot;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < 40960 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0;
    if (warp == 1) tmem_alloc(&tslot, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    const int N = 1000;
    if (mode <= 2) {  // ping-pong
        if (lane == 0 && warp < 2) {
            long long t0 = clock64();
            for (int i = 0; i < N; ++i) {
                if (warp == 0) {
                    mbar_arrive(&bar[0]);
                    if (mode == 0) mbar_wait(&bar[1], i & 1);
                    else if (mode == 1) wait_hint(&bar[1], i & 1);
                    else wait_test(&bar[1], i & 1);
                } else {
                    if (mode == 0) mbar_wait(&bar[0], i & 1);
                    else if (mode == 1) wait_hint(&bar[0], i & 1);
                    else wait_test(&bar[0], i & 1);
                    mbar_arrive(&bar[1]);
                }
            }
            if (warp == 0) out[mode] = (clock64() - t0) / N;
        }
    } else if (warp == 1 && lane == 0) {
        const uint32_t sa = smem_u32(sm);
        const uint64_t ad = smem_desc(sa, 16, 1024, 2), bd = smem_desc(sa + 8192, 16, 1024, 2);  // 256 rows x 128 B fit in the 40 KB buffer
        const int n = mode == 5 ? 256 : 64;
        const uint32_t idesc = idesc_bf16(128, n, 0, 0);
        long long t0 = clock64();
        if (mode == 3) {  // commit with nothing pending -> wait
            for (int i = 0; i < N; ++i) {
                mma_commit(&bar[2]);
                mbar_wait(&bar[2], i & 1);
            }
            out[3] = (clock64() - t0) / N;
        } else {  // one MMA + commit + wait (latency), then 64 MMAs + commit (throughput)
            for (int i = 0; i < 200; ++i) {
                mma_bf16(tmem, ad, bd, idesc, i > 0);
                mma_commit(&bar[2]);
                mbar_wait(&bar[2], i & 1);
            }
            const long long lat = (clock64() - t0) / 200;
            t0 = clock64();
            for (int r = 0; r < 20; ++r) {
                for (int i = 0; i < 64; ++i) mma_bf16(tmem, ad + (i & 3) * 2, bd + (i & 3) * 2, idesc, 1);
                mma_commit(&bar[3]);
                mbar_wait(&bar[3], r & 1);
            }
            const long long thr = (clock64() - t0) / (20 * 64);
            out[mode == 4 ? 4 : 6] = lat;
            out[mode == 4 ? 5 : 7] = thr;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, 512);
}

int main() {
    long long *d, h[8] = {0};
    cudaMalloc(&d, sizeof h);
    cudaMemset(d, 0, sizeof h);
    for (int m = 0; m <= 5; ++m) {
        bench<<<1, 128>>>(d, m);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("mode %d: %s\n", m, cudaGetErrorString(e)); return 1; }
    }
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("mbarrier ping-pong round trip (cycles): try_wait %lld | try_wait+hint %lld | test_wait %lld\n", h[0], h[1], h[2]);
    printf("tcgen05.commit (nothing pending) -> wait: %lld cycles\n", h[3]);
    printf("MMA 128x64x16: latency (mma+commit+wait) %lld, throughput %lld cycles/MMA\n", h[4], h[5]);
    printf("MMA 128x256x16: latency %lld, throughput %lld cycles/MMA\n", h[6], h[7]);
    return 0;
}

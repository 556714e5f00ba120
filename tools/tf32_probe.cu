// tf32_probe.cu -- one tcgen05.mma.kind::tf32 (M=128, N=64, K=8) with the
// operands in K-major or MN-major 128B-swizzled shared memory, checked
// against a host fp64 product of the tf32-truncated / -rounded inputs.
// Pins the instruction-descriptor encoding (a/b format 2 = TF32) and the
// MN-major operand layout the 3xTF32 backward-filter kernel relies on.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o tools/tf32_probe tools/tf32_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_1903_06681_b200/csrc/sm100.cuh"

using namespace dc::sm100;

constexpr int M = 128, N = 64, K = 8;

__host__ __device__ inline uint32_t kmaj_off(int r, int k) {  // row r of a K-major SW128 tile
    const uint32_t b = (uint32_t)k * 4;
    return (r / 8) * 1024 + (r % 8) * 128 + ((((b >> 4) ^ (r % 8)) & 7) << 4) + (b & 15);
}
__host__ __device__ inline uint32_t mnmaj_off(int r, int k) {  // MN-major SW128: atoms of 32 rows
    const uint32_t b = (uint32_t)(r % 32) * 4;
    return (r / 32) * 1024 + k * 128 + ((((b >> 4) ^ (k % 8)) & 7) << 4) + (b & 15);
}

// MN-major, 128B rows with a 32-byte-granule swizzle (cute Swizzle<2,5,2>,
// descriptor layout type 1 = SWIZZLE_128B_BASE32B): atom = 4 K rows x 32 fp32;
// atoms along M at LBO = 512, 4-row K groups at SBO = 2048
__host__ __device__ inline uint32_t mn32_off(int r, int k) {
    const uint32_t b = (uint32_t)(r % 32) * 4, row = k % 4;
    return (r / 32) * 512 + (k / 4) * 2048 + row * 128 + ((((b >> 5) ^ row) & 3) << 5) + (b & 31);
}

__global__ void probe(const float *A, const float *B, float *D, int mode) {
    const int mn = mode > 0 ? 1 : 0;
    __shared__ __align__(1024) uint8_t sA[16384];
    __shared__ __align__(1024) uint8_t sB[8192];
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int t = threadIdx.x;
    for (int i = t; i < M * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        *reinterpret_cast<float *>(sA + (mode == 2 ? mn32_off(r, k) : mn ? mnmaj_off(r, k) : kmaj_off(r, k))) = A[i];
    }
    for (int i = t; i < N * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        *reinterpret_cast<float *>(sB + (mode == 2 ? mn32_off(r, k) : mn ? mnmaj_off(r, k) : kmaj_off(r, k))) = B[i];
    }
    if (t == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if ((t >> 5) == 0) tmem_alloc(&tslot, 64);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (t == 0) {
        // idesc: D f32 (bit 4), a/b format TF32 = 2 (bits 7-9, 10-12), majors bits 15/16
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)mn << 15) | ((uint32_t)mn << 16) |
                               ((N >> 3) << 17) | ((M >> 4) << 24);
        uint64_t ad, bd;
        if (mode == 2) {
            ad = smem_desc(smem_u32(sA), 512, 2048, 1);
            bd = smem_desc(smem_u32(sB), 512, 2048, 1);
        } else if (mn) {
            ad = smem_desc(smem_u32(sA), 1024, 4096, 2);  // LBO = next 32-row atom, SBO = next 8 K rows
            bd = smem_desc(smem_u32(sB), 1024, 4096, 2);
        } else {
            ad = smem_desc(smem_u32(sA), 16, 1024, 2);
            bd = smem_desc(smem_u32(sB), 16, 1024, 2);
        }
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(0u));
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    const int w = t >> 5, lane = t & 31;
    for (int c = 0; c < N / 16; ++c) {
        uint32_t v[16];
        tmem_ld16(tmem + ((uint32_t)(w * 32) << 16) + c * 16, v);
        tmem_ld_wait();
        for (int e = 0; e < 16; ++e) D[(w * 32 + lane) * N + c * 16 + e] = __uint_as_float(v[e]);
    }
    tc_fence_before();
    __syncthreads();
    if (w == 0) tmem_dealloc(tmem, 64);
}

static float trunc_tf32(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u &= 0xffffe000u;
    memcpy(&x, &u, 4);
    return x;
}
static float round_tf32(float x) {
    uint32_t u;
    memcpy(&u, &x, 4);
    u += 0x1000u;
    u &= 0xffffe000u;
    memcpy(&x, &u, 4);
    return x;
}

int main() {
    std::vector<float> A(M * K), B(N * K), D(M * N);
    srand(7);
    for (auto &v : A) v = (float)((rand() / (double)RAND_MAX) * 2 - 1);
    for (auto &v : B) v = (float)((rand() / (double)RAND_MAX) * 2 - 1);
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    int fails = 0;
    const char *names[3] = {"K-major SW128", "MN-major SW128", "MN-major SW128_BASE32B"};
    for (int mode = 0; mode < 3; ++mode) {
        const int mn = mode;
        cudaMemset(dD, 0, D.size() * 4);
        probe<<<1, 128>>>(dA, dB, dD, mode);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("%s: CUDA error %s\n", names[mn], cudaGetErrorString(e));
            return 2;
        }
        cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
        double et = 0, er = 0, ex = 0, mx = 0;
        for (int m = 0; m < M; ++m)
            for (int n = 0; n < N; ++n) {
                double st = 0, sr = 0, sx = 0;
                for (int k = 0; k < K; ++k) {
                    st += (double)trunc_tf32(A[m * K + k]) * trunc_tf32(B[n * K + k]);
                    sr += (double)round_tf32(A[m * K + k]) * round_tf32(B[n * K + k]);
                    sx += (double)A[m * K + k] * B[n * K + k];
                }
                const double g = D[m * N + n];
                et = fmax(et, fabs(g - st));
                er = fmax(er, fabs(g - sr));
                ex = fmax(ex, fabs(g - sx));
                mx = fmax(mx, fabs(sx));
            }
        printf("%s: max|D - trunc| = %.3e  max|D - round| = %.3e  max|D - exact| = %.3e  (max|D| %.3f)\n",
               names[mn], et, er, ex, mx);
        if (fmin(et, er) > 1e-5 && mode != 1) ++fails;
    }
    printf(fails ? "TF32 PROBE FAILED\n" : "TF32 PROBE OK\n");
    return fails ? 1 : 0;
}

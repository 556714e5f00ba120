// tma32_probe.cu -- which TMA swizzle mode writes the MN-major tf32 operand
// layout tcgen05 expects (descriptor layout type 1, SWIZZLE_128B_BASE32B =
// cute Swizzle<2,5,2>: byte bits [5,7) ^= bits [7,9))? Loads a [8 k][128 m]
// fp32 tile (m contiguous) with box {32 m, 8 k} under each 128B swizzle mode,
// dumps shared memory, then runs one kind::tf32 MMA (M=128, N=64, K=8) with
// A and B both MN-major from the TMA-written tiles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -o tools/tma32_probe tools/tma32_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cmath>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>
#include "../paper_1903_06681_b200/csrc/sm100.cuh"

using namespace dc::sm100;
constexpr int M = 128, N = 64, K = 8;

__global__ void probe(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                      float *D, uint8_t *dump, int layout) {
    __shared__ __align__(1024) uint8_t sA[4096];
    __shared__ __align__(1024) uint8_t sB[2048];
    __shared__ uint64_t bar, mbar;
    __shared__ uint32_t tslot;
    const int t = threadIdx.x;
    if (t == 0) {
        mbar_init(&bar, 1);
        mbar_init(&mbar, 1);
        fence_mbar_init();
    }
    if ((t >> 5) == 0) tmem_alloc(&tslot, 64);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tslot;
    if (t == 0) {
        mbar_arrive_expect_tx(&bar, 4096 + 2048);
        for (int a = 0; a < 4; ++a) tma_load_2d(sA + a * 1024, &amap, &bar, a * 32, 0);
        for (int a = 0; a < 2; ++a) tma_load_2d(sB + a * 1024, &bmap, &bar, a * 32, 0);
    }
    mbar_wait(&bar, 0);
    for (int i = t; i < 4096; i += blockDim.x) dump[i] = sA[i];
    if (t == 0 && layout >= 0) {
        const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (1u << 16) | ((N >> 3) << 17) |
                               ((M >> 4) << 24);
        // A: M atoms (32 fp32) 1024 B apart (one box each), 4-row K groups 512 B apart
        const uint64_t ad = smem_desc(smem_u32(sA), 1024, 512, (uint32_t)layout);
        const uint64_t bd = smem_desc(smem_u32(sB), 1024, 512, (uint32_t)layout);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(idesc), "r"(0u));
        mma_commit(&mbar);
    }
    if (layout >= 0) {
        mbar_wait(&mbar, 0);
        tc_fence_after();
        const int w = t >> 5, lane = t & 31;
        for (int c = 0; c < N / 16; ++c) {
            uint32_t v[16];
            tmem_ld16(tmem + ((uint32_t)(w * 32) << 16) + c * 16, v);
            tmem_ld_wait();
            for (int e = 0; e < 16; ++e) D[(w * 32 + lane) * N + c * 16 + e] = __uint_as_float(v[e]);
        }
    }
    tc_fence_before();
    __syncthreads();
    if ((t >> 5) == 0) tmem_dealloc(tmem, 64);
}

typedef CUresult (*EncodeFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                             const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    EncodeFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    std::vector<float> A(K * M), B(K * N), D(M * N);
    for (int i = 0; i < K * M; ++i) A[i] = (float)((i * 7919) % 1000) / 500.f - 1.f;
    for (int i = 0; i < K * N; ++i) B[i] = (float)((i * 104729) % 1000) / 500.f - 1.f;
    float *dA, *dB, *dD;
    uint8_t *dDump;
    cudaMalloc(&dA, A.size() * 4);
    cudaMalloc(&dB, B.size() * 4);
    cudaMalloc(&dD, D.size() * 4);
    cudaMalloc(&dDump, 4096);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    const CUtensorMapSwizzle modes[4] = {CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                                         CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B_FLIP_8B,
                                         CU_TENSOR_MAP_SWIZZLE_128B_ATOM_64B};
    const char *names[4] = {"128B", "128B_ATOM_32B", "128B_ATOM_32B_FLIP_8B", "128B_ATOM_64B"};
    for (int mi = 0; mi < 4; ++mi) {
        CUtensorMap am, bm;
        cuuint64_t dimsA[2] = {M, K}, strA[1] = {M * 4}, dimsB[2] = {N, K}, strB[1] = {N * 4};
        cuuint32_t box[2] = {32, 8}, es[2] = {1, 1};
        CUresult r1 = enc(&am, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, dimsA, strA, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          modes[mi], CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        CUresult r2 = enc(&bm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, dimsB, strB, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          modes[mi], CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r1 != CUDA_SUCCESS || r2 != CUDA_SUCCESS) {
            printf("%s: encode failed %d %d\n", names[mi], (int)r1, (int)r2);
            continue;
        }
        // (a) the layout TMA wrote: does element (k, m) of box 0 sit at the
        // Swizzle<2,5,2> position k*128 + (((m*4 >> 5) ^ (k & 3)) << 5) + (m*4 & 31)?
        probe<<<1, 128>>>(am, bm, dD, dDump, -1);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("%s: CUDA error %s\n", names[mi], cudaGetErrorString(e));
            return 2;
        }
        std::vector<uint8_t> dump(4096);
        cudaMemcpy(dump.data(), dDump, 4096, cudaMemcpyDeviceToHost);
        int bad252 = 0, bad253 = 0;
        for (int k = 0; k < K; ++k)
            for (int m = 0; m < 32; ++m) {
                float v;
                const uint32_t b = m * 4;
                const uint32_t o252 = k * 128 + ((((b >> 5) ^ (k & 3)) & 3) << 5) + (b & 31);
                const uint32_t o253 = k * 128 + ((((b >> 5) ^ ((k >> 1) & 3)) & 3) << 5) + (b & 31);
                memcpy(&v, dump.data() + o252, 4);
                bad252 += v != A[k * M + m];
                memcpy(&v, dump.data() + o253, 4);
                bad253 += v != A[k * M + m];
            }
        printf("%s: mismatches vs Swizzle<2,5,2> (bits 5-6 ^= 7-8): %d, vs bits 5-6 ^= 8-9: %d of 256\n", names[mi],
               bad252, bad253);
        // (b) one MMA with both operands as TMA wrote them, descriptor layout 1 (BASE32B) and 2 (SW128)
        for (int layout : {1, 2}) {
            cudaMemset(dD, 0, D.size() * 4);
            probe<<<1, 128>>>(am, bm, dD, dDump, layout);
            e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("  layout %d: CUDA error %s\n", layout, cudaGetErrorString(e));
                return 2;
            }
            cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
            double err = 0;
            for (int m = 0; m < M; ++m)
                for (int n = 0; n < N; ++n) {
                    double s = 0;
                    for (int k = 0; k < K; ++k) {
                        uint32_t ua, ub;
                        float a = A[k * M + m], bb = B[k * N + n];
                        memcpy(&ua, &a, 4), memcpy(&ub, &bb, 4);
                        ua &= 0xffffe000u, ub &= 0xffffe000u;
                        memcpy(&a, &ua, 4), memcpy(&bb, &ub, 4);
                        s += (double)a * bb;
                    }
                    err = fmax(err, fabs(s - D[m * N + n]));
                }
            printf("  MMA MN-major, descriptor layout %d: max|D - ref| = %.3e\n", layout, err);
        }
    }
    return 0;
}

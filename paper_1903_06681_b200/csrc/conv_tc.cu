// conv_tc.cu -- sm_100a implicit-GEMM convolution kernels (tcgen05 + TMEM + TMA).
//
// Forward (Eq. 1) and backward-data (Eq. 3) run on
// one kernel, conv_gemm_kernel: GEMM M = 128 output pixels (a TH x TW spatial
// tile of one sample), N = output channels, K = taps x input channels. The A
// operand of tap t is a TMA box of the NHWC input buffer at the tap-shifted
// coordinates (element stride = conv stride); out-of-buffer coordinates are
// zero-filled by TMA, which realises the zero padding without a second code
// path. The B operand is a [N][taps*cin] weight matrix (K-major). One
// elected thread issues tcgen05.mma into a TMEM accumulator; a 4-warp
// epilogue reads TMEM (tcgen05.ld) and stores bf16 NHWC.
//
// Backward-filter (Eq. 2) runs on wgrad_kernel: GEMM
// M = 128 (tap, input channel) pairs, N = filters, K = output pixels of the
// owned block (dy without halo); both operands MN-major; the
// K range is split across CTAs and reduced in a fixed order (deterministic).
#include <cstdio>
#include <mutex>

#include "common.hpp"
#include "conv_tc.cuh"
#include "launch.cuh"
#include "sm100.cuh"

namespace dc {
using namespace sm100;

static __device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
    const uint32_t a = smem_u32(p);
    return p + ((1024 - (a & 1023)) & 1023);
}

static __device__ __forceinline__ uint32_t pack_bf16x2(uint32_t lo, uint32_t hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
    return *reinterpret_cast<uint32_t *>(&v);
}

static __host__ __device__ inline uint32_t tmem_cols_for(int bn) {
    uint32_t c = 32;
    while ((int)c < bn) c <<= 1;
    return c;
}

// ============================================================================
// Forward / backward-data implicit GEMM
// ============================================================================
__global__ void __launch_bounds__(128, 1)
    conv_gemm_kernel(const __grid_constant__ CUtensorMap amap,
                     const __grid_constant__ CUtensorMap bmap,
                     const __grid_constant__ ConvGemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    const int A_BYTES = 128 * p.bkc * 2;
    const int B_BYTES = p.bn * p.bkc * 2;
    uint8_t *sA = smem;
    uint8_t *sB = smem + p.stages * A_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(sB + p.stages * B_BYTES);
    uint64_t *empty = full + p.stages;
    uint64_t *done = empty + p.stages;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;

    // ---- which output tile ----
    const int tile = blockIdx.x;
    int r = 0;
    while (r + 1 < p.nrect && tile >= p.rect_start[r + 1]) ++r;
    const int lt = tile - p.rect_start[r];
    const int twl = p.rect_twl[r];
    const int TW = 1 << twl, TH = 128 >> twl;
    const int i0 = p.rect[r].h0 + (lt / p.rect_tiles_w[r]) * TH;
    const int j0 = p.rect[r].w0 + (lt % p.rect_tiles_w[r]) * TW;
    const int n = blockIdx.y;
    const int o0 = blockIdx.z * p.bn;
    const int KB = p.T * p.kc;
    const uint32_t ncols = tmem_cols_for(p.bn);

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(tmem_slot, ncols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ===== TMA producer =====
        tma_prefetch(&amap);
        tma_prefetch(&bmap);
        const int ah0 = p.s_in * i0 + p.origin_h, aw0 = p.s_in * j0 + p.origin_w;
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % p.stages, round = kb / p.stages;
            if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
            const int t = kb / p.kc, cc = kb - t * p.kc;
            mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
            tma_load_4d(sA + s * A_BYTES, &amap, &full[s], cc * p.bkc, aw0 + p.tap_w[t],
                        ah0 + p.tap_h[t], n);
            tma_load_2d(sB + s * B_BYTES, &bmap, &full[s], (t * p.kc + cc) * p.bkc, o0);
        }
    } else if (warp == 1 && lane == 0) {
        // ===== MMA issuer (single thread) =====
        const uint32_t idesc = idesc_bf16(128, p.bn, 0, 0);
        const uint32_t layout = swizzle_layout(p.bkc * 2);
        const uint32_t sbo = 8 * p.bkc * 2;
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % p.stages, round = kb / p.stages;
            mbar_wait(&full[s], round & 1);
            tc_fence_after();
            const uint32_t a_base = smem_u32(sA + s * A_BYTES);
            const uint32_t b_base = smem_u32(sB + s * B_BYTES);
            for (int k = 0; k < p.bkc / 16; ++k) {
                const uint64_t ad = smem_desc(a_base + k * 32, 16, sbo, layout);
                const uint64_t bd = smem_desc(b_base + k * 32, 16, sbo, layout);
                mma_bf16(tmem, ad, bd, idesc, (kb | k) != 0);
            }
            mma_commit(&empty[s]);
        }
        mma_commit(done);
    }
    __syncwarp();

    // ===== epilogue: TMEM -> registers -> bf16 NHWC =====
    mbar_wait(done, 0);
    tc_fence_after();
    const int m = warp * 32 + lane;
    const int i = i0 + (m >> twl), j = j0 + (m & (TW - 1));
    const bool valid = i < p.rect[r].h0 + p.rect[r].nh && j < p.rect[r].w0 + p.rect[r].nw;
    __nv_bfloat16 *orow = p.out + (long long)n * p.out_sn +
                          (long long)(p.out_h0 + p.out_dh * i) * p.out_sh +
                          (long long)(p.out_w0 + p.out_dw * j) * p.out_sw + o0;
    const uint32_t t_lane = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c16 = 0; c16 < p.bn / 16; ++c16) {
        uint32_t v[16];
        if (KB > 0) {
            tmem_ld16(t_lane + c16 * 16, v);
            tmem_ld_wait();
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = 0;
        }
        if (valid && o0 + c16 * 16 < p.nout_p) {
            uint4 lo, hi;
            lo.x = pack_bf16x2(v[0], v[1]);
            lo.y = pack_bf16x2(v[2], v[3]);
            lo.z = pack_bf16x2(v[4], v[5]);
            lo.w = pack_bf16x2(v[6], v[7]);
            hi.x = pack_bf16x2(v[8], v[9]);
            hi.y = pack_bf16x2(v[10], v[11]);
            hi.z = pack_bf16x2(v[12], v[13]);
            hi.w = pack_bf16x2(v[14], v[15]);
            uint4 *dst = reinterpret_cast<uint4 *>(orow + c16 * 16);
            dst[0] = lo;
            dst[1] = hi;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, ncols);
}

// ============================================================================
// Backward-filter implicit GEMM (split-K over output pixels)
// ============================================================================
__global__ void __launch_bounds__(128, 1)
    wgrad_kernel(const __grid_constant__ CUtensorMap xmap,
                 const __grid_constant__ CUtensorMap dymap,
                 const __grid_constant__ WgradParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    const int PPM = 128 / p.bkc;             // (tap, chunk) pairs per M tile
    const int A_BOX = 64 * p.bkc * 2;        // one x box: 64 pixels x bkc channels
    const int A_BYTES = 128 * 64 * 2;        // PPM boxes
    const int B_BOX = 64 * p.bf * 2;
    const int B_BYTES = p.bn * 64 * 2;
    uint8_t *sA = smem;
    uint8_t *sB = smem + p.stages * A_BYTES;
    uint64_t *full = reinterpret_cast<uint64_t *>(sB + p.stages * B_BYTES);
    uint64_t *empty = full + p.stages;
    uint64_t *done = empty + p.stages;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const int mt = blockIdx.x, f0 = blockIdx.y * p.bn, split = blockIdx.z;
    const int b_begin = (int)((long long)split * p.nblocks / p.splits);
    const int b_end = (int)((long long)(split + 1) * p.nblocks / p.splits);
    const int KB = b_end - b_begin;
    const int TW = 1 << p.tw_log2, TH = 64 >> p.tw_log2;
    const uint32_t ncols = tmem_cols_for(p.bn);

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc(tmem_slot, ncols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        tma_prefetch(&xmap);
        tma_prefetch(&dymap);
        const int per_n = p.tiles_h * p.tiles_w;
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % p.stages, round = kb / p.stages;
            if (round > 0) mbar_wait(&empty[s], (round - 1) & 1);
            const int blk = b_begin + kb;
            const int n = blk / per_n, rem = blk - n * per_n;
            const int i0 = (rem / p.tiles_w) * TH, j0 = (rem % p.tiles_w) * TW;
            mbar_arrive_expect_tx(&full[s], A_BYTES + B_BYTES);
            for (int q = 0; q < PPM; ++q) {
                int pair = mt * PPM + q;
                if (pair >= p.pairs_total) pair = p.pairs_total - 1;  // rows discarded below
                const int t = pair / p.kc, cc = pair - t * p.kc;
                tma_load_4d(sA + s * A_BYTES + q * A_BOX, &xmap, &full[s], cc * p.bkc,
                            p.s_in * j0 + p.origin_w + p.tap_w[t],
                            p.s_in * i0 + p.origin_h + p.tap_h[t], n);
            }
            for (int q = 0; q < p.bn / p.bf; ++q)
                tma_load_4d(sB + s * B_BYTES + q * B_BOX, &dymap, &full[s], f0 + q * p.bf, j0, i0,
                            n);
        }
    } else if (warp == 1 && lane == 0) {
        const uint32_t idesc = idesc_bf16(128, p.bn, 1, 1);
        const uint32_t la = swizzle_layout(p.bkc * 2), lb = swizzle_layout(p.bf * 2);
        const uint32_t a_sbo = 8 * p.bkc * 2, b_sbo = 8 * p.bf * 2;
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % p.stages, round = kb / p.stages;
            mbar_wait(&full[s], round & 1);
            tc_fence_after();
            const uint32_t a_base = smem_u32(sA + s * A_BYTES);
            const uint32_t b_base = smem_u32(sB + s * B_BYTES);
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // 64 pixels = 4 x UMMA_K(16)
                const uint64_t ad = smem_desc(a_base + k * 2 * a_sbo, A_BOX, a_sbo, la);
                const uint64_t bd = smem_desc(b_base + k * 2 * b_sbo, B_BOX, b_sbo, lb);
                mma_bf16(tmem, ad, bd, idesc, (kb | k) != 0);
            }
            mma_commit(&empty[s]);
        }
        mma_commit(done);
    }
    __syncwarp();

    mbar_wait(done, 0);
    tc_fence_after();
    const int m = warp * 32 + lane;
    const int pair = mt * PPM + m / p.bkc;
    const int t = pair / p.kc, c = (pair - t * p.kc) * p.bkc + (m % p.bkc);
    const bool valid = pair < p.pairs_total && c < p.C;  // (dW holds the C logical channels)
    float *wrow = p.ws + (long long)split * p.ws_split + (long long)t * p.C + c;
    const long long fstride = (long long)p.T * p.C;
    const uint32_t t_lane = tmem + ((uint32_t)(warp * 32) << 16);
    for (int c16 = 0; c16 < p.bn / 16; ++c16) {
        uint32_t v[16];
        if (KB > 0) {
            tmem_ld16(t_lane + c16 * 16, v);
            tmem_ld_wait();
        } else {
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = 0;
        }
        if (valid) {
#pragma unroll
            for (int e = 0; e < 16; ++e) {
                const int f = f0 + c16 * 16 + e;
                if (f < p.F) wrow[f * fstride] = __uint_as_float(v[e]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, ncols);
}

// Deterministic split-K reduction: dw[i] = sum_{s in order} ws[s][i]
// (16-byte vectors; scalar when n is not a multiple of 4).
__global__ void splitk_reduce_kernel(const float *__restrict__ ws, int splits, long long n, long long split_stride,
                                     float *__restrict__ dw) {
    pdl_wait();  // (launch.cuh: PDL)
    const bool vec = (n % 4) == 0 && (reinterpret_cast<uintptr_t>(dw) & 15) == 0;
    const long long nv = vec ? n / 4 : n;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nv;
         i += (long long)gridDim.x * blockDim.x) {
        if (vec) {
            const float4 *w4 = reinterpret_cast<const float4 *>(ws);
            float4 acc = w4[i];
            for (int s = 1; s < splits; ++s) {
                const float4 v = w4[s * (split_stride / 4) + i];
                acc.x += v.x;
                acc.y += v.y;
                acc.z += v.z;
                acc.w += v.w;
            }
            reinterpret_cast<float4 *>(dw)[i] = acc;
        } else {
            float acc = ws[i];
            for (int s = 1; s < splits; ++s) acc += ws[s * split_stride + i];
            dw[i] = acc;
        }
    }
}

struct TapTable {  // grid.z = tap j (of any stride phase)
    int8_t a[kMaxTaps], b[kMaxTaps];  // source tap of w
    uint8_t T[kMaxTaps], t[kMaxTaps];  // its phase's tap count and index in it
    int off[kMaxTaps];                 // element offset of its phase's [Cp][T][Fp] block
};

// Backward-data weights: wt[c][t][f] = w[f][a_t][b_t][c].
// 32 x 32 (f, c) tiles through shared memory so that both the read of
// w[f][a][b][c] (c contiguous) and the write of wt[c][t][f] (f contiguous) are
// coalesced. grid = (ceil(Cp/32), ceil(Fp/32), T), block = 32 x 8.
__global__ void weight_transform_kernel(const __nv_bfloat16 *__restrict__ w,
                                        __nv_bfloat16 *__restrict__ wt_base, int F, int Fp, int C,
                                        int Cp, int K, const __grid_constant__ TapTable tt) {
    pdl_wait();  // (launch.cuh: PDL)
    __shared__ __nv_bfloat16 tile[32][33];
    const int c0 = blockIdx.x * 32, f0 = blockIdx.y * 32, j = blockIdx.z;
    const int T = tt.T[j], t = tt.t[j];
    __nv_bfloat16 *__restrict__ wt = wt_base + tt.off[j];
    const int tx = threadIdx.x, ty = threadIdx.y;
    const long long tap_off = ((long long)tt.a[j] * K + tt.b[j]) * Cp;
    for (int r = ty; r < 32; r += 8) {
        const int f = f0 + r, c = c0 + tx;
        __nv_bfloat16 v = __float2bfloat16(0.0f);
        if (f < F && c < C) v = w[(long long)f * K * K * Cp + tap_off + c];
        tile[r][tx] = v;
    }
    __syncthreads();
    for (int r = ty; r < 32; r += 8) {
        const int c = c0 + r, f = f0 + tx;
        if (c < Cp && f < Fp) wt[((long long)c * T + t) * Fp + f] = tile[tx][r];
    }
}

// ============================================================================
// host side
// ============================================================================
typedef CUresult (*PFN_encodeTiled)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                     const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                     const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &ptr, 12000,
                                             cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_encodeTiled>(ptr);
    });
    DC_REQUIRE(fn != nullptr, DC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
    return fn;
}

void make_tmap(CUtensorMap *m, const void *ptr, int rank, const uint64_t *dims,
               const uint64_t *strides_bytes, const uint32_t *box, const uint32_t *estrides,
               int swizzle_bytes) {
    const CUtensorMapSwizzle sw = swizzle_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                  : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                  : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                        : CU_TENSOR_MAP_SWIZZLE_NONE;
    cuuint64_t d[5], s[4];
    cuuint32_t b[5], e[5];
    for (int i = 0; i < rank; ++i) {
        d[i] = dims[i];
        b[i] = box[i];
        e[i] = estrides ? estrides[i] : 1;
        if (i < rank - 1) s[i] = strides_bytes[i];
    }
    CUresult r = get_encode()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void *>(ptr), d,
                              s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DC_REQUIRE(r == CUDA_SUCCESS, DC_ERR_CUDA,
               "cuTensorMapEncodeTiled failed (%d): rank %d dims %llu,%llu box %u,%u swz %d", (int)r,
               rank, (unsigned long long)d[0], (unsigned long long)(rank > 1 ? d[1] : 0), b[0],
               rank > 1 ? b[1] : 0, swizzle_bytes);
}

void make_tmap_ex(CUtensorMap *m, const void *ptr, int rank, const uint64_t *dims, const uint64_t *strides_bytes,
                  const uint32_t *box, const uint32_t *estrides, CUtensorMapDataType dt, CUtensorMapSwizzle sw) {
    cuuint64_t d[5], s[4];
    cuuint32_t b[5], e[5];
    for (int i = 0; i < rank; ++i) {
        d[i] = dims[i];
        b[i] = box[i];
        e[i] = estrides ? estrides[i] : 1;
        if (i < rank - 1) s[i] = strides_bytes[i];
    }
    CUresult r = get_encode()(m, dt, rank, const_cast<void *>(ptr), d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    DC_REQUIRE(r == CUDA_SUCCESS, DC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d): rank %d dims %llu,%llu box %u,%u",
               (int)r, rank, (unsigned long long)d[0], (unsigned long long)(rank > 1 ? d[1] : 0), b[0],
               rank > 1 ? b[1] : 0);
}

size_t conv_gemm_smem_bytes(int bkc, int bn, int stages) {
    return 1024 + (size_t)stages * (128 * bkc * 2 + bn * bkc * 2) + (2 * stages + 1) * 8 + 16;
}
size_t wgrad_smem_bytes(int bkc, int bf, int bn, int stages) {
    (void)bkc;
    (void)bf;
    return 1024 + (size_t)stages * (128 * 64 * 2 + bn * 64 * 2) + (2 * stages + 1) * 8 + 16;
}

#define CUDA_OK(x)                                                                        \
    do {                                                                                  \
        cudaError_t _e = (x);                                                             \
        DC_REQUIRE(_e == cudaSuccess, DC_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(_e)); \
    } while (0)

void launch_conv_gemm(const CUtensorMap &amap, const CUtensorMap &bmap, const ConvGemmParams &p,
                      int nsamples, int nout_tiles, cudaStream_t st) {
    const int tiles = p.rect_start[p.nrect];
    if (tiles == 0 || nsamples == 0 || nout_tiles == 0) return;
    const size_t smem = tmem_kernel_smem(conv_gemm_smem_bytes(p.bkc, p.bn, p.stages));
    static std::once_flag once;
    std::call_once(once, [] {
        cudaFuncSetAttribute(conv_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             227 * 1024);
    });
    if (g_dry_run) return;
    conv_gemm_kernel<<<dim3(tiles, nsamples, nout_tiles), 128, smem, st>>>(amap, bmap, p);
    CUDA_OK(cudaGetLastError());
    ++g_launches;
}

void launch_wgrad(const CUtensorMap &amap, const CUtensorMap &bmap, const WgradParams &p,
                  int m_tiles, int n_tiles, cudaStream_t st) {
    const size_t smem = tmem_kernel_smem(wgrad_smem_bytes(p.bkc, p.bf, p.bn, p.stages));
    static std::once_flag once;
    std::call_once(once, [] {
        cudaFuncSetAttribute(wgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    });
    if (g_dry_run) return;
    wgrad_kernel<<<dim3(m_tiles, n_tiles, p.splits), 128, smem, st>>>(amap, bmap, p);
    CUDA_OK(cudaGetLastError());
    ++g_launches;
}

void launch_splitk_reduce(const float *ws, int splits, long long n, long long split_stride, float *dw,
                          cudaStream_t st) {
    DC_REQUIRE(split_stride % 4 == 0 && split_stride >= n, DC_ERR_ARG, "split-K workspace stride");
    const long long nv = n % 4 == 0 ? n / 4 : n;
    const int blocks = (int)std::max<long long>(1, std::min<long long>((nv + 255) / 256, 148 * 8));
    launch_k(splitk_reduce_kernel, dim3(blocks), dim3(256), 0, st, 1, "split-K reduce", ws, splits, n, split_stride,
             dw);
}

void launch_weight_transform_multi(const __nv_bfloat16 *w, __nv_bfloat16 *wt_base, int F, int Fp, int C, int Cp,
                                   int K, int ntaps, const int8_t *ka, const int8_t *kb, const int *T,
                                   const int *t, const long long *off, cudaStream_t st) {
    if (ntaps == 0) return;
    DC_REQUIRE(ntaps <= kMaxTaps, DC_ERR_ARG, "too many taps");
    TapTable tt{};
    for (int j = 0; j < ntaps; ++j) {
        tt.a[j] = ka[j], tt.b[j] = kb[j];
        tt.T[j] = (uint8_t)T[j], tt.t[j] = (uint8_t)t[j];
        DC_REQUIRE(off[j] < (1LL << 31), DC_ERR_ARG, "weight block too large");
        tt.off[j] = (int)off[j];
    }
    launch_k(weight_transform_kernel, dim3((Cp + 31) / 32, (Fp + 31) / 32, ntaps), dim3(32, 8), 0, st, 1,
             "weight transform", w, wt_base, F, Fp, C, Cp, K, tt);
}

// Sub-pixel backward-data weights (stride 2): row n = phase * Cp + c, phase =
// 2 rho_h + rho_w, tap (dh, dw) of the D x D dy window starting at offset
// dmin: wt[n][dh * D + dw][f] = w[f][a_h][a_w][c] with a = rho + P - 2 (d + dmin),
// zero when a falls outside the filter (the phase does not use that tap).
__global__ void subpix_weight_kernel(const __nv_bfloat16 *__restrict__ w, __nv_bfloat16 *__restrict__ wt, int F,
                                     int Fp, int C, int Cp, int K, int P, int dmin, int D) {
    pdl_wait();  // (launch.cuh: PDL)
    const int n = blockIdx.x, tap = blockIdx.y, T = D * D;
    const int ph = n / Cp, c = n - ph * Cp, rh = ph >> 1, rw = ph & 1;
    const int dh = tap / D, dw = tap - dh * D;
    const int ah = rh + P - 2 * (dh + dmin), aw = rw + P - 2 * (dw + dmin);
    const bool in = c < C && ah >= 0 && ah < K && aw >= 0 && aw < K;
    for (int f = threadIdx.x; f < Fp; f += blockDim.x) {
        __nv_bfloat16 v = __float2bfloat16(0.0f);
        if (in && f < F) v = w[(((long long)f * K + ah) * K + aw) * Cp + c];
        wt[((long long)n * T + tap) * Fp + f] = v;
    }
}

void launch_subpix_weights(const __nv_bfloat16 *w, __nv_bfloat16 *wt, int F, int Fp, int C, int Cp, int K, int P,
                           int dmin, int D, cudaStream_t st) {
    launch_k(subpix_weight_kernel, dim3(4 * Cp, D * D), dim3(64), 0, st, 1, "sub-pixel weights", w, wt, F, Fp, C,
             Cp, K, P, dmin, D);
}

void launch_weight_transform(const __nv_bfloat16 *w, __nv_bfloat16 *wt, int F, int Fp, int C,
                             int Cp, int K, int T, const int8_t *ka, const int8_t *kb,
                             cudaStream_t st) {
    int Ts[kMaxTaps], ts[kMaxTaps];
    long long off[kMaxTaps];
    for (int i = 0; i < T; ++i) Ts[i] = T, ts[i] = i, off[i] = 0;
    launch_weight_transform_multi(w, wt, F, Fp, C, Cp, K, T, ka, kb, Ts, ts, off, st);
}


// Loads this file's kernels now (CUDA lazy loading would otherwise load a
// kernel at its first launch, which waits for the device: with the spinning
// halo / BN protocol kernels of a loopback group in flight, that wait never
// ends).
void preload_conv_tc() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(conv_gemm_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(wgrad_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(splitk_reduce_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(weight_transform_kernel));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(subpix_weight_kernel));
}

}  // namespace dc

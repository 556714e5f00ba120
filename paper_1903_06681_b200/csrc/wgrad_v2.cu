// wgrad_v2.cu -- backward-filter (Eq. 2) as a tile-reuse
// implicit GEMM on sm_100a:
//   D[(tap, c), f] = sum over the owned output pixels of X_tap[pixel, c] * DY[pixel, f]
// K = output pixels, processed in blocks of 8 output rows x 8 output cols.
// For each block the x tile that ALL taps read is loaded once into shared
// memory (128B-swizzled rows of 64 channels, row pitch 16 pixels, one plane
// per column parity for stride 2); an "MN atom" of the A operand is 64
// channels of one tap, i.e. the same tile at a shifted start address, and an
// M = 128 tile pairs two atoms (LBO = their distance). dy (without halo,
// PAPER.md:143) is streamed once per block. A CTA keeps the accumulators of
// all its M tiles in TMEM across its whole split-K range; partial sums go to
// a workspace reduced in a fixed order (splitk_reduce_kernel).
#include <algorithm>
#include <mutex>

#include "common.hpp"
#include "conv_v2.cuh"
#include "sm100.cuh"
#include "wgrad_v2.cuh"

namespace dc {
using namespace sm100;

namespace {
__device__ __forceinline__ uint8_t *align1024w(uint8_t *p) {
    const uint32_t a = smem_u32(p);
    return p + ((1024 - (a & 1023)) & 1023);
}
}  // namespace

constexpr int kWMaxStages = 8;

__global__ void __launch_bounds__(192, 1)
    wgrad_v2_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap dymap,
                    const __grid_constant__ WgradV2Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024w(smem_raw);
    uint8_t *sX = smem;
    uint8_t *sD = sX + p.stages * p.x_stage_bytes;
    uint64_t *full = reinterpret_cast<uint64_t *>(sD + p.stages * p.dy_stage_bytes);
    uint64_t *empty = full + kWMaxStages;
    uint64_t *done = empty + kWMaxStages;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(done + 1);

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const int mg = blockIdx.x, f0 = blockIdx.y * p.bn, split = blockIdx.z;
    const int mt0 = mg * p.G;
    const int G = min(p.G, p.n_mtiles - mt0);
    const int a_lo = 2 * mt0;
    const int cg_lo = a_lo / p.T;
    const int a_hi = min(2 * (mt0 + G), p.natoms) - 1;
    const int cg_hi = a_hi / p.T;
    const int ncg = cg_hi - cg_lo + 1;
    const int b_begin = (int)((long long)split * p.nblocks / p.splits);
    const int b_end = (int)((long long)(split + 1) * p.nblocks / p.splits);
    const int KB = b_end - b_begin;
    const uint32_t ncols = 512;

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(done, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, ncols);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        // ===================== TMA producer (warp-uniform) =====================
        if (elect_one()) {
            tma_prefetch(&xmap);
            tma_prefetch(&dymap);
        }
        const int per_n = p.tiles_h * p.tiles_w;
        const uint32_t x_bytes = ncg * p.s_in * p.PH * 16 * 128;
        const uint32_t d_bytes = (p.bn / 64) * 64 * 64 * 2;
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % p.stages;
            if (kb >= p.stages) mbar_wait(&empty[s], ((kb / p.stages) - 1) & 1);
            const int blk = b_begin + kb;
            const int n = blk / per_n, rem = blk - n * per_n;
            const int i0 = (rem / p.tiles_w) * 8, j0 = (rem % p.tiles_w) * 8;
            if (elect_one()) {
                mbar_arrive_expect_tx(&full[s], x_bytes + d_bytes);
                uint8_t *xs = sX + s * p.x_stage_bytes;
                const int h0 = p.s_in * i0 + p.origin_h, w0 = p.s_in * j0 + p.origin_w;
                for (int c = 0; c < ncg; ++c)
                    for (int par = 0; par < p.s_in; ++par)
                        tma_load_4d(xs + (c * p.s_in + par) * p.x_plane_bytes, &xmap, &full[s],
                                    (cg_lo + c) * 64, w0 + par, h0, n);
                uint8_t *ds = sD + s * p.dy_stage_bytes;
                for (int q = 0; q < p.bn / 64; ++q)
                    tma_load_4d(ds + q * 64 * 64 * 2, &dymap, &full[s], f0 + q * 64, j0, i0, n);
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // ===================== tcgen05.mma issuer (warp-uniform) =====================
        // A (x, MN-major SW128): atom = 64 channels of one tap; K rows = 8 output
        // pixels of one output row (128 B each); SBO = next output row.
        const uint32_t a_sbo = p.s_in * 16 * 128;
        uint64_t adesc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            adesc[i] = 0;
            if (i < G) {
                int a0 = 2 * (mt0 + i), a1 = a0 + 1;
                if (a1 >= p.natoms) a1 = a0;
                auto off = [&](int a) -> uint32_t {
                    const int cg = a / p.T, t = a - cg * p.T;
                    const int th = t / p.kw, tw = t - th * p.kw;
                    return (uint32_t)(((cg - cg_lo) * p.s_in + (tw % p.s_in)) * p.x_plane_bytes +
                                      (th * 16 + tw / p.s_in) * 128);
                };
                uint32_t o0 = off(a0), o1 = off(a1);
                const bool swap = o1 < o0;
                if (swap) {
                    const uint32_t t = o0;
                    o0 = o1;
                    o1 = t;
                }
                adesc[i] = smem_desc(smem_u32(sX) + o0, o1 - o0 > 0 ? o1 - o0 : 16, a_sbo, 2);
            }
        }
        // B (dy, MN-major SW128): atom = 64 filters; K rows = 8 pixels x 128 B;
        // SBO = 1024 (next 8 pixels = next output row), LBO = next 64 filters.
        const uint64_t bdesc0 = smem_desc(smem_u32(sD), 64 * 64 * 2, 1024, 2);
        const uint32_t idesc = idesc_bf16(128, p.bn, 1, 1);
        const uint32_t acc_cols = p.bn_cols;
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % p.stages;
            mbar_wait(&full[s], (kb / p.stages) & 1);
            tc_fence_after();
            if (elect_one()) {
                const uint32_t xo = (uint32_t)(s * p.x_stage_bytes) >> 4;
                const uint64_t bd = bdesc0 + ((uint32_t)(s * p.dy_stage_bytes) >> 4);
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    if (i < G) {
#pragma unroll
                        for (int k = 0; k < 4; ++k)  // 64 pixels = 4 x K16 (2 output rows each)
                            mma_bf16(tmem + i * acc_cols, adesc[i] + xo + k * ((2 * a_sbo) >> 4),
                                     bd + k * (2048 >> 4), idesc, (kb | k) != 0);
                    }
                mma_commit(&empty[s]);
            }
            __syncwarp();
        }
        if (elect_one()) mma_commit(done);
        __syncwarp();
    } else {
        // ===================== epilogue: partial dW -> workspace =====================
        mbar_wait(done, 0);
        tc_fence_after();
        const int eq = warp & 3;
        const int m = eq * 32 + lane;
        float *wsb = p.ws + (long long)split * p.ws_split;
        const long long fstride = (long long)p.T * p.cp;
        for (int i = 0; i < G; ++i) {
            int a0 = 2 * (mt0 + i), a1 = a0 + 1;
            const bool phantom = a1 >= p.natoms;
            if (phantom) a1 = a0;
            // recompute the pair order the issuer used
            auto off = [&](int a) -> uint32_t {
                const int cg = a / p.T, t = a - cg * p.T;
                const int th = t / p.kw, tw = t - th * p.kw;
                return (uint32_t)(((cg - cg_lo) * p.s_in + (tw % p.s_in)) * p.x_plane_bytes +
                                  (th * 16 + tw / p.s_in) * 128);
            };
            const bool swap = off(a1) < off(a0);
            const int a = (m < 64) == !swap ? a0 : a1;  // rows 0-63: the atom at the lower address
            const bool valid = !(phantom && m >= 64);
            const int cg = a / p.T, t = a - cg * p.T;
            const int c = cg * 64 + (m & 63);
            float *wrow = wsb + (long long)t * p.cp + c;
            const uint32_t t_lane = tmem + i * p.bn_cols + ((uint32_t)(eq * 32) << 16);
            for (int c16 = 0; c16 < p.bn / 16; ++c16) {
                uint32_t v[16];
                if (KB > 0) {
                    tmem_ld16(t_lane + c16 * 16, v);
                    tmem_ld_wait();
                } else {
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = 0;
                }
                if (valid && c < p.cp) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const int f = f0 + c16 * 16 + e;
                        if (f < p.F) wrow[f * fstride] = __uint_as_float(v[e]);
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, ncols);
}

size_t wgrad_v2_smem_bytes(const WgradV2Params &p) {
    return 1024 + (size_t)p.stages * (p.x_stage_bytes + p.dy_stage_bytes) + (2 * kWMaxStages + 1) * 8 + 16;
}

bool wgrad_v2_configure(WgradV2Params &p, int smem_limit) {
    if (p.cp % 64 != 0 || p.Fp % 64 != 0 || p.kh * p.kw != p.T) return false;
    p.PH = p.s_in * 7 + p.kh;
    if (p.PH > 256 || 8 + (p.kw - 1) / p.s_in > 16) return false;
    p.x_plane_bytes = p.PH * 16 * 128;
    p.bn = p.Fp <= 256 ? p.Fp : 256;
    p.bn_cols = p.bn <= 32 ? 32 : p.bn <= 64 ? 64 : p.bn <= 128 ? 128 : 256;
    p.natoms = (p.cp / 64) * p.T;
    p.n_mtiles = (p.natoms + 1) / 2;
    p.G = std::max(1, std::min(8, 512 / p.bn_cols));
    // channel groups an M group can touch: atoms [2 mt0, 2 mt0 + 2G) span
    const int span_atoms = 2 * p.G;
    const int ncg_max = std::min(p.cp / 64, (span_atoms + p.T - 2) / p.T + 1);
    p.x_stage_bytes = ncg_max * p.s_in * p.x_plane_bytes;
    p.dy_stage_bytes = (p.bn / 64) * 64 * 64 * 2;
    const int fixed = 1024 + (2 * kWMaxStages + 1) * 8 + 16;
    p.stages = std::min(kWMaxStages, (smem_limit - fixed) / (p.x_stage_bytes + p.dy_stage_bytes));
    if (p.stages < 2) {
        // fewer M tiles per CTA -> fewer channel groups per stage
        while (p.G > 1 && p.stages < 2) {
            p.G /= 2;
            const int ncg2 = std::min(p.cp / 64, (2 * p.G + p.T - 2) / p.T + 1);
            p.x_stage_bytes = ncg2 * p.s_in * p.x_plane_bytes;
            p.stages = std::min(kWMaxStages, (smem_limit - fixed) / (p.x_stage_bytes + p.dy_stage_bytes));
        }
    }
    return p.stages >= 2;
}

void launch_wgrad_v2(const CUtensorMap &xmap, const CUtensorMap &dymap, const WgradV2Params &p,
                     cudaStream_t st) {
    static std::once_flag once;
    std::call_once(once, [] {
        cudaFuncSetAttribute(wgrad_v2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kV2SmemLimit);
    });
    const int mgroups = (p.n_mtiles + p.G - 1) / p.G;
    const int ntiles = (p.Fp + p.bn - 1) / p.bn;
    wgrad_v2_kernel<<<dim3(mgroups, ntiles, p.splits), 192, wgrad_v2_smem_bytes(p), st>>>(xmap, dymap, p);
    cudaError_t e = cudaGetLastError();
    DC_REQUIRE(e == cudaSuccess, DC_ERR_CUDA, "wgrad_v2 launch: %s", cudaGetErrorString(e));
    ++g_launches;
}

}  // namespace dc

// wgrad_v2.cu -- backward-filter (Eq. 2) as a tile-reuse
// implicit GEMM on sm_100a:
//   D[(tap, c), f] = sum over the owned output pixels of X_tap[pixel, c] * DY[pixel, f]
// K = output pixels, processed in blocks of 8 output rows x 8 output cols.
// For each block the x tile that ALL taps read is loaded once into shared
// memory (swizzled rows of cgw channels, row pitch bw+(kw-1)/s pixels, one plane per
// column parity for stride 2). An "MN atom" of the A operand is cgw channels
// of one tap, i.e. the same tile at a shifted start address; an M = 128 tile
// stacks 128/cgw atoms at a uniform distance (LBO):
//   mode 0 (cgw = 64, >= 2 taps): two taps of one channel group (any pair;
//          LBO = their distance, the lower address first);
//   mode 1 (cgw = 16/32): 128/cgw taps of one filter column (th, th+1, ...):
//          LBO = one input row of the tile; taps past the filter are phantoms;
//   mode 2 (1x1, cgw = 64): the single tap of two channel groups.
// dy (without halo) is streamed once per block. A CTA keeps
// the accumulators of all its M tiles in TMEM across its split-K range;
// partial sums go to a workspace reduced in a fixed order
// (splitk_reduce_kernel) -> deterministic (the default; DC_DW_ATOMIC lets small
// dW splits add with fp32 reductions instead).
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "common.hpp"
#include "conv_v2.cuh"
#include "sm100.cuh"
#include "wgrad_v2.cuh"
#include "launch.cuh"

namespace dc {
using namespace sm100;

namespace {
__device__ __forceinline__ uint8_t *align1024w(uint8_t *p) {
    const uint32_t a = smem_u32(p);
    return p + ((1024 - (a & 1023)) & 1023);
}

// Atom `a` (0 .. 128/cgw - 1) of M tile `mt`: its tap (or -1: phantom) and
// channel group, and its byte offset inside the CTA's x stage.
struct Atom {
    int tap, cg;
    uint32_t off;
};
__host__ __device__ inline Atom atom_of(const WgradV2Params &p, int mt, int a, int cg_lo) {
    Atom r{-1, 0, 0};
    const int A = 128 / p.cgw;
    auto offset = [&](int cg, int th, int tw) -> uint32_t {
        return (uint32_t)(((cg - cg_lo) * p.s_in + (tw % p.s_in)) * p.x_plane_bytes +
                          (th * p.pitch + tw / p.s_in) * p.cgw * p.esz);
    };
    if (p.mode == 2) {  // 1x1: channel groups A mt .. A mt + A - 1
        const int cg = A * mt + a;
        r.cg = cg < p.ncg ? cg : A * mt;
        r.tap = cg < p.ncg ? 0 : -1;
        r.off = offset(r.cg, 0, 0);
    } else if (p.mode == 0) {  // pairs of taps inside one channel group
        const int per = (p.T + 1) / 2;
        const int cg = mt / per, pair = mt % per;
        const int t = 2 * pair + a;
        r.cg = cg;
        r.tap = t < p.T ? t : -1;
        const int tt = t < p.T ? t : 2 * pair;
        r.off = offset(cg, tt / p.kw, tt % p.kw);
    } else {  // filter column tw, taps th = thb*A + a
        const int nthb = (p.kh + A - 1) / A;
        const int per = p.kw * nthb;
        const int cg = mt / per, rem = mt % per;
        const int tw = rem % p.kw, thb = rem / p.kw;
        const int th = thb * A + a;
        r.cg = cg;
        r.tap = th < p.kh ? th * p.kw + tw : -1;
        r.off = offset(cg, th, tw);  // phantom rows exist in the tile (PH padded)
    }
    return r;
}
}  // namespace

constexpr int kWMaxStages = 8;

// The MMAs of one pixel block: G M tiles x 4 K16 steps, fully unrolled (the
// descriptors are loop-invariant per CTA; only the stage offset moves).
// (KIND 1: K = 8 pixel steps of kind::tf32, B rows 1024 bytes per step)
template <int KIND, int G, int NKS>
__device__ __forceinline__ void wgrad_issue(uint32_t tmem, const uint64_t (&adesc)[8], uint32_t xo, uint64_t bd,
                                            uint32_t ak16, uint32_t acc_cols, uint32_t idesc, bool first) {
    constexpr uint32_t bk16 = (KIND == 1 ? 1024 : 2048) >> 4;
#pragma unroll
    for (int i = 0; i < G; ++i)
#pragma unroll
        for (int k = 0; k < NKS; ++k) {  // NKS x K steps of 16 (bf16) / 8 (tf32) pixels
            if constexpr (KIND == 1)
                mma_tf32(tmem + i * acc_cols, adesc[i] + xo + k * ak16, bd + k * bk16, idesc,
                         (first && k == 0) ? 0u : 1u);
            else
                mma_bf16(tmem + i * acc_cols, adesc[i] + xo + k * ak16, bd + k * bk16, idesc,
                         (first && k == 0) ? 0u : 1u);
        }
}
template <int KIND, int NKS>
__device__ __forceinline__ void wgrad_issue_g(int G, uint32_t tmem, const uint64_t (&adesc)[8], uint32_t xo,
                                              uint64_t bd, uint32_t ak16, uint32_t acc_cols, uint32_t idesc,
                                              bool first) {
    switch (G) {
    case 1: wgrad_issue<KIND, 1, NKS>(tmem, adesc, xo, bd, ak16, acc_cols, idesc, first); break;
    case 2: wgrad_issue<KIND, 2, NKS>(tmem, adesc, xo, bd, ak16, acc_cols, idesc, first); break;
    case 3: wgrad_issue<KIND, 3, NKS>(tmem, adesc, xo, bd, ak16, acc_cols, idesc, first); break;
    case 4: wgrad_issue<KIND, 4, NKS>(tmem, adesc, xo, bd, ak16, acc_cols, idesc, first); break;
    case 5: wgrad_issue<KIND, 5, NKS>(tmem, adesc, xo, bd, ak16, acc_cols, idesc, first); break;
    case 6: wgrad_issue<KIND, 6, NKS>(tmem, adesc, xo, bd, ak16, acc_cols, idesc, first); break;
    case 7: wgrad_issue<KIND, 7, NKS>(tmem, adesc, xo, bd, ak16, acc_cols, idesc, first); break;
    default: wgrad_issue<KIND, 8, NKS>(tmem, adesc, xo, bd, ak16, acc_cols, idesc, first); break;
    }
}

template <int KIND>
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
    const int A = 128 / p.cgw;
    // this CTA's M tiles: [mt0, mt0 + G) (never crossing a channel group in modes 0/1)
    const int f0 = blockIdx.y * p.bn, split = blockIdx.z;
    int mt0, G;
    if (p.mode == 2) {
        mt0 = blockIdx.x * p.G;
        G = min(p.G, p.n_mtiles - mt0);
    } else {
        const int per_cg = p.n_mtiles / p.ncg, groups = (per_cg + p.G - 1) / p.G;
        const int cg = blockIdx.x / groups, gi = blockIdx.x % groups;
        mt0 = cg * per_cg + gi * p.G;
        G = min(p.G, per_cg - gi * p.G);
    }
    const int cg_lo = atom_of(p, mt0, 0, 0).cg;
    const int cg_hi = p.mode == 2 ? min(p.ncg, A * (mt0 + G)) - 1 : cg_lo;
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
    pdl_wait();  // (launch.cuh: PDL) the prologue above touched only smem / TMEM

    if (warp == 0) {
        // ===================== TMA producer (warp-uniform) =====================
        if (elect_one()) {
            tma_prefetch(&xmap);
            tma_prefetch(&dymap);
        }
        const int per_n = p.tiles_h * p.tiles_w;
        const uint32_t x_bytes = ncg * p.s_in * p.PH * p.pitch * p.cgw * p.esz;  // bytes the boxes deliver
        const int fbox = 128 / p.esz;  // filters per dy box (one 128-byte row)
        const uint32_t d_bytes = (p.bn / fbox) * 8 * p.bw * 128;
        for (int kb = 0; kb < KB; ++kb) {
            const int s = kb % p.stages;
            if (kb >= p.stages) mbar_wait(&empty[s], ((kb / p.stages) - 1) & 1);
            // 3xTF32: pass 0 x_hi dy_hi, 1 x_hi dy_lo, 2 x_lo dy_hi (one accumulation)
            const int pass = (b_begin + kb) / p.nblocks_pix;
            const int blk = b_begin + kb - pass * p.nblocks_pix;
            const int xc = pass == 2 ? p.x_lo : 0, fc = pass == 1 ? p.dy_lo : 0;
            const int n = blk / per_n, rem = blk - n * per_n;
            const int i0 = (rem / p.tiles_w) * 8, j0 = (rem % p.tiles_w) * p.bw;
            if (elect_one()) {
                mbar_arrive_expect_tx(&full[s], x_bytes + d_bytes);
                uint8_t *xs = sX + s * p.x_stage_bytes;
                const int h0 = p.s_in * i0 + p.origin_h, w0 = p.s_in * j0 + p.origin_w;
                for (int c = 0; c < ncg; ++c)
                    for (int par = 0; par < p.s_in; ++par)
                        tma_load_4d(xs + (c * p.s_in + par) * p.x_plane_bytes, &xmap, &full[s],
                                    (cg_lo + c) * p.cgw + xc, w0 + par, h0, n);
                uint8_t *ds = sD + s * p.dy_stage_bytes;
                for (int q = 0; q < p.bn / fbox; ++q)
                    tma_load_4d(ds + q * 8 * p.bw * 128, &dymap, &full[s], f0 + q * fbox + fc, j0, i0, n);
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // ===================== tcgen05.mma issuer (warp-uniform) =====================
        // A (x, MN-major, swizzle = cgw*2 bytes): K rows = 8 output pixels of one
        // output row (cgw*2 bytes each); SBO = next output row; LBO = next atom.
        // K rows = pixels: 8-pixel groups (SBO) are the next 8 output pixels of a
        // row (bw = 16) or the next output row (bw = 8); a K16 step is 16 pixels
        // tf32 (bw = 8): a K = 8 step is one output row, two groups of 4 pixels
        // (SBO = 4 rows of 128 B), 32-byte-granule swizzle (layout 1)
        const uint32_t row_bytes = p.s_in * p.pitch * p.cgw * p.esz;
        const uint32_t a_sbo = KIND == 1 ? 4 * 128 : p.bw == 16 ? 8 * p.cgw * 2 : row_bytes;
        const uint32_t layout = KIND == 1 ? kLayoutSw128Base32B : swizzle_layout(p.cgw * 2);
        uint64_t adesc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            adesc[i] = 0;
            if (i < G) {
                const Atom a0 = atom_of(p, mt0 + i, 0, cg_lo), a1 = atom_of(p, mt0 + i, 1, cg_lo);
                uint32_t lo = a0.off, lbo;
                if (p.mode == 0) {  // arbitrary pair: lower address first
                    lo = min(a0.off, a1.off);
                    lbo = max(a0.off, a1.off) - lo;
                    if (lbo == 0) lbo = 16;  // phantom partner: rows discarded
                } else {
                    lbo = a1.off - a0.off;  // uniform spacing (input row / channel group)
                }
                adesc[i] = smem_desc(smem_u32(sX) + lo, lbo, a_sbo, layout);
            }
        }
        // B (dy, MN-major SW128): atom = 64 filters; K rows = 8 pixels x 128 B;
        // SBO = 1024 (next 8 pixels = next output row), LBO = next 64 filters.
        // (tf32: atom = 32 filters, 4-pixel groups: SBO = 512, layout 1)
        const uint64_t bdesc0 = KIND == 1 ? smem_desc(smem_u32(sD), 8 * p.bw * 128, 512, kLayoutSw128Base32B)
                                          : smem_desc(smem_u32(sD), 8 * p.bw * 128, 1024, 2);
        const uint32_t idesc = KIND == 1 ? idesc_tf32(128, p.bn, 1, 1) : idesc_bf16(128, p.bn, 1, 1);
        const uint32_t acc_cols = p.bn_cols;
        const uint32_t ak16 = (KIND == 1 || p.bw == 16 ? row_bytes : 2 * row_bytes) >> 4;
        const uint32_t xstep = (uint32_t)p.x_stage_bytes >> 4, dstep = (uint32_t)p.dy_stage_bytes >> 4;
        int s = 0;
        uint32_t ph = 0, xo = 0;
        uint64_t bd = bdesc0;
        for (int kb = 0; kb < KB; ++kb) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            if (elect_one()) {
                if (KIND == 1 || p.bw == 16)  // 8 steps: 8 x 16 (bf16) or 8 x 8 (tf32, bw 8) pixels
                    wgrad_issue_g<KIND, 8>(G, tmem, adesc, xo, bd, ak16, acc_cols, idesc, kb == 0);
                else
                    wgrad_issue_g<KIND, 4>(G, tmem, adesc, xo, bd, ak16, acc_cols, idesc, kb == 0);
                mma_commit(&empty[s]);
            }
            __syncwarp();
            if (++s == p.stages) {
                s = 0, ph ^= 1, xo = 0, bd = bdesc0;
            } else {
                xo += xstep, bd += dstep;
            }
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
        const long long fstride = (long long)p.T * p.C;  // dW holds the C logical channels
        for (int i = 0; i < G; ++i) {
            const Atom a0 = atom_of(p, mt0 + i, 0, cg_lo);
            int ai = m / p.cgw;
            if (p.mode == 0) {  // rows 0-63 hold the atom at the lower address
                const Atom a1 = atom_of(p, mt0 + i, 1, cg_lo);
                if (a1.off < a0.off) ai = 1 - ai;
            }
            const Atom at = atom_of(p, mt0 + i, ai, cg_lo);
            const int c = at.cg * p.cgw + (m % p.cgw);
            const bool valid = at.tap >= 0 && c < p.C;
            float *wrow = wsb + (long long)(valid ? at.tap : 0) * p.C + c;
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
                if (valid && p.atomic_out) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const int f = f0 + c16 * 16 + e;
                        if (f < p.F) atomicAdd(&wrow[f * fstride], __uint_as_float(v[e]));  // RED.ADD.F32
                    }
                } else if (valid) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        const int f = f0 + c16 * 16 + e;
                        if (f < p.F) wrow[f * fstride] = __uint_as_float(v[e]);
                    }
                }
            }
        }
        (void)A;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, ncols);
}

size_t wgrad_v2_smem_bytes(const WgradV2Params &p) {
    return 1024 + (size_t)p.stages * (p.x_stage_bytes + p.dy_stage_bytes) + (2 * kWMaxStages + 1) * 8 + 16;
}

int wgrad_v2_mgroups(const WgradV2Params &p) {
    if (p.mode == 2) return (p.n_mtiles + p.G - 1) / p.G;
    const int per_cg = p.n_mtiles / p.ncg;
    return p.ncg * ((per_cg + p.G - 1) / p.G);
}

static bool wgrad_v2_configure_bw(WgradV2Params &p, int smem_limit, int bw) {
    const bool tf32 = p.kind == 1;
    if ((!tf32 && p.Fp % 64 != 0) || p.kh * p.kw != p.T) return false;
    p.esz = tf32 ? 4 : 2;
    if (tf32) {
        // MN-major tf32 atoms are 128-byte rows: 32 channels (the last group
        // may reach into the lo half / past the buffer: those rows are
        // discarded, or TMA zero-fills them)
        p.cgw = 32;
        p.ncg = (p.cp + 31) / 32;
        bw = 8;
    } else {
        p.cgw = p.cp % 64 == 0 ? 64 : p.cp % 32 == 0 ? 32 : 16;
        p.ncg = p.cp / p.cgw;
    }
    if (8 + (p.kw - 1) / p.s_in > 32) return false;
    const int A = 128 / p.cgw;
    if (tf32) {
        p.mode = p.T == 1 ? 2 : 1;
        p.n_mtiles = p.T == 1 ? (p.ncg + A - 1) / A : p.ncg * p.kw * ((p.kh + A - 1) / A);
    } else if (p.T == 1 && p.cgw == 64) {
        p.mode = 2;
        p.n_mtiles = (p.ncg + 1) / 2;
    } else if (p.cgw == 64) {
        p.mode = 0;
        p.n_mtiles = p.ncg * ((p.T + 1) / 2);
    } else {
        p.mode = 1;
        p.n_mtiles = p.ncg * p.kw * ((p.kh + A - 1) / A);
    }
    // tile rows: 8 output rows -> s*7 + kh input rows (+ phantom rows of mode 1)
    const int kh_alloc = p.mode == 1 ? ((p.kh + A - 1) / A) * A : p.kh;
    p.PH = p.s_in * 7 + kh_alloc;
    if (p.PH > 256) return false;
    // row pitch = the 8 + (kw-1)/s columns one parity plane needs; the
    // swizzle is a function of the smem address, so rows need not start on
    // a swizzle-atom boundary (only 16-byte alignment)
    // pixel blocks of 8 rows x bw columns (16 by default: half the barrier
    // round trips per pixel and fewer halo columns than 8 x 8)
    p.bw = bw;
    p.pitch = p.bw + (p.kw - 1) / p.s_in;
    p.x_plane_bytes = (p.PH * p.pitch * p.cgw * p.esz + 1023) / 1024 * 1024;
    // N tile 256 (2 M tiles per x / dy stage in TMEM) once the launch has
    // >= 8192 output pixels, else 128 (4 M tiles per stage, half the bytes per
    // MMA). Measured, cold L2 (profiles/r1_wgrad_bn_sweep.txt): 256 wins
    // 8-25% from 16K pixels up (512-ch 128^2 N = 8: 561 -> 458 us; 256-ch
    // 256^2: 510 -> 470 us), ties at 4K-8K, loses up to 14% below (512-ch
    // 32^2 N = 1: 31 -> 36 us).
    const int bn_cap = p.pixels_hint >= 8192 ? 256 : 128;
    // (tf32: N tiles of whole 32-filter dy boxes; filters past F are discarded)
    p.bn = tf32 ? std::min<int>(bn_cap, (p.Fp + 31) / 32 * 32) : p.Fp <= bn_cap ? p.Fp : bn_cap;
    p.bn_cols = p.bn <= 32 ? 32 : p.bn <= 64 ? 64 : p.bn <= 128 ? 128 : 256;
    p.G = std::max(1, std::min(8, 512 / p.bn_cols));
    if (p.mode != 2) {  // equal groups per channel group (e.g. 5 M tiles: 3 + 2, not 4 + 1):
        // the largest group sets the time, the loads are paid per group
        const int per_cg = p.n_mtiles / p.ncg;
        p.G = (per_cg + (per_cg + p.G - 1) / p.G - 1) / ((per_cg + p.G - 1) / p.G);
    }
    p.dy_stage_bytes = (p.bn / (128 / p.esz)) * 8 * p.bw * 128;
    const int fixed = 1024 + (2 * kWMaxStages + 1) * 8 + 16;
    for (;;) {
        const int ncg_stage = p.mode == 2 ? std::min(p.ncg, A * p.G) : 1;
        p.x_stage_bytes = (ncg_stage * p.s_in * p.x_plane_bytes + 1023) / 1024 * 1024;
        p.stages = std::min(kWMaxStages, (smem_limit - fixed) / (p.x_stage_bytes + p.dy_stage_bytes));
        if (p.stages >= 2 || p.G == 1) break;
        p.G /= 2;
    }
    return p.stages >= 2;
}

bool wgrad_v2_configure(WgradV2Params &p, int smem_limit) {
    // 8 x 16 pixel blocks unless two stages of them do not fit (stride 2 with
    // 256-filter tiles), then 8 x 8 (tf32: always 8 x 8)
    const WgradV2Params in = p;
    if (wgrad_v2_configure_bw(p, smem_limit, 16)) return true;
    p = in;
    return wgrad_v2_configure_bw(p, smem_limit, 8);
}

void launch_wgrad_v2(const CUtensorMap &xmap, const CUtensorMap &dymap, const WgradV2Params &p,
                     cudaStream_t st) {
    static std::once_flag once;
    std::call_once(once, [] {
        cudaFuncSetAttribute(wgrad_v2_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kV2SmemLimit);
        cudaFuncSetAttribute(wgrad_v2_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kV2SmemLimit);
    });
    const int ntiles = (p.Fp + p.bn - 1) / p.bn;
    launch_k(p.kind == 1 ? wgrad_v2_kernel<1> : wgrad_v2_kernel<0>, dim3(wgrad_v2_mgroups(p), ntiles, p.splits),
             dim3(192), tmem_kernel_smem(wgrad_v2_smem_bytes(p)), st, 1, p.kind == 1 ? "wgrad_v2 (tf32)" : "wgrad_v2", xmap, dymap, p);
}


// Loads this file's kernels now (CUDA lazy loading would otherwise load a
// kernel at its first launch, which waits for the device: with the spinning
// halo / BN protocol kernels of a loopback group in flight, that wait never
// ends).
void preload_wgrad_v2() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(wgrad_v2_kernel<0>));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(wgrad_v2_kernel<1>));
}

}  // namespace dc

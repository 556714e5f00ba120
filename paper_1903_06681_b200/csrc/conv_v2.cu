// conv_v2.cu -- persistent tile-reuse implicit-GEMM convolution on sm_100a
// (forward Eq. 1 PAPER.md:61 and backward-data Eq. 3).
//
// Warp roles (224 threads, 1 CTA per SM, persistent over output tiles):
//   warp 0      TMA producer: per tile and channel group, the halo'd input
//               tile as 16-byte core-matrix planes (one box per 8-channel
//               chunk and column parity); weights either resident (loaded
//               once) or streamed per (tap, channel group) through a ring.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer: for each
//               tap, the A descriptor is the same smem tile at a shifted
//               start address (no data movement per tap).
//   warps 2-5   epilogue: tcgen05.ld (32 lanes x 16 cols) -> bf16 -> NHWC
//               global stores (+ fused BN statistics); double-buffered TMEM
//               accumulators let the epilogue of tile i overlap the MMAs of
//               tile i+1.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

#include "common.hpp"
#include "conv_v2.cuh"
#include "launch.cuh"
#include "sm100.cuh"

namespace dc {
using namespace sm100;

namespace {
__device__ __forceinline__ uint8_t *align1024(uint8_t *p) {
    const uint32_t a = smem_u32(p);
    return p + ((1024 - (a & 1023)) & 1023);
}
// fp32 output column `col` of GEMM pixel (i, j) of sample n: plain out, or
// the scatter target of the column's channel block (ConvV2Params::scat)
__device__ __forceinline__ float *f32_out(const ConvV2Params &p, int n, int i, int j, int col) {
    float *base = reinterpret_cast<float *>(p.out);
    if (p.scat_seg) {
        const int ow = col / p.scat_seg;
        base = p.scat[ow];
        col -= ow * p.scat_seg;
    }
    return base + (long long)n * p.out_sn + (long long)(p.out_h0 + p.out_dh * i) * p.out_sh +
           (long long)(p.out_w0 + p.out_dw * j) * p.out_sw + col;
}
__device__ __forceinline__ uint32_t pack2(uint32_t lo, uint32_t hi) {
    __nv_bfloat162 v = __floats2bfloat162_rn(__uint_as_float(lo), __uint_as_float(hi));
    return *reinterpret_cast<uint32_t *>(&v);
}
__host__ __device__ inline uint32_t pow2_cols(int n) {
    uint32_t c = 32;
    while ((int)c < n) c <<= 1;
    return c;
}
struct TileCoord {
    int o0, n, i0, j0, r;
};
__device__ __forceinline__ TileCoord decode(const ConvV2Params &p, int u) {
    const int per_o = p.nsamples * p.rect_start[p.nrect];
    TileCoord c;
    const int ot = u / per_o;
    int rem = u - ot * per_o;
    c.n = rem / p.rect_start[p.nrect];
    const int lt = rem - c.n * p.rect_start[p.nrect];
    int r = 0;
    while (r + 1 < p.nrect && lt >= p.rect_start[r + 1]) ++r;
    const int t = lt - p.rect_start[r];
    c.r = r;
    c.i0 = p.rect[r].h0 + (t / p.rect_tiles_w[r]) * ((128 >> p.tw_log2) * p.tpw);
    c.j0 = p.rect[r].w0 + (t % p.rect_tiles_w[r]) * (1 << p.tw_log2);
    c.o0 = ot * p.bn;
    return c;
}
}  // namespace

constexpr int kMaxBar = 16;
// streamed weights: taps whose slots the MMA warp awaits before issuing them (conv_v2_kernel)
constexpr int kTapGroup = 3;

// one tcgen05.mma of the kernel's CTA group (1: this SM; 2: the pair, M = 256)
// KIND 0: kind::f16 (bf16 x bf16 -> fp32); KIND 1: kind::tf32 (fp32 operands
// read as tf32, 8 per 32-byte K step: the same smem geometry as 16 bf16)
template <int KIND>
__device__ __forceinline__ void mma_k(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if constexpr (KIND == 1)
        mma_tf32(d, a, b, idesc, acc);
    else
        mma_bf16(d, a, b, idesc, acc);
}

// Streamed weights: the MMAs of one weight slot (one tap of one channel group):
// NK x K16 steps for each of TPW stacked tiles, fully unrolled (compile-time
// multiples of hoisted strides, no per-MMA descriptor arithmetic chains).
template <int KIND, int NK, int TPW>
__device__ __forceinline__ void issue_slot(uint32_t d_tmem, uint64_t ad, uint64_t bd, uint32_t a_kstep,
                                           uint32_t a_tile16, uint32_t acc_cols, uint32_t idesc, bool first) {
#pragma unroll
    for (int k16 = 0; k16 < NK; ++k16)
#pragma unroll
        for (int tt = 0; tt < TPW; ++tt)
            mma_k<KIND>(d_tmem + tt * acc_cols, ad + k16 * a_kstep + tt * a_tile16, bd + 2 * k16, idesc,
                       (first && k16 == 0) ? 0u : 1u);
}
template <int KIND>
__device__ __forceinline__ void issue_slot_any(int nk16, int tpw, uint32_t d_tmem, uint64_t ad, uint64_t bd,
                                               uint32_t a_kstep, uint32_t a_tile16, uint32_t acc_cols,
                                               uint32_t idesc, bool first) {
    switch ((nk16 << 4) | tpw) {
    case 0x41: issue_slot<KIND, 4, 1>(d_tmem, ad, bd, a_kstep, a_tile16, acc_cols, idesc, first); break;
    case 0x42: issue_slot<KIND, 4, 2>(d_tmem, ad, bd, a_kstep, a_tile16, acc_cols, idesc, first); break;
    case 0x21: issue_slot<KIND, 2, 1>(d_tmem, ad, bd, a_kstep, a_tile16, acc_cols, idesc, first); break;
    case 0x22: issue_slot<KIND, 2, 2>(d_tmem, ad, bd, a_kstep, a_tile16, acc_cols, idesc, first); break;
    case 0x11: issue_slot<KIND, 1, 1>(d_tmem, ad, bd, a_kstep, a_tile16, acc_cols, idesc, first); break;
    default: issue_slot<KIND, 1, 2>(d_tmem, ad, bd, a_kstep, a_tile16, acc_cols, idesc, first); break;
    }
}

// Fully unrolled MMA issue for one channel group of one tile (resident
// weights): every descriptor offset is a compile-time multiple of a runtime
// stride hoisted out of the loop, so the single issuing thread spends a few
// uniform instructions per tcgen05.mma instead of a dependent chain of
// constant loads and 64-bit adds per tap (measured: ~180 cycles per tap).
template <int KIND, int KH, int KW, int NK, int SSH, int TPW>
__device__ __forceinline__ void issue_taps(uint32_t d_tmem, uint64_t a_stage, uint64_t bd,
                                           uint32_t a_row16, uint32_t a_col16, uint32_t a_par16,
                                           uint32_t a_kstep, uint32_t b_slot16, uint32_t idesc,
                                           bool first_group, uint32_t acc_cols, uint32_t a_tile16) {
#pragma unroll
    for (int th = 0; th < KH; ++th)
#pragma unroll
        for (int tw = 0; tw < KW; ++tw) {
            const uint64_t ad = a_stage + (uint32_t)th * a_row16 + (uint32_t)(tw >> SSH) * a_col16 +
                                (uint32_t)(tw & SSH) * a_par16;
            const uint64_t b = bd + (uint32_t)(th * KW + tw) * b_slot16;
#pragma unroll
            for (int k = 0; k < NK; ++k)
#pragma unroll
                for (int tt = 0; tt < TPW; ++tt)  // the tiles of the work item share the B slice
                    mma_k<KIND>(d_tmem + tt * acc_cols, ad + (uint32_t)k * a_kstep + tt * a_tile16, b + 2 * k,
                               idesc, (first_group && th == 0 && tw == 0 && k == 0) ? 0u : 1u);
        }
}

// Dispatch to an unrolled specialisation; false if none matches.
template <int KIND>
__device__ __forceinline__ bool issue_taps_fixed(const ConvV2Params &p, int nk16, uint32_t d_tmem,
                                                 uint64_t a_stage, uint64_t bd, uint32_t a_kstep,
                                                 uint32_t b_slot16, uint32_t idesc, bool first,
                                                 uint32_t acc_cols, uint32_t a_tile16) {
    const int key = (p.tpw << 16) | (p.kh << 12) | (p.kw << 8) | (nk16 << 4) | p.s_shift;
#define DC_TAPS(KH, KW, NK, SS)                                                                   \
    case ((1 << 16) | (KH << 12) | (KW << 8) | (NK << 4) | SS):                                   \
        issue_taps<KIND, KH, KW, NK, SS, 1>(d_tmem, a_stage, bd, p.a_row16, p.a_col16, p.a_par16,        \
                                      a_kstep, b_slot16, idesc, first, acc_cols, a_tile16);       \
        return true;                                                                              \
    case ((2 << 16) | (KH << 12) | (KW << 8) | (NK << 4) | SS):                                   \
        issue_taps<KIND, KH, KW, NK, SS, 2>(d_tmem, a_stage, bd, p.a_row16, p.a_col16, p.a_par16,        \
                                      a_kstep, b_slot16, idesc, first, acc_cols, a_tile16);       \
        return true;
    switch (key) {
        DC_TAPS(3, 3, 4, 0)  // 3x3 stride 1, 64-channel groups (fwd and bwd-data)
        DC_TAPS(1, 1, 4, 0)  // 1x1 (fwd, bwd-data, stride-2 phase)
        DC_TAPS(3, 3, 1, 0)
        DC_TAPS(3, 3, 2, 0)
        DC_TAPS(5, 5, 4, 0)
        DC_TAPS(7, 7, 1, 1)  // ResNet conv1 forward (C=3 -> 16, stride 2)
        DC_TAPS(3, 3, 2, 1)  // mesh conv1_1 forward (C=18 -> 32, stride 2)
        DC_TAPS(3, 3, 4, 1)  // 3x3 stride-2 forward, 64-channel groups (planes)
        DC_TAPS(4, 4, 4, 0)  // conv1 backward-data phases (7x7 / 2)
        DC_TAPS(4, 3, 4, 0)
        DC_TAPS(3, 4, 4, 0)
        DC_TAPS(2, 2, 4, 0)  // 3x3 / 2 backward-data phases
        DC_TAPS(2, 1, 4, 0)
        DC_TAPS(1, 2, 4, 0)
    default:
        return false;
    }
#undef DC_TAPS
}


// Per-channel sums of 16 channel values over the warp's 32 lanes (pixels):
// a fixed-order fp32 pairwise transpose-reduce; afterwards lanes 2k and 2k+1
// hold halves of channel k in a[0] / q[0] (caller adds them, lane order).
__device__ __forceinline__ void warp_chunk_reduce(float (&a)[16], float (&q)[16], uint32_t lane) {
#pragma unroll
    for (int w = 8; w >= 1; w >>= 1) {
        const bool up = (lane & (2 * w)) != 0;
#pragma unroll
        for (int j = 0; j < w; ++j) {
            const float sa = up ? a[j] : a[j + w], ka = up ? a[j + w] : a[j];
            const float sq = up ? q[j] : q[j + w], kq = up ? q[j + w] : q[j];
            a[j] = ka + __shfl_xor_sync(0xffffffffu, sa, 2 * w);
            q[j] = kq + __shfl_xor_sync(0xffffffffu, sq, 2 * w);
        }
    }
}

// warp 0 TMA, 1 MMA, 2-5 epilogue, 7-10 second epilogue group (p.epi2: the
// two groups split each tile's 16-column chunks, so twice as many TMEM loads
// and stores are in flight; warp 6 and, without epi2, 7-10 idle)
constexpr int kV2Threads = 352;

template <int KIND>
__global__ void __launch_bounds__(kV2Threads, 1)
    conv_v2_kernel(const __grid_constant__ CUtensorMap amap, const __grid_constant__ CUtensorMap bmap,
                   const __grid_constant__ ConvV2Params p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = align1024(smem_raw);
    uint8_t *sB = smem;  // B first: its slots need 1024-byte alignment (swizzle)
    const int b_bytes =
        p.b_resident ? p.T * (p.ncg / p.ksplit) * p.b_slot_bytes : p.b_stages * p.b_slot_bytes;
    uint8_t *sA = sB + b_bytes;
    uint64_t *bars = reinterpret_cast<uint64_t *>(sA + p.a_stages * p.a_stage_bytes);
    uint64_t *a_full = bars, *a_empty = bars + kMaxBar;
    uint64_t *b_full = bars + 2 * kMaxBar, *b_empty = bars + 3 * kMaxBar;
    uint64_t *acc_full = bars + 4 * kMaxBar, *acc_empty = acc_full + 2;
    uint64_t *b_res = acc_empty + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(b_res + 1);
    double *bn_acc = reinterpret_cast<double *>(b_res + 2);  // [4 or 8 epilogue warps][2][bn] (bn_stats)

    const int warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    // TMEM: NB accumulator buffers (double-buffered when they fit) of tpw tiles x acc_cols
    const uint32_t acc_cols = pow2_cols(p.bn);
    const int NB = 2 * p.tpw * (int)acc_cols <= 512 ? 2 : 1;
    const uint32_t buf_cols = p.tpw * acc_cols;
    const uint32_t ncols = NB * buf_cols;

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.a_stages; ++s) {
            mbar_init(&a_full[s], 1);
            mbar_init(&a_empty[s], 1);
        }
        for (int s = 0; s < p.b_stages; ++s) {
            mbar_init(&b_full[s], 1);
            mbar_init(&b_empty[s], p.cluster);  // released by the MMAs of every CTA that reads it
        }
        for (int s = 0; s < 2; ++s) {
            mbar_init(&acc_full[s], 1);
            mbar_init(&acc_empty[s], p.epi2 ? 8 : 4);
        }
        mbar_init(b_res, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc(tmem_slot, ncols);
    tc_fence_before();
    if (p.cluster > 1)
        cluster_sync();  // the partner's barriers exist before any multicast reaches them
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // everything above touched only this CTA's smem / TMEM: with PDL it overlaps
    // the previous kernel's tail; global memory only after its completion
    pdl_wait();
    // Work units: a CTA (cluster == 1) or a CTA pair (cluster == 2: tiles 2k and
    // 2k+1 of the same N tile, each CTA loading half of every weight stage and
    // multicasting it to both; an odd tail tile gives the second CTA a phantom
    // copy of its partner's tile whose results are not stored).
    const int cl = p.cluster;
    const uint32_t cr = cl > 1 ? cluster_ctarank() : 0;
    const int ks = p.ksplit;
    const int unit = blockIdx.x / cl;
    const int split = unit % ks;
    const int w0_ = unit / ks, w_step = (gridDim.x / cl) / ks;
    const int per_o = p.nsamples * p.rect_start[p.nrect];
    const int per_o2 = (per_o + cl - 1) / cl;
    const int total_w = cl > 1 ? p.nout_tiles * per_o2 : p.total_tiles;
    auto item_of = [&](int w, bool &phantom) -> int {
        if (cl == 1) {
            phantom = false;
            return w;
        }
        const int ot = w / per_o2, kk = w - ot * per_o2;
        const int lt = 2 * kk + (int)cr;
        phantom = lt >= per_o;
        return ot * per_o + (phantom ? 2 * kk : lt);
    };
    const int g0 = split * p.ncg / ks, g1 = (split + 1) * p.ncg / ks;

    if (warp == 0) {
        // ============ TMA producer: the whole warp runs the (warp-uniform) ============
        // ============ loop, one elected lane issues the copies             ============
        if (elect_one()) {
            tma_prefetch(&amap);
            tma_prefetch(&bmap);
        }
        int cur_o0 = -1;
        int a_it = 0, b_it = 0;
        for (int w = w0_; w < total_w; w += w_step) {
            bool phantom;
            const TileCoord c = decode(p, item_of(w, phantom));
            if (p.b_resident && c.o0 != cur_o0) {
                // (a resident weight tile never changes for a CTA: nout_tiles == 1)
                if (elect_one()) {
                    mbar_arrive_expect_tx(b_res, p.T * (g1 - g0) * p.bn * p.cg * 2);
                    for (int g = g0; g < g1; ++g)
                        for (int t = 0; t < p.T; ++t)
                            tma_load_2d(sB + ((g - g0) * p.T + t) * p.b_slot_bytes, &bmap, b_res,
                                        t * p.cin_p + g * p.cg, c.o0);
                }
                __syncwarp();
                cur_o0 = c.o0;
            }
            const int h0 = p.s_in * c.i0 + p.origin_h, w0 = p.s_in * c.j0 + p.origin_w;
            for (int g = g0; g < g1; ++g) {
                const int s = a_it % p.a_stages;
                if (a_it >= p.a_stages) mbar_wait(&a_empty[s], ((a_it / p.a_stages) - 1) & 1);
                // 3xTF32 (a_seg > 0): the weights' K segments [w_hi | w_lo | w_hi]
                // pair with the input's [x_hi | x_hi | x_lo]; the input buffer holds
                // [x_hi | x_lo], so channels past the first segment read a_seg lower
                int a_c = g * p.cg;
                if (p.a_seg > 0 && a_c >= p.a_seg) a_c -= p.a_seg;
                if (elect_one()) {
                    uint8_t *dst = sA + s * p.a_stage_bytes;
                    if (p.a_swz) {
                        // one box per column parity: PH rows x PWs cols x cg channels
                        mbar_arrive_expect_tx(&a_full[s], p.s_in * p.PH * p.PWs * p.cg * 2);
                        for (int par = 0; par < p.s_in; ++par)
                            tma_load_4d(dst + par * p.plane_bytes, &amap, &a_full[s], a_c,
                                        w0 + par, h0, c.n);
                    } else {
                        mbar_arrive_expect_tx(&a_full[s], (p.cg / 8) * p.s_in * p.PH * p.PWs * 16);
                        for (int k8 = 0; k8 < p.cg / 8; ++k8)
                            for (int par = 0; par < p.s_in; ++par)
                                tma_load_4d(dst + (k8 * p.s_in + par) * p.plane_bytes, &amap,
                                            &a_full[s], a_c + k8 * 8, w0 + par, h0, c.n);
                    }
                }
                __syncwarp();
                ++a_it;
                if (!p.b_resident) {
                    for (int t = 0; t < p.T; ++t) {
                        const int sb = b_it % p.b_stages;
                        if (b_it >= p.b_stages) mbar_wait(&b_empty[sb], ((b_it / p.b_stages) - 1) & 1);
                        if (elect_one()) {
                            mbar_arrive_expect_tx(&b_full[sb], p.bn * p.cg * 2);
                            if (cl > 1)  // my half of the slot, into both CTAs
                                tma_load_2d_mc(sB + sb * p.b_slot_bytes + cr * (p.bn / 2) * p.cg * 2, &bmap,
                                               &b_full[sb], t * p.cin_p + g * p.cg, c.o0 + (int)cr * (p.bn / 2),
                                               0x3);
                            else
                                tma_load_2d(sB + sb * p.b_slot_bytes, &bmap, &b_full[sb],
                                            t * p.cin_p + g * p.cg, c.o0);
                        }
                        __syncwarp();
                        ++b_it;
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ============ tcgen05.mma issuer: warp-uniform loop, elected lane issues ============
        auto commit = [&](uint64_t *bar) { mma_commit(bar); };
        // Descriptor arithmetic: the start-address field is bits [0,14) in 16-byte
        // units and never carries (smem < 256 KB), so an operand at byte offset
        // `off` from a base descriptor is base + (off >> 4).
        const uint32_t idesc = KIND == 1 ? idesc_tf32(128, p.bn, 0, 0) : idesc_bf16(128, p.bn, 0, 0);
        const uint32_t sA_u = smem_u32(sA), sB_u = smem_u32(sB);
        const uint64_t a_desc0 = p.a_swz ? smem_desc(sA_u, 16, p.a_sbo, swizzle_layout(p.a_swz))
                                                : smem_desc(sA_u, p.s_in * p.plane_bytes, p.a_sbo, 0);
        const uint64_t b_desc0 = smem_desc(sB_u, 16, 8 * p.cg * 2, swizzle_layout(p.cg * 2));
        const uint32_t a_kstep = p.a_kstep16, b_slot16 = p.b_slot_bytes >> 4;
        // second tile of a work item: 16 output rows (= 16 SBO strides) further down
        const uint32_t a_tile16 = (16 * p.a_sbo) >> 4;
        const int nk16 = p.cg / 16;
        int a_it = 0, b_it = 0, acc_it = 0;
        bool res_ready = false;
        for (int w = w0_; w < total_w; w += w_step) {
            if (p.b_resident && !res_ready) {
                mbar_wait(b_res, 0);
                res_ready = true;
            }
            const int acc = acc_it % NB;
            if (acc_it >= NB) mbar_wait(&acc_empty[acc], ((acc_it / NB) - 1) & 1);
            tc_fence_after();
            const uint32_t d_tmem = tmem + acc * buf_cols;
            for (int g = g0; g < g1; ++g) {
                const int s = a_it % p.a_stages;
                mbar_wait(&a_full[s], (a_it / p.a_stages) & 1);
                tc_fence_after();
                const uint64_t a_stage = a_desc0 + ((uint32_t)(s * p.a_stage_bytes) >> 4);
                if (p.b_resident) {
                    if (elect_one()) {
                        uint64_t bd = b_desc0 + (uint32_t)((g - g0) * p.T) * b_slot16;
                        if (!issue_taps_fixed<KIND>(p, nk16, d_tmem, a_stage, bd, a_kstep, b_slot16, idesc, g == g0,
                                                    acc_cols, a_tile16)) {
                        uint64_t arow = a_stage;
                        for (int th = 0; th < p.kh; ++th) {
                            for (int tw = 0; tw < p.kw; ++tw) {
                                const uint64_t ad = arow + (uint32_t)(tw >> p.s_shift) * p.a_col16 +
                                                    (uint32_t)(tw & p.s_shift) * p.a_par16;
                                for (int k16 = 0; k16 < nk16; ++k16)
                                    for (int tt = 0; tt < p.tpw; ++tt)
                                        mma_k<KIND>(d_tmem + tt * acc_cols, ad + k16 * a_kstep + tt * a_tile16,
                                                    bd + 2 * k16, idesc, ((g - g0) | th | tw | k16) != 0);
                                bd += b_slot16;
                            }
                            arow += p.a_row16;
                        }
                        }
                        commit(&a_empty[s]);
                    }
                    __syncwarp();
                } else {
                    // warp-uniform tap counters (no division), descriptors built
                    // outside the elected branch, unrolled slot issue
                    if (p.bn_stats || p.bn > 128) {
                        uint64_t arow = a_stage;
                        int tw = 0, sb = b_it % p.b_stages;
                        uint32_t ph = (b_it / p.b_stages) & 1;
                        for (int t = 0; t < p.T; ++t) {
                            mbar_wait(&b_full[sb], ph);
                            tc_fence_after();
                            const uint64_t ad = arow + (uint32_t)(tw >> p.s_shift) * p.a_col16 +
                                                (uint32_t)(tw & p.s_shift) * p.a_par16;
                            const uint64_t bd = b_desc0 + (uint32_t)sb * b_slot16;
                            const bool first = g == g0 && t == 0;
                            if (elect_one()) {
                                issue_slot_any<KIND>(nk16, p.tpw, d_tmem, ad, bd, a_kstep, a_tile16, acc_cols, idesc,
                                                     first);
                                if (cl > 1)
                                    mma_commit_mc(&b_empty[sb], 0x3);  // the slot is shared by both CTAs
                                else
                                    mma_commit(&b_empty[sb]);
                            }
                            __syncwarp();
                            ++b_it;
                            if (++sb == p.b_stages) sb = 0, ph ^= 1;
                            if (++tw == p.kw) tw = 0, arow += p.a_row16;
                        }
                    } else {
                        // taps in groups of up to kTapGroup (<= b_stages): all their
                        // weight slots awaited, then their MMAs issued back to back --
                        // one wait / fence / warp hand-off per group instead of per
                        // tap keeps the tensor pipe's queue from draining between
                        // taps. The producer runs b_stages slots ahead, so it fills
                        // the later slots of a group without waiting for this
                        // group's commits. Measured in the bench step: 128-wide
                        // tiles' backward-data 688 -> 628 us; the per-tap loop above
                        // stays for the forwards with the fused BN statistics
                        // epilogue (its warps share the MMA warp's scheduler: 729 ->
                        // 787 us grouped) and for 256-wide tiles (stride-2 forwards
                        // 322 -> 369 us grouped).
                        const int tg = p.b_stages < kTapGroup ? p.b_stages : kTapGroup;
                        uint64_t arow = a_stage;
                        int tw = 0, sb = b_it % p.b_stages;
                        uint32_t ph = (b_it / p.b_stages) & 1;
                        for (int t = 0; t < p.T;) {
                            const int n = p.T - t < tg ? p.T - t : tg;
                            int sbs[kTapGroup];
                            uint64_t ads[kTapGroup];
    #pragma unroll
                            for (int j = 0; j < kTapGroup; ++j)
                                if (j < n) {
                                    mbar_wait(&b_full[sb], ph);
                                    sbs[j] = sb;
                                    ads[j] = arow + (uint32_t)(tw >> p.s_shift) * p.a_col16 +
                                             (uint32_t)(tw & p.s_shift) * p.a_par16;
                                    if (++sb == p.b_stages) sb = 0, ph ^= 1;
                                    if (++tw == p.kw) tw = 0, arow += p.a_row16;
                                }
                            tc_fence_after();
                            const bool first = g == g0 && t == 0;
                            if (elect_one()) {
    #pragma unroll
                                for (int j = 0; j < kTapGroup; ++j)
                                    if (j < n) {
                                        issue_slot_any<KIND>(nk16, p.tpw, d_tmem, ads[j],
                                                             b_desc0 + (uint32_t)sbs[j] * b_slot16, a_kstep, a_tile16,
                                                             acc_cols, idesc, first && j == 0);
                                        if (cl > 1)
                                            mma_commit_mc(&b_empty[sbs[j]], 0x3);  // the slot is shared by both CTAs
                                        else
                                            mma_commit(&b_empty[sbs[j]]);
                                    }
                            }
                            __syncwarp();
                            b_it += n;
                            t += n;
                        }
                    }
                    if (elect_one()) commit(&a_empty[s]);
                    __syncwarp();
                }
                ++a_it;
            }
            if (elect_one()) commit(&acc_full[acc]);
            __syncwarp();
            ++acc_it;
        }
    } else if (warp < 6 || (p.epi2 && warp > 6)) {  // (warp 6 idles)
        // ========================= epilogue =========================
        const int eq = warp & 3;  // TMEM lane quarter this warp may access
        const int m = eq * 32 + lane;
        const int ti = m >> p.tw_log2, tj = m & ((1 << p.tw_log2) - 1);
        const int egrp = warp >= 7;                      // chunk half of this warp's group
        const int ewarp = warp < 6 ? warp - 2 : warp - 3;  // 0..3 group 0, 4..7 group 1
        double *my_acc = bn_acc + ewarp * 2 * p.bn;
        if (p.bn_stats)
            for (int i = lane; i < 2 * p.bn; i += 32) my_acc[i] = 0.0;
        __syncwarp();
        // BN partial of this CTA: bn_part[blockIdx.x][2][nout_p]. Work items
        // run in ascending N-tile order, so a CTA's items form contiguous
        // segments of one N tile each; a segment's sums (the 4 / 8 warps in a
        // fixed order) are stored when the N tile changes and at the end;
        // channels of N tiles this CTA never ran stay zero.
        const int n_epi = p.epi2 ? 8 : 4;
        double *bn_dst = p.bn_part + (long long)blockIdx.x * 2 * p.nout_p;
        auto epi_bar = [&]() {
            if (p.epi2)
                asm volatile("bar.sync 1, 256;" ::: "memory");
            else
                asm volatile("bar.sync 1, 128;" ::: "memory");
        };
        auto seg_flush = [&](const int o0) {
            epi_bar();
            for (int i = ewarp * 32 + lane; i < 2 * p.bn; i += 32 * n_epi) {
                const int k = i / p.bn, ch = i - k * p.bn;
                if (o0 + ch < p.nout_p) {
                    double t = 0.0;
                    for (int w4 = 0; w4 < n_epi; ++w4) t += bn_acc[w4 * 2 * p.bn + k * p.bn + ch];
                    bn_dst[k * p.nout_p + o0 + ch] = t;
                }
            }
            epi_bar();
        };
        if (p.bn_stats && p.nout_tiles > 1)
            for (int i = ewarp * 32 + lane; i < 2 * p.nout_p; i += 32 * n_epi) bn_dst[i] = 0.0;
        int seg_o0 = -1;
        if (p.bn_stats == 2) {
            // N tile <= 64 channels: every thread always holds the same <= 64
            // channels, so it accumulates x and x^2 in registers across tiles
            // (fp32, sequential) and the warp reduction runs once per 16 items
            // (error depth <= 2 * 16 + 5) instead of per tile
            float rs[64], rq[64];
#pragma unroll
            for (int k = 0; k < 64; ++k) rs[k] = rq[k] = 0.f;
            auto flush = [&]() {
#pragma unroll
                for (int c16 = 0; c16 < 4; ++c16)
                    if (c16 < p.bn / 16) {
                        float a[16], q[16];
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            a[e] = rs[c16 * 16 + e], q[e] = rq[c16 * 16 + e];
                            rs[c16 * 16 + e] = rq[c16 * 16 + e] = 0.f;
                        }
                        warp_chunk_reduce(a, q, lane);
                        const float a_o = __shfl_xor_sync(0xffffffffu, a[0], 1);
                        const float q_o = __shfl_xor_sync(0xffffffffu, q[0], 1);
                        if ((lane & 1) == 0) {
                            const int ch = c16 * 16 + ((lane >> 1) & 15);
                            my_acc[ch] += (double)(a[0] + a_o);
                            my_acc[p.bn + ch] += (double)(q[0] + q_o);
                        }
                    }
            };
            int acc_it = 0, since = 0;
            for (int w = w0_; w < total_w; w += w_step) {
                bool phantom;
                const TileCoord c = decode(p, item_of(w, phantom));
                const int acc = acc_it % NB;
                mbar_wait(&acc_full[acc], (acc_it / NB) & 1);
                tc_fence_after();
                for (int tt = 0; tt < p.tpw; ++tt) {
                    const int i = c.i0 + tt * 16 + ti, j = c.j0 + tj;
                    const bool valid = !phantom && i < p.rect[c.r].h0 + p.rect[c.r].nh &&
                                       j < p.rect[c.r].w0 + p.rect[c.r].nw;
                    __nv_bfloat16 *orow = p.out + (long long)c.n * p.out_sn +
                                          (long long)(p.out_h0 + p.out_dh * i) * p.out_sh +
                                          (long long)(p.out_w0 + p.out_dw * j) * p.out_sw + c.o0;
                    const uint32_t t_lane = tmem + acc * buf_cols + tt * acc_cols + ((uint32_t)(eq * 32) << 16);
#pragma unroll
                    for (int c16 = 0; c16 < 4; ++c16)
                        if (c16 < p.bn / 16) {
                            uint32_t v[16];
                            tmem_ld16(t_lane + c16 * 16, v);
                            tmem_ld_wait();
                            const bool st_ok = valid && c.o0 + c16 * 16 < p.nout_p;
                            uint32_t pk[8];
#pragma unroll
                            for (int e = 0; e < 8; ++e) pk[e] = pack2(v[2 * e], v[2 * e + 1]);
                            if (st_ok) st_global_v8(orow + c16 * 16, pk);
#pragma unroll
                            for (int e = 0; e < 16; ++e) {
                                const float xv = st_ok ? __uint_as_float((e & 1) ? (pk[e >> 1] & 0xffff0000u)
                                                                                 : (pk[e >> 1] << 16))
                                                       : 0.f;
                                rs[c16 * 16 + e] += xv;
                                rq[c16 * 16 + e] = fmaf(xv, xv, rq[c16 * 16 + e]);  // x^2 exact
                            }
                        }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[acc]);
                ++acc_it;
                if (++since == 16) flush(), since = 0;
            }
            flush();
        } else {
        int acc_it = 0;
        for (int w = w0_; w < total_w; w += w_step) {
            bool phantom;
            const TileCoord c = decode(p, item_of(w, phantom));
            if (p.bn_stats && c.o0 != seg_o0) {
                if (seg_o0 >= 0) {
                    seg_flush(seg_o0);
                    for (int i = lane; i < 2 * p.bn; i += 32) my_acc[i] = 0.0;
                    __syncwarp();
                }
                seg_o0 = c.o0;
            }
            const int acc = acc_it % NB;
            mbar_wait(&acc_full[acc], (acc_it / NB) & 1);
            tc_fence_after();
            for (int tt = 0; tt < p.tpw; ++tt) {
            const int i = c.i0 + tt * 16 + ti, j = c.j0 + tj;
            const bool valid = !phantom && i < p.rect[c.r].h0 + p.rect[c.r].nh &&
                               j < p.rect[c.r].w0 + p.rect[c.r].nw;
            __nv_bfloat16 *orow = p.out + (long long)c.n * p.out_sn +
                                  (long long)(p.out_h0 + p.out_dh * i) * p.out_sh +
                                  (long long)(p.out_w0 + p.out_dw * j) * p.out_sw + c.o0;
            const uint32_t t_lane = tmem + acc * buf_cols + tt * acc_cols + ((uint32_t)(eq * 32) << 16);
            float *wrow = ks > 1 ? p.ws + (long long)split * p.nsamples * p.ws_h * p.ws_w * p.nout_p +
                                       (((long long)c.n * p.ws_h + i) * p.ws_w + j) * p.nout_p + c.o0
                                 : nullptr;
            // TMEM loads double-buffered: chunk c16 + 1 is in flight while
            // chunk c16 is packed and stored (tcgen05.wait::ld covers both)
            auto body = [&](const uint32_t (&v)[16], const int c16) {
                if (ks > 1) {
                    if (valid && c.o0 + c16 * 16 < p.nout_p) {
                        float4 *dst = reinterpret_cast<float4 *>(wrow + c16 * 16);
                        // (fp32 outputs pad channels to 8: a chunk may hold one valid half)
                        const int nq = c.o0 + c16 * 16 + 8 < p.nout_p ? 4 : 2;
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            if (q < nq)
                            dst[q] = make_float4(__uint_as_float(v[4 * q]), __uint_as_float(v[4 * q + 1]),
                                                 __uint_as_float(v[4 * q + 2]), __uint_as_float(v[4 * q + 3]));
                    }
                } else if (p.out_f32) {
                    // fp32 output (3xTF32 path, channel-parallel partials): 16
                    // columns = two 32-byte halves, the second only when the
                    // (8-padded) channel count reaches it
                    float *of = f32_out(p, c.n, i, j, c.o0 + c16 * 16);
                    if (valid) {
                        if (c.o0 + c16 * 16 < p.nout_p) st_global_v8(of, *reinterpret_cast<const uint32_t(*)[8]>(&v[0]));
                        if (c.o0 + c16 * 16 + 8 < p.nout_p)
                            st_global_v8(of + 8, *reinterpret_cast<const uint32_t(*)[8]>(&v[8]));
                    }
                } else {
                    const bool st_ok = valid && c.o0 + c16 * 16 < p.nout_p;
                    uint32_t pk[8];
#pragma unroll
                    for (int e = 0; e < 8; ++e) pk[e] = pack2(v[2 * e], v[2 * e + 1]);
                    if (st_ok) {
                        if (p.subpix) {  // this 16-channel chunk belongs to one stride phase
                            const int col = c.o0 + c16 * 16, ph = col / p.sub_cp, ch = col - ph * p.sub_cp;
                            const int row = p.out_h0 + p.out_dh * i + (ph >> 1);
                            const int cw = p.out_w0 + p.out_dw * j + (ph & 1);
                            if (row >= 0 && row < p.out_hmax && cw >= 0 && cw < p.out_wmax)
                                st_global_v8(p.out + (long long)c.n * p.out_sn + (long long)row * p.out_sh +
                                                 (long long)cw * p.out_sw + ch,
                                             pk);
                        } else {
                            st_global_v8(orow + c16 * 16, pk);  // a whole 32-byte sector
                        }
                    }
                    if (p.bn_stats) {
                        // statistics of the stored bf16 values: an fp32 pairwise
                        // transpose-reduce over the warp's 32 pixels (fixed order;
                        // |error| <= 5 * 2^-24 * sum|x|), then fp64
                        float a[16], q[16];
#pragma unroll
                        for (int e = 0; e < 16; ++e) {
                            const float xv = st_ok ? __uint_as_float((e & 1) ? (pk[e >> 1] & 0xffff0000u)
                                                                             : (pk[e >> 1] << 16))
                                                   : 0.f;
                            a[e] = xv;
                            q[e] = xv * xv;  // exact: 8-bit significand
                        }
#pragma unroll
                        for (int w = 8; w >= 1; w >>= 1) {
                            const bool up = (lane & (2 * w)) != 0;
#pragma unroll
                            for (int j = 0; j < w; ++j) {
                                const float sa = up ? a[j] : a[j + w], ka = up ? a[j + w] : a[j];
                                const float sq = up ? q[j] : q[j + w], kq = up ? q[j + w] : q[j];
                                a[j] = ka + __shfl_xor_sync(0xffffffffu, sa, 2 * w);
                                q[j] = kq + __shfl_xor_sync(0xffffffffu, sq, 2 * w);
                            }
                        }
                        // lanes 2k and 2k+1 hold channel k's halves
                        const float a_o = __shfl_xor_sync(0xffffffffu, a[0], 1);
                        const float q_o = __shfl_xor_sync(0xffffffffu, q[0], 1);
                        if ((lane & 1) == 0) {
                            const int ch = c16 * 16 + ((lane >> 1) & 15);  // within this N tile
                            my_acc[ch] += (double)(a[0] + a_o);
                            my_acc[p.bn + ch] += (double)(q[0] + q_o);
                        }
                    }
                }
            };
            const int nc16 = p.bn / 16;
            const int c_lo = p.epi2 && egrp ? (nc16 + 1) / 2 : 0;
            const int c_hi = p.epi2 && !egrp ? (nc16 + 1) / 2 : nc16;
            uint32_t va[16], vb[16];
            if (c_lo < c_hi) {
                tmem_ld16(t_lane + c_lo * 16, va);
                tmem_ld_wait();
            }
            for (int c16 = c_lo; c16 < c_hi; c16 += 2) {
                if (c16 + 1 < c_hi) tmem_ld16(t_lane + (c16 + 1) * 16, vb);
                body(va, c16);
                tmem_ld_wait();
                if (c16 + 1 < c_hi) {
                    if (c16 + 2 < c_hi) tmem_ld16(t_lane + (c16 + 2) * 16, va);
                    body(vb, c16 + 1);
                    tmem_ld_wait();
                }
            }
            }  // tt
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[acc]);
            ++acc_it;
        }
        }  // (bn_stats != 2)
        if (p.bn_stats) seg_flush(seg_o0 < 0 ? 0 : seg_o0);  // the last (or only) segment
    }
    tc_fence_before();
    if (p.cluster > 1)
        cluster_sync();  // no CTA leaves while its partner may still multicast into it
    else
        __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, ncols);
}

// ---------------------------------------------------------------------------
size_t conv_v2_smem_bytes(const ConvV2Params &p) {
    const size_t b = p.b_resident ? (size_t)p.T * (p.ncg / p.ksplit) * p.b_slot_bytes
                                  : (size_t)p.b_stages * p.b_slot_bytes;
    return 1024 + b + (size_t)p.a_stages * p.a_stage_bytes + (4 * kMaxBar + 5) * 8 + 16 +
           (p.bn_stats ? (size_t)(p.epi2 ? 8 : 4) * 2 * p.bn * sizeof(double) : 0);
}

// Pair tiles only when the launch has this many tpw = 1 work items
// (measured: pairing wins 1.5x on 128^2..512^2 layers, loses on 64^2/32^2).
constexpr int kPairMinItems = 200;

bool conv_v2_configure(ConvV2Params &p, int smem_limit) {
    int kh = 1, kw = 1;
    for (int t = 0; t < p.T; ++t) {
        kh = std::max(kh, (int)p.tap_h[t] + 1);
        kw = std::max(kw, (int)p.tap_w[t] + 1);
    }
    const int cg_nat = p.cin_p % 64 == 0 ? 64 : p.cin_p % 32 == 0 ? 32 : 16;
    p.cg = p.cg > 0 && p.cg < cg_nat ? p.cg : cg_nat;  // a caller may ask for narrower stages
    p.ncg = p.cin_p / p.cg;
    const int TW = 1 << p.tw_log2, TH = 128 >> p.tw_log2;
    if (TW != 8 && !(TW == 128 && p.s_in == 1)) return false;
    if (p.tpw < 1) p.tpw = 1;
    if (TW != 8) p.tpw = 1;
    p.PH = p.s_in * (TH * p.tpw - 1) + kh;
    const int pitch = TW + (kw - 1) / p.s_in;  // pixels per smem row
    if (pitch * p.s_in <= 256) {
        // swizzled rows of cg channels (32/64/128-byte swizzle), one plane per
        // column parity (TMA element stride = s_in). The swizzle is a function
        // of the absolute smem address (measured), so a tap shift only moves
        // the start address and the row pitch can be exactly the TW + (kw-1)/s
        // pixels a tile needs; planes start on 1 KB boundaries.
        p.a_swz = p.cg * 2;
        p.PWs = pitch;
        p.plane_bytes = (int)round_up((int64_t)p.PH * p.PWs * p.cg * 2, 1024);
        p.a_stage_bytes = p.s_in * p.plane_bytes;
        p.a_sbo = TW == 8 ? p.s_in * p.PWs * p.cg * 2 : 8 * p.cg * 2;
    } else {
        p.a_swz = 0;
        p.PWs = TW + (kw - 1) / p.s_in;
        if (p.PWs * p.s_in > 256 || p.PH > 256) return false;
        p.plane_bytes = (int)round_up((int64_t)p.PH * p.PWs * 16, 128);
        p.a_stage_bytes = (p.cg / 8) * p.s_in * p.plane_bytes;
        p.a_sbo = TW == 8 ? p.s_in * p.PWs * 16 : 8 * 16;
    }
    p.kh = kh;
    p.kw = kw;
    for (int t = 0; t < p.T; ++t)  // the tap list must be the row-major (th, tw) grid
        if (p.tap_h[t] != t / kw || p.tap_w[t] != t % kw || p.T != kh * kw) return false;
    p.s_shift = p.s_in == 2 ? 1 : 0;
    if (p.a_swz) {
        p.a_row16 = (p.PWs * p.cg * 2) >> 4;
        p.a_col16 = (p.cg * 2) >> 4;
        p.a_par16 = p.plane_bytes >> 4;
        p.a_kstep16 = 32 >> 4;  // next 16 channels inside the swizzled row
    } else {
        p.a_row16 = (p.PWs * 16) >> 4;
        p.a_col16 = 1;
        p.a_par16 = p.plane_bytes >> 4;
        p.a_kstep16 = (2 * p.s_in * p.plane_bytes) >> 4;
    }
    p.b_slot_bytes = (int)round_up((int64_t)p.bn * p.cg * 2, 1024);
    const int fixed = 1024 + (4 * kMaxBar + 5) * 8 + 16 + (p.bn_stats ? 4 * 2 * p.bn * 8 : 0);
    if (p.ksplit < 1 || p.ncg % p.ksplit) return false;
    const int resident_b = p.T * (p.ncg / p.ksplit) * p.b_slot_bytes;
    // prefer resident weights with >= 2 A stages
    if (p.nout_tiles == 1 && resident_b + 2 * p.a_stage_bytes + fixed <= smem_limit &&
        resident_b <= 160 * 1024) {
        p.b_resident = 1;
        p.b_stages = 0;
        p.a_stages = std::min(4, (smem_limit - fixed - resident_b) / p.a_stage_bytes);
        // resident weights: a work item of two stacked tiles halves the per-item
        // overheads (barriers, accumulator hand-off) and the A halo rows
        if (p.tpw == 1 && TW == 8 && p.work_hint >= kPairMinItems) {
            ConvV2Params q = p;
            q.tpw = 2;
            if (conv_v2_configure(q, smem_limit) && q.tpw == 2 && q.b_resident && q.a_stages >= 2) p = q;
        }
    } else {
        p.b_resident = 0;
        p.a_stages = 2;
        p.b_stages = std::min(8, (smem_limit - fixed - p.a_stages * p.a_stage_bytes) / p.b_slot_bytes);
        if (p.b_stages < 2) {
            p.a_stages = 1;  // (cannot happen for cg <= 64, bn <= 256)
            p.b_stages = std::min(8, (smem_limit - fixed - p.a_stage_bytes) / p.b_slot_bytes);
        }
        if (p.b_stages < 2) return false;
        // streamed weights: let a work item cover two stacked 16 x 8 tiles that
        // share every weight stage (halves the L2 weight traffic per FLOP)
        if (p.tpw == 1 && TW == 8 && p.work_hint >= kPairMinItems) {
            ConvV2Params q = p;
            q.tpw = 2;
            if (conv_v2_configure(q, smem_limit) && q.tpw == 2 && q.a_stages >= 2 && q.b_stages >= 2) {
                p = q;
            } else if (p.cg == 64 && p.s_in == 2 && p.allow_cg32) {
                // stride 2: a 32-row stacked tile pair is too tall for 64-channel
                // stages; 32-channel stages make it fit (same weight reuse)
                q.cg = 32;
                if (conv_v2_configure(q, smem_limit) && q.tpw == 2 && q.a_stages >= 2 && q.b_stages >= 2) p = q;
            }
        }
    }
    // streamed weights: CTA pairs multicast each weight stage (half each), which
    // halves the L2 -> SM weight traffic without reducing the number of CTAs
    // (CTA pairs with cta_group::2 were measured slower in the step with cold
    // inputs and resident weights -- profiles/r2_cg2_resident_ab.txt -- and removed)
    p.cluster = (!p.b_resident && p.bn % 32 == 0 && p.kind == 0) ? 2 : 1;
    return p.a_stages >= 1 && p.a_stages <= kMaxBar && p.b_stages <= kMaxBar;
}

// out[pixel][o] = bf16( sum_{s in order} ws[s][pixel][o] ) over the launch's rects.
__global__ void conv_v2_reduce_kernel(const __grid_constant__ ConvV2Params p) {
    pdl_wait();  // (launch.cuh: PDL)
    const int vecs = p.nout_p / 8;
    long long npix_rects = 0;
    for (int r = 0; r < p.nrect; ++r) npix_rects += (long long)p.rect[r].nh * p.rect[r].nw;
    const long long work = npix_rects * p.nsamples * vecs;
    const long long split_stride = (long long)p.nsamples * p.ws_h * p.ws_w * p.nout_p;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < work;
         idx += (long long)gridDim.x * blockDim.x) {
        const int v = (int)(idx % vecs);
        long long pix = idx / vecs;
        const int n = (int)(pix / npix_rects);
        long long rp = pix - (long long)n * npix_rects;
        int r = 0;
        while (rp >= (long long)p.rect[r].nh * p.rect[r].nw) {
            rp -= (long long)p.rect[r].nh * p.rect[r].nw;
            ++r;
        }
        const int i = p.rect[r].h0 + (int)(rp / p.rect[r].nw), j = p.rect[r].w0 + (int)(rp % p.rect[r].nw);
        const float *src = p.ws + (((long long)n * p.ws_h + i) * p.ws_w + j) * p.nout_p + v * 8;
        float4 a = reinterpret_cast<const float4 *>(src)[0], b = reinterpret_cast<const float4 *>(src)[1];
        for (int s = 1; s < p.ksplit; ++s) {
            const float4 *q = reinterpret_cast<const float4 *>(src + s * split_stride);
            const float4 c = q[0], d = q[1];
            a.x += c.x, a.y += c.y, a.z += c.z, a.w += c.w;
            b.x += d.x, b.y += d.y, b.z += d.z, b.w += d.w;
        }
        if (p.out_f32) {
            float4 *of = reinterpret_cast<float4 *>(f32_out(p, n, i, j, v * 8));
            of[0] = a, of[1] = b;
            continue;
        }
        uint4 o;
        o.x = pack2(__float_as_uint(a.x), __float_as_uint(a.y));
        o.y = pack2(__float_as_uint(a.z), __float_as_uint(a.w));
        o.z = pack2(__float_as_uint(b.x), __float_as_uint(b.y));
        o.w = pack2(__float_as_uint(b.z), __float_as_uint(b.w));
        *reinterpret_cast<uint4 *>(p.out + (long long)n * p.out_sn + (long long)(p.out_h0 + p.out_dh * i) * p.out_sh +
                                   (long long)(p.out_w0 + p.out_dw * j) * p.out_sw + v * 8) = o;
    }
}

void launch_conv_v2_reduce(const ConvV2Params &p, cudaStream_t st) {
    long long npix = 0;
    for (int r = 0; r < p.nrect; ++r) npix += (long long)p.rect[r].nh * p.rect[r].nw;
    const long long work = npix * p.nsamples * (p.nout_p / 8);
    if (work == 0) return;
    const int blocks = (int)std::min<long long>((work + 255) / 256, device_sm_count() * 8);
    launch_k(conv_v2_reduce_kernel, dim3(blocks), dim3(256), 0, st, 1, "conv_v2 reduce", p);
}

int device_sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

int launch_conv_v2(const CUtensorMap &amap, const CUtensorMap &bmap, const ConvV2Params &p_in,
                   cudaStream_t st) {
    if (p_in.total_tiles == 0) return 0;
    ConvV2Params p = p_in;
    // second epilogue warp group, where the epilogue paces the tile loop
    // (measured A/B, N = 8 mesh layers, cold L2): the sub-pixel backward-data
    // (4 phases per tile, short K: conv1_1 1183 -> 783 us) and 256-wide N
    // tiles (conv3_2 fwd 579 -> 518 us, 512-ch 32^2 47.5 -> 45.3 us); it
    // slows the 64/128-wide stride-1/2 tiles (conv1_2 bwd-data 633 -> 680 us,
    // conv2_1 fwd 322 -> 343 us). Not for the register-accumulated BN path
    // (bn_stats == 2) and only while the wider BN scratch still fits.
    p.epi2 = 0;
    if (p.bn_stats != 2 && (p.subpix || p.bn >= 256)) {
        p.epi2 = 1;
        if (conv_v2_smem_bytes(p) > (size_t)kV2SmemLimit) p.epi2 = 0;
    }
    static std::once_flag once;
    std::call_once(once, [] {
        cudaFuncSetAttribute(conv_v2_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kV2SmemLimit);
        cudaFuncSetAttribute(conv_v2_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, kV2SmemLimit);
    });
    if (p.cluster > 1) {
        // persistent CTA pairs: as many as can be co-resident (GPCs need not hold
        // an even number of free SMs), a multiple of the split-K factor
        const size_t smem = tmem_kernel_smem(conv_v2_smem_bytes(p));
        DC_REQUIRE(p.kind == 0, DC_ERR_ARG, "conv_v2: tf32 runs without CTA pairs");
        auto kern = conv_v2_kernel<0>;
        const size_t key = smem;
        static std::map<size_t, int> max_clusters;
        if (!max_clusters.count(key)) {
            cudaLaunchConfig_t cfg{};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 2, at[0].val.clusterDim.y = 1, at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(2 * (device_sm_count() / 2));
            cfg.blockDim = dim3(kV2Threads);
            cfg.dynamicSmemBytes = smem;
            cfg.attrs = at, cfg.numAttrs = 1;
            int n = 0;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
            DC_REQUIRE(e == cudaSuccess && n > 0, DC_ERR_CUDA, "cluster occupancy: %s", cudaGetErrorString(e));
            max_clusters[key] = n;
        }
        const int per_o = p.nsamples * p.rect_start[p.nrect];
        const int total_w = p.nout_tiles * ((per_o + 1) / 2);
        const int cap_units = p.max_ctas > 0 ? std::min(max_clusters[key], p.max_ctas / 2) : max_clusters[key];
        const int units = p.ksplit * std::max(1, std::min(total_w, cap_units / p.ksplit));
        launch_k(kern, dim3(2 * units), dim3(kV2Threads), smem, st, 2, "conv_v2 (pairs)", amap, bmap, p);
        return 2 * units;
    }
    const int sms = p.max_ctas > 0 ? std::min(p.max_ctas, device_sm_count()) : device_sm_count();
    const int grid = p.ksplit * std::max(1, std::min(p.total_tiles, sms / p.ksplit));
    if (g_dry_run) return grid;
    launch_k(p.kind == 1 ? conv_v2_kernel<1> : conv_v2_kernel<0>, dim3(grid), dim3(kV2Threads),
             tmem_kernel_smem(conv_v2_smem_bytes(p)), st, 1, p.kind == 1 ? "conv_v2 (tf32)" : "conv_v2", amap, bmap,
             p);
    return grid;
}


// Loads this file's kernels now (CUDA lazy loading would otherwise load a
// kernel at its first launch, which waits for the device: with the spinning
// halo / BN protocol kernels of a loopback group in flight, that wait never
// ends).
void preload_conv_v2() {
    cudaFuncAttributes a;
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(conv_v2_kernel<0>));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(conv_v2_kernel<1>));
    cudaFuncGetAttributes(&a, reinterpret_cast<const void *>(conv_v2_reduce_kernel));
}

}  // namespace dc

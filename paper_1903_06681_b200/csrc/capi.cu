// capi.cu -- L5: the C ABI of libdconv (include/dconv.h).
//
// Orchestrates one layer of spatially / hybrid-partitioned convolution on
// this rank: plan (L1, plan.cpp), sm_100a kernels (L2, conv_tc.cu, halo.cu),
// communication (L3: NCCL + CUDA-IPC peer mappings), model (L4,
// perfmodel.cpp). Stream structure:
//   forward       comm stream: x halo exchange  ||  caller stream: interior
//                 tiles; then boundary tiles after the exchange event.
//   backward      comm stream: dy halo exchange ||  caller stream: filter
//                 gradient (needs no dy halo); then data
//                 gradient, with the dW allreduce on the comm stream
//                 concurrently.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <array>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.hpp"
#include "conv_tc.cuh"
#include "conv_v2.cuh"
#include "halo.cuh"
#include "launch.cuh"
#include "wgrad_v2.cuh"
#include "tf32.cuh"
#include "bn.cuh"
#include "redist.cuh"
#include "cfpar.cuh"
#include "pool.cuh"
#include "subsample.cuh"
#include "plan.hpp"

namespace dc {
thread_local uint64_t g_launches = 0;
thread_local bool g_no_pdl = false;
thread_local bool g_dry_run = false;
static thread_local std::string g_err;
void set_last_error(const std::string &m) { g_err = m; }

double model_layer_cost(const ConvGeom &g, Grid d, bool include_allreduce);
void preload_conv_tc();
void preload_conv_v2();
void preload_halo();
void preload_tf32();
void preload_wgrad_v2();
void preload_bn();
void preload_redist();
void preload_cfpar();
void preload_pool();
void preload_subsample();
// Every kernel of the library loaded into this context (see preload_*):
// once, at communicator creation.
void preload_kernels() {
    static std::once_flag once;
    std::call_once(once, [] {
        preload_conv_tc();
        preload_conv_v2();
        preload_halo();
        preload_tf32();
        preload_wgrad_v2();
        preload_bn();
        preload_redist();
        preload_cfpar();
        preload_pool();
        preload_subsample();
    });
}
bool model_choose(const ConvGeom &g, int world, Grid &best, double &best_t, Grid fix);
}  // namespace dc

using namespace dc;

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t _e = (x);                                                              \
        DC_REQUIRE(_e == cudaSuccess, DC_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(_e));  \
    } while (0)
#define NK(x)                                                                              \
    do {                                                                                   \
        ncclResult_t _r = (x);                                                             \
        DC_REQUIRE(_r == ncclSuccess, DC_ERR_COMM, "%s: %s", #x, ncclGetErrorString(_r));  \
    } while (0)

struct dc_plan_s;
struct dc_redist_s;
struct dc_cplan_s;
struct dc_pool_s;

namespace dc {
// Loopback group: `world` virtual ranks of one process on ONE device
// (dc_comm_create_local). Every cross-rank pointer (halo flags, margined
// buffers, BN mailboxes) is a plain device pointer of the same process,
// resolved through this registry, so the P2P protocols run unchanged on one
// GPU (tests; the NCCL transports need real ranks).
struct LocalGroup {
    int world = 1;
    std::mutex mu;
    std::map<std::pair<int, int>, dc_plan_s *> plans;  // (plan sequence number, rank)
    std::map<int, std::array<int, 3>> grids;            // sequence number -> grid of its first rank
    std::map<std::pair<int, int>, dc_redist_s *> redists;  // (redistribution sequence number, rank)
    std::map<std::pair<int, int>, dc_cplan_s *> cplans;    // (channel plan sequence number, rank)
};
}  // namespace dc

struct dc_comm_s {
    int rank = 0, world = 1, device = 0;
    ncclComm_t nccl = nullptr;
    // dW allreduces queued with DC_ALLREDUCE_ASYNC: their own communicator
    // (so they never serialise behind / ahead of halo or BN traffic) and stream
    ncclComm_t grad_nccl = nullptr;
    cudaStream_t s_grad = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    bool grad_pending = false;  // allreduces queued since the last dc_comm_sync
    // DC_ALLREDUCE_ASYNC bucket (the dW allreduces overlap the
    // later layers' work, one at a time): layers' dW buffers collected until
    // bucket_cap bytes, then issued as ONE grouped NCCL call on s_grad
    std::vector<std::pair<float *, size_t>> bucket;
    size_t bucket_bytes = 0, bucket_cap = 4u << 20;
    std::shared_ptr<LocalGroup> group;  // loopback group (no NCCL), or null
    int plan_seq = 0;                   // plans created on this communicator (loopback registry key)
    int redist_seq = 0;                 // redistributions created on it (likewise)
    int cplan_seq = 0;                  // channel / filter parallel plans (likewise)
    // loopback: the virtual rank's two streams (its compute stream, handed to
    // the caller by dc_comm_stream, and the side stream every plan of the rank
    // uses for exchanges / boundary tiles), created back to back for all ranks
    // so that no two of them share a hardware queue (see dc_comm_create_local)
    cudaStream_t s_main = nullptr, s_side = nullptr;
    // real ranks: the side-stream set every plan of this communicator shares
    // (exchanges / boundary tiles on s_side, backward-data stride phases on
    // s_ph, host imports on s_copy) -- a handful of streams per process
    // however many layers, so that streams never alias onto one hardware
    // queue (a spinning protocol kernel ahead of unrelated work in an aliased
    // queue would stall that work; peers waiting for it would never finish)
    cudaStream_t s_ph[4] = {nullptr, nullptr, nullptr, nullptr};
    cudaStream_t s_copy = nullptr;
};

namespace {

struct BufState {  // a margined buffer (X or DY) known to the plan
    void *ptr = nullptr;
    size_t bytes = 0;
    bool owned = false;
    std::map<int, void *> peer;  // peer rank -> that rank's buffer mapped here
    uint32_t *dev_epoch = nullptr;  // P2P protocol epoch {epoch, blocks done} (device)
    void *stage = nullptr;       // NCCL baseline staging: [send | recv]
    size_t stage_bytes = 0;
};

enum { FLAG_READY = 0, FLAG_DATA = 1 };

}  // namespace

// Split-K basis (reading R25): the conv kernels' split-K factor
// over channel groups -- the only choice that changes how an output element
// is summed -- is picked for the GLOBAL layer (undivided: basis 1), whatever
// the plan's grid, so every partition and the 1-GPU plan of the same layer sum
// each y / dx element in the same order (north_star: partitioned output
// bit-identical to 1 GPU). (Measured: a basis of 8 -- splits sized for the
// 8-way shards -- cost the 1-GPU mesh2k_n8 step 2.5 ms on its 64^2 / 32^2
// 512-channel layers; an in-kernel split-order reduction chained the splits'
// epilogues and was slower still.)
constexpr int kSplitKBasis = 1;

struct dc_plan_s {
    RankPlan rp;
    dc_comm_s *comm = nullptr;
    bool is_virtual = false;
    ncclComm_t bn_comm = nullptr;
    bool bn_comm_owned = false;
    int bn_group = 1;
    cudaStream_t s_comm = nullptr;
    bool s_comm_shared = false;  // s_comm, s_ph, s_copy are the communicator's (not destroyed here)
    cudaStream_t s_ph[4] = {nullptr, nullptr, nullptr, nullptr};  // stride-phase streams (bwd-data)
    cudaEvent_t ev_ph[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    BufState buf[2];                 // 0: X, 1: DY
    BufState dense[2];               // dc_buffer_alloc'd dense 0: Y, 1: DX (redistribution targets)
    uint32_t *flags = nullptr;       // [2 buf][2 kind][world]
    std::map<int, uint32_t *> peer_flags;
    uint32_t *dev_epochs = nullptr;  // [2 buf][epoch, blocks done] (local)
    float *wsplit = nullptr;         // 3xTF32 forward weights [F][T][hi | lo | hi]
    void *xsub = nullptr;            // 1x1 stride-2 forward: the gathered input pixels
    size_t xsub_bytes = 0;
    size_t wsplit_bytes = 0;
    __nv_bfloat16 *wt = nullptr;     // backward-data weights, all phases (fp32 plans: fp32 words)
    size_t wt_bytes = 0;
    float *ws = nullptr;             // split-K workspace (backward-filter)
    size_t ws2_bytes = 0;
    float *ws2 = nullptr;            // split-K workspace (forward / backward-data)
    size_t ws_bytes = 0;
    double *bn_part = nullptr;
    size_t bn_part_bytes = 0;
    double *bn_sums = nullptr;
    float *bn_coef = nullptr;        // BN apply / backward coefficients [4][Fp]
    size_t bn_coef_bytes = 0;
    double *bnb_part = nullptr;      // BN backward partials [blocks][2][Fp]
    size_t bnb_part_bytes = 0;
    double *bn_scratch = nullptr;    // (mean / var outputs the backward's group sum does not need)
    size_t bn_scratch_bytes = 0;
    double *bn_fpart = nullptr;      // fused BN partials of the last DC_BN_STATS forward
    size_t bn_fpart_bytes = 0;
    const void *bn_fused_y = nullptr;  // its y (stats of any other tensor: the staged pass, bn.cu)
    int bn_fused_slots = 0;
    uint64_t fwd_epoch = 0;          // forwards run by this plan
    uint64_t bn_fused_epoch = 0;     // the forward whose partials bn_fpart holds (0: none)
    // P2P BN statistics mailbox of THIS plan's BN group (halo.cuh: BnP2P):
    // [flags, 256 B][2 parities][bn_group][2 Fp doubles]; per plan, so every
    // member takes part in every epoch (a member is at most one epoch ahead)
    uint8_t *bn_mail = nullptr;
    uint32_t *bn_epoch = nullptr;
    std::vector<uint8_t *> bn_peer_mail;  // member k's mailbox (mine at my index)
    bool bn_p2p = false;
    int seq = -1;                    // creation index on the communicator (loopback registry key)
    // dc_tensor_import staging: host -> device copies and the import kernel
    // on an internal copy stream (DC_IMPORT_ASYNC), joined by the next call
    // that reads the buffer
    cudaStream_t s_copy = nullptr;
    cudaEvent_t ev_copy_in[2] = {nullptr, nullptr}, ev_copy_out[2] = {nullptr, nullptr};
    bool import_pending[2] = {false, false};
    void *stage[2] = {nullptr, nullptr};
    size_t stage_bytes[2] = {0, 0};
    std::vector<void *> grave;       // outgrown workspaces (freed with the plan; see ensure_alloc)
    double predicted = 0.0;
    // set by a channel / filter parallel plan on its sub-plans (dc_cconv_*):
    // every conv GEMM of this plan stores fp32 partials scattered by
    // output-channel block (GemmLaunch::scat)
    float *scat[8] = {};
    int scat_seg = 0;

    ~dc_plan_s() {
        for (void *q : grave) cudaFree(q);
        for (auto &b : buf) {
            if (!(comm && comm->group))
                for (auto &kv : b.peer) cudaIpcCloseMemHandle(kv.second);
            if (b.owned && b.ptr) cudaFree(b.ptr);
            if (b.stage) cudaFree(b.stage);
        }
        for (auto &b : dense)
            if (b.owned && b.ptr) cudaFree(b.ptr);
        const bool ipc = !(comm && comm->group);
        if (comm && comm->group) {
            std::lock_guard<std::mutex> lk(comm->group->mu);
            comm->group->plans.erase({seq, rp.rank});
        }
        if (ipc) {
            for (auto &kv : peer_flags) cudaIpcCloseMemHandle(kv.second);
            for (size_t k = 0; k < bn_peer_mail.size(); ++k)
                if (bn_peer_mail[k] && bn_peer_mail[k] != bn_mail) cudaIpcCloseMemHandle(bn_peer_mail[k]);
        }
        if (bn_mail) cudaFree(bn_mail);
        if (bn_epoch) cudaFree(bn_epoch);
        for (int i = 0; i < 2; ++i) {
            if (stage[i]) cudaFree(stage[i]);
            if (ev_copy_in[i]) cudaEventDestroy(ev_copy_in[i]);
            if (ev_copy_out[i]) cudaEventDestroy(ev_copy_out[i]);
        }
        if (s_copy && !s_comm_shared) cudaStreamDestroy(s_copy);
        if (flags) cudaFree(flags);
        if (dev_epochs) cudaFree(dev_epochs);
        if (wt) cudaFree(wt);
        if (wsplit) cudaFree(wsplit);
        if (xsub) cudaFree(xsub);
        if (ws) cudaFree(ws);
        if (ws2) cudaFree(ws2);
        if (bn_part) cudaFree(bn_part);
        if (bn_sums) cudaFree(bn_sums);
        if (bn_fpart) cudaFree(bn_fpart);
        if (bn_coef) cudaFree(bn_coef);
        if (bnb_part) cudaFree(bnb_part);
        if (bn_scratch) cudaFree(bn_scratch);
        for (auto e : ev)
            if (e) cudaEventDestroy(e);
        if (s_comm && !s_comm_shared) cudaStreamDestroy(s_comm);
        for (auto sp : s_ph)
            if (sp && !s_comm_shared) cudaStreamDestroy(sp);
        for (auto e : ev_ph)
            if (e) cudaEventDestroy(e);
        if (bn_comm_owned && bn_comm) ncclCommAbort(bn_comm);  // (see dc_comm_destroy)
    }
    int world() const { return rp.grid.size(); }
    int ks_world = 0;  // dc_plan_set_splitk_world (0: kSplitKBasis)
    int splitk_world() const { return ks_world > 0 ? ks_world : kSplitKBasis; }
    ncclComm_t nccl() const { return comm ? comm->nccl : nullptr; }
    uint32_t *flag(uint32_t *base, int which, int kind, int src) const {
        return base + ((which * 2 + kind) * world() + src);
    }
};

namespace {

// Grow a plan workspace. The old block is NOT freed here: cudaFree waits for
// the whole device, and a compute call may run while this rank's (or, in a
// loopback group, another virtual rank's) halo / BN kernels spin on the device
// for a peer -- it is kept until the plan is destroyed (workspaces only grow
// to a layer's largest need, once).
template <class T>
void ensure_alloc(std::vector<void *> &grave, T *&p, size_t &have, size_t need) {
    if (need <= have) return;
    if (p) grave.push_back(p);
    p = nullptr;
    CK(cudaMalloc(reinterpret_cast<void **>(&p), need));
    have = need;
}

// ---------------------------------------------------------------------------
// shard descriptors
// ---------------------------------------------------------------------------
dc_shard_desc_t describe(const RankPlan &rp, dc_tensor_t t) {
    const ConvGeom &g = rp.g;
    dc_shard_desc_t d{};
    d.n0 = rp.nrange.lo;
    d.n = rp.nrange.size();
    auto fill = [&](int64_t h0, int64_t h, int64_t w0, int64_t w, int64_t c, int64_t cp, int64_t hn,
                    int64_t hs, int64_t hw, int64_t he) {
        d.h0 = h0, d.h = h, d.w0 = w0, d.w = w, d.c = c, d.c_pad = cp;
        d.halo_n = (int32_t)hn, d.halo_s = (int32_t)hs, d.halo_w = (int32_t)hw,
        d.halo_e = (int32_t)he;
        d.hb = hn + h + hs;
        d.wb = hw + w + he;
        d.stride_w = cp;
        d.stride_h = d.wb * cp;
        d.stride_n = d.hb * d.wb * cp;
        d.bytes = (size_t)(d.n * d.stride_n) * g.esz();
    };
    // fp32 (3xTF32) plans: the margined x / dy buffers hold each pixel as
    // [hi (c_pad/2) | lo (c_pad/2)] fp32 (tf32.cuh), y / dx plain fp32
    const int split = g.dt ? 2 : 1;
    switch (t) {
    case DC_X:
        fill(rp.h.in.lo, rp.h.in.size(), rp.w.in.lo, rp.w.in.size(), g.C, split * g.Cp, rp.h.x_halo_lo(),
             rp.h.x_halo_hi(), rp.w.x_halo_lo(), rp.w.x_halo_hi());
        break;
    case DC_DX:
        fill(rp.h.in.lo, rp.h.in.size(), rp.w.in.lo, rp.w.in.size(), g.C, g.Cp, 0, 0, 0, 0);
        break;
    case DC_Y:
        fill(rp.h.out.lo, rp.h.out.size(), rp.w.out.lo, rp.w.out.size(), g.F, g.Fp, 0, 0, 0, 0);
        break;
    case DC_DY:
        fill(rp.h.out.lo, rp.h.out.size(), rp.w.out.lo, rp.w.out.size(), g.F, split * g.Fp,
             rp.h.d_halo_lo(), rp.h.d_halo_hi(), rp.w.d_halo_lo(), rp.w.d_halo_hi());
        break;
    case DC_W:
    case DC_DW: {
        // w: [F][K][K][Cp] bf16 (TMA rows) or fp32; dW: fp32 [F][K][K][C], no
        // padding (what the allreduce sends: F C K^2 words)
        const int64_t cp = t == DC_W ? g.Cp : g.C;
        d.n0 = 0, d.n = g.F, d.h = g.K, d.w = g.K, d.c = g.C, d.c_pad = cp;
        d.hb = g.K, d.wb = g.K;
        d.stride_w = cp, d.stride_h = g.K * cp, d.stride_n = g.K * g.K * cp;
        d.bytes = (size_t)(g.F * g.K * g.K * cp) * (t == DC_W ? g.esz() : 4);
        break;
    }
    default:
        fail(DC_ERR_ARG, "unknown tensor kind");
    }
    return d;
}

// ---------------------------------------------------------------------------
// kernel configuration helpers
// ---------------------------------------------------------------------------
int pick_bkc(int64_t cin_p) { return cin_p % 64 == 0 ? 64 : cin_p % 32 == 0 ? 32 : 16; }
// GEMM N tile: all output channels up to 256, a multiple of 16 (tcgen05 with
// M = 128 needs N % 16 == 0; fp32 plans pad channels only to 8, the extra
// weight rows are TMA zero fill and the epilogue stores only nout_p)
int pick_bn(int64_t nout_p) {
    const int64_t n16 = round_up(nout_p, 16);
    return n16 <= 256 ? (int)n16 : 256;
}
int pick_stages(int bkc, int bn) {
    const int stage = 128 * bkc * 2 + bn * bkc * 2;
    if (stage <= 32 * 1024) return std::max(2, std::min(8, (96 * 1024) / stage));
    return std::max(2, std::min(8, (192 * 1024) / stage));
}
// Tile shape of `pixels`-pixel tiles (TH x TW, TW = 2^twl) with the least
// waste over an nh x nw rectangle; ties go to wider tiles.
int pick_twl(int64_t nh, int64_t nw, int pixels) {
    int best = 3;
    int64_t best_cells = -1;
    for (int twl = 3; (1 << twl) <= pixels; ++twl) {
        const int64_t tw = 1 << twl, th = pixels / tw;
        const int64_t cells = ceil_div(nh, th) * th * ceil_div(nw, tw) * tw;
        if (best_cells < 0 || cells <= best_cells) {
            best = twl;
            best_cells = cells;
        }
    }
    return best;
}

// Interior / boundary split of an nh x nw output grid: lo/hi counts of
// halo-dependent rows and cols ("decomposes ... into its
// interior domain and boundary domains").
struct Split2D {
    int64_t nh, nw, bl, bh, bwl, bwh;
};
void make_rects(const Split2D &s, std::vector<OutRect> &interior, std::vector<OutRect> &boundary) {
    interior.clear();
    boundary.clear();
    int64_t bl = std::min(s.bl, s.nh), bh = std::min(s.bh, s.nh - bl);
    int64_t bwl = std::min(s.bwl, s.nw), bwh = std::min(s.bwh, s.nw - bwl);
    const int64_t ih = s.nh - bl - bh, iw = s.nw - bwl - bwh;
    auto add = [](std::vector<OutRect> &v, int64_t h0, int64_t w0, int64_t nh, int64_t nw) {
        if (nh > 0 && nw > 0) v.push_back(OutRect{(int)h0, (int)w0, (int)nh, (int)nw});
    };
    add(interior, bl, bwl, ih, iw);
    add(boundary, 0, 0, bl, s.nw);
    add(boundary, s.nh - bh, 0, bh, s.nw);
    add(boundary, bl, 0, ih, bwl);
    add(boundary, bl, s.nw - bwh, ih, bwh);
}

// The whole output grid of a launch (union of its interior and boundary rects):
// used when there is no exchange to overlap, so all tiles run in one launch.
struct GemmLaunch;
OutRect whole_of(const std::vector<OutRect> &a, const std::vector<OutRect> &b) {
    int h = 0, w = 0;
    for (auto *v : {&a, &b})
        for (auto &r : *v) {
            h = std::max(h, r.h0 + r.nh);
            w = std::max(w, r.w0 + r.nw);
        }
    return OutRect{0, 0, h, w};
}

void set_rects(ConvGemmParams &p, const std::vector<OutRect> &rects) {
    DC_REQUIRE((int)rects.size() <= kMaxRects, DC_ERR_ARG, "too many rects");
    p.nrect = (int)rects.size();
    p.rect_start[0] = 0;
    for (int r = 0; r < p.nrect; ++r) {
        p.rect[r] = rects[r];
        const int twl = pick_twl(rects[r].nh, rects[r].nw, 128);
        const int tw = 1 << twl, th = 128 >> twl;
        p.rect_twl[r] = twl;
        p.rect_tiles_w[r] = (int)ceil_div(rects[r].nw, tw);
        p.rect_start[r + 1] = p.rect_start[r] + (int)ceil_div(rects[r].nh, th) * p.rect_tiles_w[r];
    }
}

// 4D tensor map over an NHWC buffer [n][hb][wb][cp] with a box of
// (bc channels) x (tw cols) x (th rows) x 1 sample, element stride s.
void nhwc_map(CUtensorMap *m, const void *base, int64_t n, int64_t hb, int64_t wb, int64_t cp,
              int64_t row_pitch_px, int64_t img_pitch_px, int bc, int tw, int th, int s) {
    const uint64_t dims[4] = {(uint64_t)cp, (uint64_t)wb, (uint64_t)hb, (uint64_t)n};
    const uint64_t strides[3] = {(uint64_t)(cp * 2), (uint64_t)(row_pitch_px * cp * 2),
                                 (uint64_t)(img_pitch_px * cp * 2)};
    const uint32_t box[4] = {(uint32_t)bc, (uint32_t)(tw * s), (uint32_t)(th * s), 1};
    const uint32_t es[4] = {1, (uint32_t)s, (uint32_t)s, 1};
    make_tmap(m, base, 4, dims, strides, box, es, bc * 2);
}

void weight_map(CUtensorMap *m, const void *base, int64_t rows, int64_t kcols, int bkc, int bn) {
    const uint64_t dims[2] = {(uint64_t)kcols, (uint64_t)rows};
    const uint64_t strides[1] = {(uint64_t)(kcols * 2)};
    const uint32_t box[2] = {(uint32_t)bkc, (uint32_t)bn};
    make_tmap(m, base, 2, dims, strides, box, nullptr, bkc * 2);
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
struct GemmLaunch {
    CUtensorMap amap, bmap;
    ConvGemmParams p;
    std::vector<OutRect> interior, boundary;
    int nout_tiles = 0;
    const void *w_base = nullptr;  // B matrix [w_rows][w_kcols] (for re-tiling N)
    int64_t w_rows = 0, w_kcols = 0;
    int ksplit = 1;            // v2 split-K over channel groups (from the GLOBAL shape)
    int64_t work_hint = 0;     // 16x8 tiles x N tiles of the global layer / splitk_world
    int max_ctas = 0;          // persistent grid cap (0: all SMs), leaves SMs to a concurrent launch
    // fused BN statistics: per-CTA partial slots [slot][2][nout_p] (fp64)
    double *bn_part = nullptr;
    int bn_slot = 0, bn_slot_cap = 0;
    bool bn_ok = true;
    int dep[4] = {0, 0, 0, 0};       // output rows/cols reading the halo: top, bottom, left, right
    int subpix = 0, sub_cp = 0, out_hmax = 0, out_wmax = 0;  // sub-pixel backward-data
    float *ws = nullptr;       // its fp32 partials
    int ws_h = 0, ws_w = 0;
    // 3xTF32 (fp32 plans): kind::tf32, input channels in 16-bit units a_cvirt
    // (the [hi | lo] buffer) vs the weights' K per tap cin_p (hi | lo | hi),
    // the remap boundary a_seg, fp32 output
    int kind = 0, a_seg = 0;
    int64_t a_cvirt = 0;
    bool out_f32 = false;
    int64_t cin = 0;           // K per tap of the B matrix, 16-bit units
    // channel / filter parallelism: fp32 output scattered by output-channel
    // block into the owners' receive slots (ConvV2Params::scat)
    float *scat[8] = {};
    int scat_seg = 0;
    // a 1x1 stride-1 conv on a margin-free shard is a plain GEMM over pixels:
    // the shard is launched as ONE row of n h w pixels in 1 x 128 tiles, which
    // cross image rows and samples (small images waste no tile rows)
    bool flat = false;
};

// The 1x1 stride-1 flattening applies (no padding, no margins on the input).
bool flat_ok(const ConvGeom &g, const dc_shard_desc_t &in) {
    return g.K == 1 && g.S == 1 && g.P == 0 && in.halo_n == 0 && in.halo_s == 0 && in.halo_w == 0 &&
           in.halo_e == 0 && in.n * in.hb * in.wb < (int64_t(1) << 31);
}

OutRect whole(const GemmLaunch &L) { return whole_of(L.interior, L.boundary); }

// 1x1 stride-2 forward through the gathered pixels (subsample.cuh): bf16, no
// padding, no input margins, one output rect (no halo-dependent tiles).
bool sub2_ok(const dc_plan_s *pl, const GemmLaunch &L, const dc_shard_desc_t &xd) {
    const ConvGeom &g = pl->rp.g;
    return g.K == 1 && g.S == 2 && g.P == 0 && g.dt == 0 && L.kind == 0 && !L.scat_seg && xd.halo_n == 0 &&
           xd.halo_s == 0 && xd.halo_w == 0 && xd.halo_e == 0 && L.interior.size() + L.boundary.size() == 1 &&
           pl->rp.nrange.size() * pl->rp.h.out.size() * pl->rp.w.out.size() < (int64_t(1) << 31);
}

// Split-K over channel groups for the v2 kernel, chosen from the GLOBAL problem
// (tiles of the unpartitioned layer) so that every decomposition sums each
// output element in the same order (partitioned == 1 GPU, bitwise).
int choose_ksplit(int64_t global_tiles, int64_t cin_p) {
    const int ncg = (int)(cin_p / pick_bkc(cin_p));
    int k = 1;
    while (2 * k <= ncg && ncg % (2 * k) == 0 && global_tiles * 2 * k <= device_sm_count() * 3 / 2) k *= 2;
    return k;
}
size_t ksplit_bytes(const GemmLaunch &L, int nl) {
    const OutRect b = whole(L);
    return L.ksplit > 1 ? (size_t)L.ksplit * nl * b.nh * b.nw * L.p.nout_p * 4 : 0;
}
void attach_ksplit(dc_plan_s *pl, GemmLaunch &L, int nl) {
    if (L.ksplit <= 1) return;
    const OutRect b = whole(L);
    L.ws_h = b.nh, L.ws_w = b.nw;
    ensure_alloc(pl->grave, pl->ws2, pl->ws2_bytes, ksplit_bytes(L, nl));
    L.ws = pl->ws2;
}

// Channel / filter parallel sub-plans: fp32 partials to the owners' slots.
void apply_scatter(const dc_plan_s *pl, GemmLaunch &L) {
    if (!pl->scat_seg) return;
    L.out_f32 = true;
    std::memcpy(L.scat, pl->scat, sizeof L.scat);
    L.scat_seg = pl->scat_seg;
}

void prepare_fwd(dc_plan_s *pl, const void *x, const void *w, void *y, GemmLaunch &L, cudaStream_t st) {
    const RankPlan &rp = pl->rp;
    const ConvGeom &g = rp.g;
    const dc_shard_desc_t xd = describe(rp, DC_X), yd = describe(rp, DC_Y);
    ConvGemmParams &p = L.p;
    std::memset(&p, 0, sizeof p);
    // K per tap in 16-bit units: C_pad bf16, or [w_hi | w_lo | w_hi] fp32
    // (3 x 2 C_pad) against the input's [x_hi | x_lo] (2 x 2 C_pad)
    const bool f32 = g.dt == 1;
    L.cin = f32 ? 6 * g.Cp : g.Cp;
    if (f32) {
        ensure_alloc(pl->grave, pl->wsplit, pl->wsplit_bytes, (size_t)g.F * g.K * g.K * 3 * g.Cp * 4);
        launch_weight_split(reinterpret_cast<const float *>(w), pl->wsplit, (int)g.F, g.K * g.K, (int)g.C, (int)g.Cp,
                            st);
        w = pl->wsplit;
        L.kind = 1, L.a_seg = (int)(2 * g.Cp), L.a_cvirt = 4 * g.Cp, L.out_f32 = true;
    }
    p.bkc = pick_bkc(L.cin);
    p.kc = (int)(L.cin / p.bkc);
    p.bn = pick_bn(g.Fp);
    p.stages = pick_stages(p.bkc, p.bn);
    p.T = g.K * g.K;
    DC_REQUIRE(p.T <= kMaxTaps, DC_ERR_UNSUPPORTED, "K=%d too large", g.K);
    for (int a = 0; a < g.K; ++a)
        for (int b = 0; b < g.K; ++b) {
            p.tap_h[a * g.K + b] = (int8_t)a;
            p.tap_w[a * g.K + b] = (int8_t)b;
        }
    p.s_in = g.S;
    p.origin_h = (int)(g.S * rp.h.out.lo - g.P - rp.h.xbuf.lo);
    p.origin_w = (int)(g.S * rp.w.out.lo - g.P - rp.w.xbuf.lo);
    p.out = reinterpret_cast<__nv_bfloat16 *>(y);
    p.out_sn = yd.stride_n, p.out_sh = yd.stride_h, p.out_sw = yd.stride_w;
    p.out_h0 = 0, p.out_w0 = 0, p.out_dh = 1, p.out_dw = 1;
    p.nout_p = (int)g.Fp;
    L.nout_tiles = (int)ceil_div(g.Fp, p.bn);
    // the A map's box depends on the tile shape of each rect: encoded in launch_rects
    (void)x;
    (void)xd;
    weight_map(&L.bmap, w, g.F, (int64_t)g.K * g.K * L.cin, p.bkc, p.bn);
    L.w_base = w, L.w_rows = g.F, L.w_kcols = (int64_t)g.K * g.K * L.cin;
    // halo-dependent output rows/cols (only toward existing neighbours)
    auto count = [&](const DimSplit &d, bool lo) -> int64_t {
        const bool nb = lo ? d.idx > 0 : d.idx + 1 < d.parts;
        if (!nb) return 0;
        int64_t c = 0;
        const int64_t n = d.out.size();
        for (int64_t k = 0; k < n; ++k) {
            const int64_t i = lo ? k : n - 1 - k;
            const int64_t gl = g.S * (d.out.lo + i) - g.P;
            const bool dep = lo ? gl < d.in.lo : gl + g.K - 1 >= d.in.hi;
            if (!dep) break;
            ++c;
        }
        return c;
    };
    Split2D s{rp.h.out.size(), rp.w.out.size(), count(rp.h, true), count(rp.h, false),
              count(rp.w, true), count(rp.w, false)};
    make_rects(s, L.interior, L.boundary);
    L.dep[0] = (int)s.bl, L.dep[1] = (int)s.bh, L.dep[2] = (int)s.bwl, L.dep[3] = (int)s.bwh;
    // per-rank share of the global layer (splitk_world ranks; default: this grid)
    L.work_hint = ceil_div(g.N * ceil_div(g.Ho, kV2TH) * ceil_div(g.Wo, kV2TW) * L.nout_tiles,
                           (int64_t)pl->splitk_world());
    L.ksplit = choose_ksplit(L.work_hint, L.cin);
    attach_ksplit(pl, L, (int)rp.nrange.size());
    apply_scatter(pl, L);
    L.flat = flat_ok(g, xd) && L.interior.size() + L.boundary.size() == 1;
}

// Launch a conv GEMM over `rects`; one launch per distinct tile width (the A
// box shape is baked into the tensor map).
// The persistent tile-reuse kernel (conv_v2.cu); false if it does not apply.
// One launch of the persistent tile-reuse kernel (conv_v2.cu) over `rects`
// with tile shape 2^twl columns; false if the configuration does not fit.
bool launch_v2_shape(GemmLaunch &L, const std::vector<OutRect> &rects, int twl, const void *in_base,
                     const dc_shard_desc_t &ind, int64_t cin_p, int nsamples, cudaStream_t st) {
    ConvV2Params q;
    std::memset(&q, 0, sizeof q);
    q.s_in = L.p.s_in;
    q.origin_h = L.p.origin_h;
    q.origin_w = L.p.origin_w;
    q.T = L.p.T;
    std::memcpy(q.tap_h, L.p.tap_h, sizeof q.tap_h);
    std::memcpy(q.tap_w, L.p.tap_w, sizeof q.tap_w);
    q.cin_p = (int)cin_p;
    q.ksplit = L.ksplit;
    q.kind = L.kind, q.a_seg = L.a_seg, q.out_f32 = L.out_f32 ? 1 : 0;
    q.subpix = L.subpix, q.sub_cp = L.sub_cp, q.out_hmax = L.out_hmax, q.out_wmax = L.out_wmax;
    q.ws = L.ws;
    q.ws_h = L.ws_h;
    q.ws_w = L.ws_w;
    q.nsamples = nsamples;
    q.tw_log2 = twl;
    q.out = L.p.out;
    q.out_sn = L.p.out_sn, q.out_sh = L.p.out_sh, q.out_sw = L.p.out_sw;
    q.out_h0 = L.p.out_h0, q.out_w0 = L.p.out_w0, q.out_dh = L.p.out_dh, q.out_dw = L.p.out_dw;
    q.nout_p = L.p.nout_p;
    q.max_ctas = L.max_ctas;
    if (L.scat_seg) {  // the receive slots have channel pitch scat_seg
        std::memcpy(q.scat, L.scat, sizeof q.scat);
        q.scat_seg = L.scat_seg;
        const long long cp = L.p.out_sw;
        q.out_sw = L.scat_seg, q.out_sh = L.p.out_sh / cp * L.scat_seg, q.out_sn = L.p.out_sn / cp * L.scat_seg;
    }
    const int TW = 1 << twl, TH = 128 >> twl;
    // (1) choices that change the summation order (channel-stage width) come
    // from the GLOBAL layer, so every partition computes the 1-GPU bits
    {
        ConvV2Params probe = q;
        probe.bn = L.p.bn;
        probe.nout_tiles = (int)ceil_div(L.p.nout_p, probe.bn);
        probe.work_hint = (int)std::min<int64_t>(L.work_hint * L.ksplit, 1 << 30);
        probe.allow_cg32 = 1;
        if (!conv_v2_configure(probe, kV2SmemLimit)) return false;
        q.cg = probe.cg;
        q.allow_cg32 = 0;
    }
    // (2) bitwise-neutral choices from THIS launch's work: no tile pairing
    // when the shard is too small to fill the GPU. (A narrower N tile for small
    // shards was measured slower: every N tile reloads the whole input tile.)
    int64_t local_tiles = 0;
    for (auto &r : rects) local_tiles += ceil_div(r.nh, TH) * ceil_div(r.nw, TW);
    local_tiles *= nsamples;
    q.bn = L.p.bn;
    q.nout_tiles = (int)ceil_div(L.p.nout_p, q.bn);
    q.work_hint = (int)std::min<int64_t>(local_tiles * q.nout_tiles * L.ksplit, 1 << 30);
    // fused BN statistics when the epilogue holds final values of all channels
    // (bitwise-neutral: the stage width above was chosen without them)
    // (only with enough MMA work per tile to hide the epilogue reduction: K =
    // C_pad x taps >= 1152, measured: fusing a K = 576 layer costs more than
    // the separate pass over y)
    // (N tiles <= 64: register accumulation, cheap enough for any K)
    // (several N tiles: not fused -- measured in round 1 on the N = 8 mesh
    // step, per-CTA segments per N tile moved 0.31 ms from the BN pass into
    // the forwards, conv4_1 fwd 0.31 -> 0.41 ms, for no net gain)
    const bool nt_ok = q.nout_tiles == 1 && !L.out_f32;
    // (256-wide N tiles: not fused -- measured in round 2, cold L2, N = 8:
    // conv3_1 forward 310 -> 471 us fused, conv3_2 436 -> 528 us, against a
    // ~55 us separate pass over y; 128-wide: conv2_2 579 -> 616 us, about the
    // separate pass; 64-wide register accumulation: +6 us)
    q.bn_stats = !(L.bn_part && L.ksplit == 1 && nt_ok) ? 0
                 : q.bn <= 64                                      ? 2
                 : q.bn <= 128 && (int64_t)q.cin_p * q.T >= 1152  ? 1
                                                                   : 0;
    if (L.bn_part && !q.bn_stats) L.bn_ok = false;
    if (q.bn_stats) {
        ConvV2Params t = q;
        if (!conv_v2_configure(t, kV2SmemLimit)) q.bn_stats = 0, L.bn_ok = false;
    }
    if (!conv_v2_configure(q, kV2SmemLimit)) return false;
    DC_REQUIRE((int)rects.size() <= kMaxRects, DC_ERR_ARG, "too many rects");
    q.nrect = (int)rects.size();
    q.rect_start[0] = 0;
    for (int r = 0; r < q.nrect; ++r) {
        q.rect[r] = rects[r];
        q.rect_tiles_w[r] = (int)ceil_div(rects[r].nw, TW);
        q.rect_start[r + 1] = q.rect_start[r] + (int)ceil_div(rects[r].nh, TH * q.tpw) * q.rect_tiles_w[r];
    }
    q.total_tiles = q.nout_tiles * q.nsamples * q.rect_start[q.nrect];
    CUtensorMap amap;
    const int64_t a_c = L.a_cvirt > 0 ? L.a_cvirt : cin_p;  // 16-bit units per input pixel
    const uint64_t dims[4] = {(uint64_t)a_c, (uint64_t)ind.wb, (uint64_t)ind.hb, (uint64_t)ind.n};
    const uint64_t strides[3] = {(uint64_t)(a_c * 2), (uint64_t)(ind.wb * a_c * 2),
                                 (uint64_t)(ind.hb * ind.wb * a_c * 2)};
    if (q.a_swz) {
        const uint32_t box[4] = {(uint32_t)q.cg, (uint32_t)(q.PWs * q.s_in), (uint32_t)q.PH, 1};
        const uint32_t es[4] = {1, (uint32_t)q.s_in, 1, 1};
        make_tmap(&amap, in_base, 4, dims, strides, box, es, q.a_swz);
    } else {
        const uint32_t box[4] = {8, (uint32_t)(q.PWs * q.s_in), (uint32_t)q.PH, 1};
        const uint32_t es[4] = {1, (uint32_t)q.s_in, 1, 1};
        make_tmap(&amap, in_base, 4, dims, strides, box, es, 0);
    }
    if (q.bn_stats) {
        // worst-case slot count of this launch (persistent grid <= SMs)
        if (L.bn_slot + device_sm_count() > L.bn_slot_cap) {
            q.bn_stats = 0, L.bn_ok = false;
            if (!conv_v2_configure(q, kV2SmemLimit)) return false;
        } else {
            q.bn_part = L.bn_part + (size_t)L.bn_slot * 2 * q.nout_p;
        }
    }
    int grid = 0;
    if (q.cg != L.p.bkc || q.bn != L.p.bn || q.cluster > 1) {
        // narrower channel stages, or half-height boxes (each CTA of a pair
        // loads half of every weight stage): re-tile the weights
        CUtensorMap bmap;
        weight_map(&bmap, L.w_base, L.w_rows, L.w_kcols, q.cg, q.bn / q.cluster);
        grid = launch_conv_v2(amap, bmap, q, st);
    } else {
        grid = launch_conv_v2(amap, L.bmap, q, st);
    }
    if (q.bn_stats) L.bn_slot += grid;
    if (q.ksplit > 1) launch_conv_v2_reduce(q, st);
    return true;
}

// Thin rects (boundary strips of an H split) use 1 x 128 tiles, the rest 16 x 8.
bool launch_rects_v2(GemmLaunch &L, const std::vector<OutRect> &rects, const void *in_base,
                     const dc_shard_desc_t &ind, int64_t cin_p, int nsamples, cudaStream_t st) {
    if (L.p.T == 0) return false;
    std::vector<OutRect> tall, thin;
    for (auto &r : rects)
        (L.p.s_in == 1 && r.nh < 8 && r.nw >= 64 ? thin : tall).push_back(r);
    if (!thin.empty() && !launch_v2_shape(L, thin, 7, in_base, ind, cin_p, nsamples, st))
        tall.insert(tall.end(), thin.begin(), thin.end());
    if (tall.empty()) return true;
    return launch_v2_shape(L, tall, 3, in_base, ind, cin_p, nsamples, st);
}

void launch_rects(GemmLaunch &L, const std::vector<OutRect> &rects, const void *in_base,
                  const dc_shard_desc_t &ind, int64_t cin_p, int nsamples, cudaStream_t st) {
    if (rects.empty()) return;
    if (L.flat) {  // the whole shard as one row of pixels (the rects cover it all)
        dc_shard_desc_t f = ind;
        f.wb = f.w = ind.n * ind.hb * ind.wb;
        f.n = 1, f.hb = f.h = 1;
        const int ws_h = L.ws_h, ws_w = L.ws_w;
        L.ws_h = 1, L.ws_w = (int)f.wb;
        const bool ok = launch_rects_v2(L, {OutRect{0, 0, 1, (int)f.wb}}, in_base, f, cin_p, 1, st);
        L.ws_h = ws_h, L.ws_w = ws_w;
        DC_REQUIRE(ok, DC_ERR_UNSUPPORTED, "1x1 conv: the tile-reuse kernel does not fit");
        return;
    }
    if (launch_rects_v2(L, rects, in_base, ind, cin_p, nsamples, st)) return;
    DC_REQUIRE(L.kind == 0, DC_ERR_UNSUPPORTED, "3xTF32: the tile-reuse kernel does not fit this layer");
    DC_REQUIRE(L.scat_seg == 0, DC_ERR_UNSUPPORTED, "channel-parallel partials: the tile-reuse kernel does not fit");
    L.bn_ok = false;  // (the v1 kernel has no fused statistics)
    std::map<int, std::vector<OutRect>> by_twl;
    for (auto &r : rects) by_twl[pick_twl(r.nh, r.nw, 128)].push_back(r);
    for (auto &kv : by_twl) {
        const int twl = kv.first, tw = 1 << twl, th = 128 >> twl;
        nhwc_map(&L.amap, in_base, ind.n, ind.hb, ind.wb, cin_p, ind.wb, ind.hb * ind.wb, L.p.bkc,
                 tw, th, L.p.s_in);
        set_rects(L.p, kv.second);
        launch_conv_gemm(L.amap, L.bmap, L.p, nsamples, L.nout_tiles, st);
    }
}

// ---------------------------------------------------------------------------
// halo exchange
// ---------------------------------------------------------------------------
P2PExchange build_p2p(dc_plan_s *pl, int which, void *buf);
bool is_local(const dc_plan_s *pl);
void resolve_local_peers(dc_plan_s *pl);

// The P2P protocol of one exchange of tensor `which` (0: x, 1: dy) of the
// registered buffer `buf`: my slabs -> the neighbours' mapped margins, their
// ready flags / my data counters (halo.cuh: P2PExchange).
P2PExchange build_p2p(dc_plan_s *pl, int which, void *buf) {
    const RankPlan &rp = pl->rp;
    const auto &sends = which == 0 ? rp.x_send : rp.dy_send;
    const auto &recvs = which == 0 ? rp.x_recv : rp.dy_recv;
    // bytes per pixel of the margined buffer (bf16 c_pad, or fp32 [hi | lo])
    const int64_t cp = describe(rp, which == 0 ? DC_X : DC_DY).c_pad * rp.g.esz() / 2;  // in 16-bit units
    const int vec16 = (int)(cp * 2 / 16);
    const int64_t nl = rp.nrange.size();
    BufState &B = pl->buf[which];
    const int me = rp.rank;
    DC_REQUIRE(B.ptr == buf, DC_ERR_ARG,
               "direct P2P halo exchange needs the buffer from dc_buffer_alloc (or pass DC_HALO_NCCL)");
    DC_REQUIRE(sends.size() <= 8 && recvs.size() <= 8, DC_ERR_ARG, "too many halo neighbours");
    DC_REQUIRE(B.dev_epoch != nullptr, DC_ERR_ARG, "P2P halo exchange: buffer not registered");
    resolve_local_peers(pl);
    for (auto &m : sends)
        DC_REQUIRE(B.peer.count(m.peer) && pl->peer_flags.count(m.peer), DC_ERR_ARG,
                   "P2P halo exchange: rank %d's buffer is not mapped (dc_buffer_alloc on every rank)", m.peer);
    for (auto &m : recvs)
        DC_REQUIRE(pl->peer_flags.count(m.peer), DC_ERR_ARG, "P2P halo exchange: rank %d's flags are not mapped",
                   m.peer);
    auto strides = [&](int64_t hb, int64_t wb, BlockCopy &c, bool src) {
        const long long sw = vec16, sh = wb * vec16, sn = hb * wb * vec16;
        if (src) c.s_sn = sn, c.s_sh = sh, c.s_sw = sw;
        else c.d_sn = sn, c.d_sh = sh, c.d_sw = sw;
    };
    P2PExchange x{};
    x.epoch_ctr = B.dev_epoch;
    for (auto &m : recvs) x.ready_out[x.n_ready_out++] = pl->flag(pl->peer_flags.at(m.peer), which, FLAG_READY, me);
    for (auto &m : sends) {
        x.ready_in[x.n_ready_in++] = pl->flag(pl->flags, which, FLAG_READY, m.peer);
        x.data_out[x.n_data_out++] = pl->flag(pl->peer_flags.at(m.peer), which, FLAG_DATA, me);
        BlockCopy &c = x.copies.c[x.copies.count++];
        c.src = reinterpret_cast<const uint4 *>(buf) + (m.src_row0 * m.src_wb + m.src_col0) * vec16;
        strides(m.src_hb, m.src_wb, c, true);
        c.dst = reinterpret_cast<uint4 *>(B.peer.at(m.peer)) + (m.dst_row0 * m.dst_wb + m.dst_col0) * vec16;
        strides(m.dst_hb, m.dst_wb, c, false);
        c.nn = (int)nl, c.rows = (int)m.rows.size(), c.cols = (int)m.cols.size(), c.vec16 = vec16;
    }
    for (auto &m : recvs) x.data_in[x.n_data_in++] = pl->flag(pl->flags, which, FLAG_DATA, m.peer);
    return x;
}

// Halo bytes this rank receives for tensor `which` (0: x, 1: dy).
size_t halo_recv_bytes(const dc_plan_s *pl, int which) {
    const RankPlan &rp = pl->rp;
    const int64_t px = describe(rp, which == 0 ? DC_X : DC_DY).c_pad * rp.g.esz();
    size_t b = 0;
    for (auto &m : which == 0 ? rp.x_recv : rp.dy_recv) b += (size_t)rp.nrange.size() * m.rows.size() * m.cols.size() * px;
    return b;
}

// Interior / boundary overlap of an exchange only when the
// halo is large: measured in round 2 on the mesh2k_n8 step, where every halo
// is <= 2 MB (one row), exchanging first and computing the whole shard in one
// launch beat the two-launch overlap (2 GPUs 20.46 -> 20.27 ms, 4 GPUs 12.15
// -> 11.81 ms; the whole step's exchanges cost 0.7 / 1.0 ms): a ~15 us
// exchange is cheaper than the extra boundary launch that hides it.
constexpr size_t kOverlapMinHaloBytes = size_t(8) << 20;

void exchange(dc_plan_s *pl, int which, void *buf, unsigned flags, cudaStream_t st) {
    const RankPlan &rp = pl->rp;
    const auto &sends = which == 0 ? rp.x_send : rp.dy_send;
    const auto &recvs = which == 0 ? rp.x_recv : rp.dy_recv;
    if (sends.empty() && recvs.empty()) return;
    DC_REQUIRE(!pl->is_virtual && pl->comm && (pl->comm->nccl || pl->comm->group), DC_ERR_ARG,
               "halo exchange needs a communicator (virtual plan or world 1)");
    DC_REQUIRE(!(is_local(pl) && (flags & DC_HALO_NCCL)), DC_ERR_UNSUPPORTED,
               "DC_HALO_NCCL needs real ranks (loopback group)");
    // bytes per pixel of the margined buffer (bf16 c_pad, or fp32 [hi | lo])
    const int64_t cp = describe(rp, which == 0 ? DC_X : DC_DY).c_pad * rp.g.esz() / 2;  // in 16-bit units
    const int vec16 = (int)(cp * 2 / 16);
    const int64_t nl = rp.nrange.size();
    BufState &B = pl->buf[which];
    const bool use_nccl = (flags & DC_HALO_NCCL) != 0;
    auto strides = [&](int64_t hb, int64_t wb, BlockCopy &c, bool src) {
        const long long sw = vec16, sh = wb * vec16, sn = hb * wb * vec16;
        if (src) c.s_sn = sn, c.s_sh = sh, c.s_sw = sw;
        else c.d_sn = sn, c.d_sh = sh, c.d_sw = sw;
    };
    if (use_nccl) {
        size_t send_bytes = 0, recv_bytes = 0;
        for (auto &m : sends) send_bytes += (size_t)nl * m.rows.size() * m.cols.size() * cp * 2;
        for (auto &m : recvs) recv_bytes += (size_t)nl * m.rows.size() * m.cols.size() * cp * 2;
        ensure_alloc(pl->grave, reinterpret_cast<uint8_t *&>(B.stage), B.stage_bytes, send_bytes + recv_bytes);
        uint8_t *sbuf = reinterpret_cast<uint8_t *>(B.stage), *rbuf = sbuf + send_bytes;
        CopyBatch pack{};
        size_t off = 0;
        for (auto &m : sends) {
            BlockCopy &c = pack.c[pack.count++];
            c.src = reinterpret_cast<const uint4 *>(buf) +
                    (m.src_row0 * m.src_wb + m.src_col0) * vec16;
            c.dst = reinterpret_cast<uint4 *>(sbuf + off);
            strides(m.src_hb, m.src_wb, c, true);
            c.d_sw = vec16, c.d_sh = m.cols.size() * vec16, c.d_sn = m.rows.size() * c.d_sh;
            c.nn = (int)nl, c.rows = (int)m.rows.size(), c.cols = (int)m.cols.size(), c.vec16 = vec16;
            off += (size_t)nl * m.rows.size() * m.cols.size() * cp * 2;
        }
        launch_block_copies(pack, st);
        NK(ncclGroupStart());
        off = 0;
        for (auto &m : sends) {
            const size_t b = (size_t)nl * m.rows.size() * m.cols.size() * cp * 2;
            NK(ncclSend(sbuf + off, b, ncclUint8, m.peer, pl->nccl(), st));
            off += b;
        }
        off = 0;
        for (auto &m : recvs) {
            const size_t b = (size_t)nl * m.rows.size() * m.cols.size() * cp * 2;
            NK(ncclRecv(rbuf + off, b, ncclUint8, m.peer, pl->nccl(), st));
            off += b;
        }
        NK(ncclGroupEnd());
        CopyBatch unpack{};
        off = 0;
        for (auto &m : recvs) {
            BlockCopy &c = unpack.c[unpack.count++];
            c.src = reinterpret_cast<const uint4 *>(rbuf + off);
            c.s_sw = vec16, c.s_sh = m.cols.size() * vec16, c.s_sn = m.rows.size() * c.s_sh;
            c.dst = reinterpret_cast<uint4 *>(buf) + (m.dst_row0 * m.dst_wb + m.dst_col0) * vec16;
            strides(m.dst_hb, m.dst_wb, c, false);
            c.nn = (int)nl, c.rows = (int)m.rows.size(), c.cols = (int)m.cols.size(), c.vec16 = vec16;
            off += (size_t)nl * m.rows.size() * m.cols.size() * cp * 2;
        }
        launch_block_copies(unpack, st);
        return;
    }
    // ---- direct P2P stores into the neighbours' margins + epoch flags ----
    // one kernel: ready handshake, NVLink stores, per-block completion counters
    // (halo.cu: p2p_exchange_kernel), block 0 returns when all data arrived.
    const P2PExchange x = build_p2p(pl, which, buf);
    launch_p2p_exchange(x, st);
}

// All-gather fixed-size blobs over NCCL (host in/out); used for IPC handles.
// All-gather fixed-size blobs over the communicator's NCCL (host in/out); used
// for IPC handles and for checking that every rank chose the same grid.
std::vector<uint8_t> comm_allgather(dc_comm_s *c, const void *mine, size_t n) {
    const int W = c->world;
    DC_REQUIRE(c->nccl != nullptr, DC_ERR_ARG, "all-gather needs an NCCL communicator");
    uint8_t *d = nullptr;
    cudaStream_t s = nullptr;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CK(cudaMalloc(&d, n * (W + 1)));
    CK(cudaMemcpy(d + n * W, mine, n, cudaMemcpyHostToDevice));
    NK(ncclAllGather(d + n * W, d, n, ncclUint8, c->nccl, s));
    CK(cudaStreamSynchronize(s));
    std::vector<uint8_t> out(n * W);
    CK(cudaMemcpy(out.data(), d, n * W, cudaMemcpyDeviceToHost));
    CK(cudaFree(d));
    CK(cudaStreamDestroy(s));
    return out;
}
std::vector<uint8_t> allgather_bytes(dc_plan_s *pl, const void *mine, size_t n) {
    return comm_allgather(pl->comm, mine, n);
}

std::vector<int> neighbours(const RankPlan &rp, int which) {
    std::vector<int> v;
    for (auto *L : {which == 0 ? &rp.x_send : &rp.dy_send, which == 0 ? &rp.x_recv : &rp.dy_recv})
        for (auto &m : *L)
            if (std::find(v.begin(), v.end(), m.peer) == v.end()) v.push_back(m.peer);
    return v;
}

bool is_local(const dc_plan_s *pl) { return pl->comm && pl->comm->group; }

// Loopback group: the plan of `rank` with this plan's sequence number.
dc_plan_s *local_peer(dc_plan_s *pl, int rank) {
    LocalGroup &G = *pl->comm->group;
    std::lock_guard<std::mutex> lk(G.mu);
    auto it = G.plans.find({pl->seq, rank});
    DC_REQUIRE(it != G.plans.end(), DC_ERR_ARG, "loopback group: rank %d has not created plan #%d", rank, pl->seq);
    return it->second;
}

// Loopback group: resolve the cross-rank pointers (neighbours' flags and
// margined buffers, the BN group's mailboxes) from the registry. Called before
// every use, since a buffer may be allocated after the neighbour's plan.
void resolve_local_peers(dc_plan_s *pl) {
    if (!is_local(pl) || pl->world() <= 1) return;
    std::vector<int> nb = neighbours(pl->rp, 0);
    for (int p : neighbours(pl->rp, 1))
        if (std::find(nb.begin(), nb.end(), p) == nb.end()) nb.push_back(p);
    for (int p : nb) {
        dc_plan_s *q = local_peer(pl, p);
        pl->peer_flags[p] = q->flags;
        for (int which = 0; which < 2; ++which)
            if (q->buf[which].ptr) pl->buf[which].peer[p] = q->buf[which].ptr;
    }
    if (pl->bn_p2p) {
        const int lo = pl->rp.in * pl->bn_group;
        for (int k = 0; k < pl->bn_group; ++k) pl->bn_peer_mail[k] = local_peer(pl, lo + k)->bn_mail;
    }
}

// ---------------------------------------------------------------------------
// backward-data
// ---------------------------------------------------------------------------
struct Phase {
    bool active = false;
    int T = 0;
    int8_t tap_h[kMaxTaps], tap_w[kMaxTaps], ka[kMaxTaps], kb[kMaxTaps];
    int origin_h, origin_w, out_h0, out_w0;
    int64_t nt_h, nt_w;
    int64_t bl, bh, bwl, bwh;
};

// Phase decomposition of Eq. 3 for stride S (reading R4):
// input rows u = S t + rho read dy rows t + e - m through taps a = a0 + S m.
struct DimPhase {
    int M = 0;
    int64_t t0 = 0, nt = 0;
    int origin = 0, out0 = 0;
    int a0 = 0;
    int64_t bl = 0, bh = 0;
};
DimPhase dim_phase(const DimSplit &d, int K, int S, int P, int rho) {
    DimPhase r;
    r.a0 = (rho + P) % S;
    r.M = r.a0 < K ? (int)ceil_div(K - r.a0, S) : 0;
    const int e = (rho + P - r.a0) / S;
    const int64_t q = d.in.lo, rr = d.in.hi - 1;
    r.t0 = -floor_div(-(q - rho), S);
    const int64_t t1 = floor_div(rr - rho, S);
    r.nt = std::max<int64_t>(0, t1 - r.t0 + 1);
    r.origin = (int)(r.t0 + e - d.dbuf.lo - r.M + 1);
    r.out0 = (int)(S * r.t0 + rho - q);
    if (r.M > 0) {
        if (d.idx > 0)
            for (int64_t k = 0; k < r.nt; ++k) {
                if (k + r.origin + d.dbuf.lo < d.out.lo) ++r.bl;
                else break;
            }
        if (d.idx + 1 < d.parts)
            for (int64_t k = r.nt - 1; k >= 0; --k) {
                if (k + r.origin + r.M - 1 + d.dbuf.lo >= d.out.hi) ++r.bh;
                else break;
            }
    }
    return r;
}

// Stride 2 with few input channels (C_pad <= 32): the four stride phases as ONE
// stride-1 GEMM over a D x D dy window with 4 C_pad output columns (N = 64 or
// 128 instead of four N = 16/32 GEMMs); phase taps outside the filter carry
// zero weights and the epilogue scatters each 16-column chunk to its phase's
// pixel (depth-to-space). dx = sum over the window in a fixed tap order, the
// same on every rank (partitioned == 1 GPU bitwise). False: not applicable.
bool run_bwd_data_subpix(dc_plan_s *pl, void *dy, const void *w, void *dx, unsigned flags, cudaStream_t st,
                         bool *exchanged) {
    const RankPlan &rp = pl->rp;
    const ConvGeom &g = rp.g;
    if (g.dt != 0 || g.S != 2 || g.Cp > 32 || pl->scat_seg) return false;
    const dc_shard_desc_t dyd = describe(rp, DC_DY), dxd = describe(rp, DC_DX);
    const int K = g.K, P = g.P;
    const int dmin = -(int)floor_div(K - 1 - P, 2), dmax = (int)floor_div(P + 1, 2);
    const int D = dmax - dmin + 1, T = D * D;
    if (T > kMaxTaps) return false;
    auto dim = [&](const DimSplit &d, int &t0, int &nt, int &origin, int &out0, int &omax) {
        const int64_t q = d.in.lo, r = d.in.hi;
        t0 = (int)floor_div(q, 2);
        nt = (int)(floor_div(r - 1, 2) - t0 + 1);
        origin = (int)(t0 + dmin - d.dbuf.lo);
        out0 = (int)(2 * t0 - q);
        omax = (int)(r - q);
    };
    int t0h, nth, orh, o0h, omh, t0w, ntw, orw, o0w, omw;
    dim(rp.h, t0h, nth, orh, o0h, omh);
    dim(rp.w, t0w, ntw, orw, o0w, omw);
    if (nth <= 0 || ntw <= 0) return true;  // nothing owned
    const int64_t rows = 4 * g.Cp, kcols = (int64_t)T * g.Fp;
    ensure_alloc(pl->grave, pl->wt, pl->wt_bytes, (size_t)rows * kcols * 2);
    GemmLaunch L;
    ConvGemmParams &p = L.p;
    std::memset(&p, 0, sizeof p);
    p.bkc = pick_bkc(g.Fp);
    p.kc = (int)(g.Fp / p.bkc);
    p.bn = (int)rows;
    p.stages = pick_stages(p.bkc, p.bn);
    p.T = T;
    for (int t = 0; t < T; ++t) p.tap_h[t] = (int8_t)(t / D), p.tap_w[t] = (int8_t)(t % D);
    p.s_in = 1;
    p.origin_h = orh, p.origin_w = orw;
    p.out = reinterpret_cast<__nv_bfloat16 *>(dx);
    p.out_sn = dxd.stride_n, p.out_sh = dxd.stride_h, p.out_sw = dxd.stride_w;
    p.out_h0 = o0h, p.out_w0 = o0w, p.out_dh = 2, p.out_dw = 2;
    p.nout_p = (int)rows;
    L.nout_tiles = 1;
    L.subpix = 1, L.sub_cp = (int)g.Cp, L.out_hmax = omh, L.out_wmax = omw;
    L.w_base = pl->wt, L.w_rows = rows, L.w_kcols = kcols;
    L.cin = g.Fp;
    weight_map(&L.bmap, pl->wt, rows, kcols, p.bkc, p.bn);
    L.ksplit = 1;  // (the split-K reduce has no sub-pixel mapping)
    L.work_hint = ceil_div(g.N * ceil_div(ceil_div(g.H, 2), kV2TH) * ceil_div(ceil_div(g.W, 2), kV2TW),
                           (int64_t)pl->splitk_world());
    if ((flags & DC_EXCHANGE) && (!rp.dy_send.empty() || !rp.dy_recv.empty())) {
        exchange(pl, 1, dy, flags, st);
        *exchanged = true;
    }
    launch_subpix_weights(reinterpret_cast<const __nv_bfloat16 *>(w), pl->wt, (int)g.F, (int)g.Fp, (int)g.C,
                          (int)g.Cp, K, P, dmin, D, st);
    const std::vector<OutRect> whole_rect{OutRect{0, 0, nth, ntw}};
    return launch_v2_shape(L, whole_rect, 3, dy, dyd, g.Fp, (int)rp.nrange.size(), st);
}

// 1x1 stride 2 (bf16, no padding): of the four stride phases one holds the
// tap and three only zeros. The tap's GEMM runs flattened over the whole dy
// buffer into a dense temporary, then one pass writes dx (the products at the
// even positions, zeros elsewhere) -- instead of four phase launches, three of
// them zero-weight GEMMs. False: not applicable (dy window != dy buffer).
bool run_bwd_data_sub2(dc_plan_s *pl, const std::vector<Phase> &ph, std::vector<GemmLaunch> &L, void *dy,
                       const dc_shard_desc_t &dyd, const dc_shard_desc_t &dxd, void *dx, int64_t kc,
                       cudaStream_t st) {
    const ConvGeom &g = pl->rp.g;
    if (!(g.K == 1 && g.S == 2 && g.P == 0 && g.dt == 0 && !pl->scat_seg) || ph.size() != 4) return false;
    const Phase &f = ph[0];
    if (!f.active || f.T != 1 || ph[1].T || ph[2].T || ph[3].T || L[0].scat_seg) return false;
    if (f.origin_h != 0 || f.origin_w != 0 || f.nt_h != dyd.hb || f.nt_w != dyd.wb || dyd.halo_n || dyd.halo_s ||
        dyd.halo_w || dyd.halo_e || dyd.n * dyd.hb * dyd.wb >= (int64_t(1) << 31))
        return false;
    GemmLaunch &G = L[0];
    if (G.interior.size() + G.boundary.size() != 1) return false;
    ensure_alloc(pl->grave, pl->xsub, pl->xsub_bytes, (size_t)(dyd.n * f.nt_h * f.nt_w * g.Cp * 2));
    G.p.out = reinterpret_cast<__nv_bfloat16 *>(pl->xsub);
    G.p.out_sw = g.Cp, G.p.out_sh = f.nt_w * g.Cp, G.p.out_sn = f.nt_h * f.nt_w * g.Cp;
    G.p.out_h0 = 0, G.p.out_w0 = 0, G.p.out_dh = 1, G.p.out_dw = 1;
    G.flat = true;
    launch_rects(G, {whole(G)}, dy, dyd, kc, (int)pl->rp.nrange.size(), st);
    launch_scatter2(pl->xsub, dyd.n, f.nt_h, f.nt_w, (int)(g.Cp * 2), f.out_h0, f.out_w0, dxd.h, dxd.w, dx, st);
    return true;
}

void run_bwd_data(dc_plan_s *pl, void *dy, const void *w, void *dx, unsigned flags,
                  cudaStream_t st) {
    bool exchanged = false;
    if (run_bwd_data_subpix(pl, dy, w, dx, flags, st, &exchanged)) return;
    if (exchanged) flags &= ~DC_EXCHANGE;  // (the sub-pixel launch did not configure)
    const RankPlan &rp = pl->rp;
    const ConvGeom &g = rp.g;
    const dc_shard_desc_t dyd = describe(rp, DC_DY), dxd = describe(rp, DC_DX);
    const int S = g.S;
    // K per tap of a phase GEMM in 16-bit units: F_pad bf16, or the 3xTF32
    // [w_hi | w_lo | w_hi] fp32 segments against dy's [hi | lo] (tf32.cuh)
    const bool f32 = g.dt == 1;
    const int64_t kc = f32 ? 6 * g.Fp : g.Fp;
    // per-phase weights: [Cp][T][kc] each (16-bit units), at increasing offsets
    std::vector<Phase> ph;
    size_t wt_need = 0;
    for (int rh = 0; rh < S; ++rh)
        for (int rw = 0; rw < S; ++rw) {
            DimPhase a = dim_phase(rp.h, g.K, S, g.P, rh), b = dim_phase(rp.w, g.K, S, g.P, rw);
            Phase f;
            f.active = a.nt > 0 && b.nt > 0;
            f.T = a.M * b.M;
            for (int mh = 0; mh < a.M; ++mh)
                for (int mw = 0; mw < b.M; ++mw) {
                    const int t = mh * b.M + mw;
                    f.tap_h[t] = (int8_t)mh;
                    f.tap_w[t] = (int8_t)mw;
                    f.ka[t] = (int8_t)(a.a0 + S * (a.M - 1 - mh));
                    f.kb[t] = (int8_t)(b.a0 + S * (b.M - 1 - mw));
                }
            f.origin_h = a.origin, f.origin_w = b.origin;
            f.out_h0 = a.out0, f.out_w0 = b.out0;
            f.nt_h = a.nt, f.nt_w = b.nt;
            f.bl = a.bl, f.bh = a.bh, f.bwl = b.bl, f.bwh = b.bh;
            ph.push_back(f);
            wt_need += (size_t)g.Cp * std::max(f.T, 1) * kc * 2;
        }
    ensure_alloc(pl->grave, pl->wt, pl->wt_bytes, wt_need);
    {   // the rotated / transposed weights of every active phase in one launch
        int8_t ka[kMaxTaps], kb[kMaxTaps];
        int Ts[kMaxTaps], ts[kMaxTaps];
        long long offs[kMaxTaps];
        int nt = 0;
        size_t o = 0;
        for (auto &f : ph) {
            if (f.active)
                for (int t = 0; t < f.T; ++t) {
                    ka[nt] = f.ka[t], kb[nt] = f.kb[t], Ts[nt] = f.T, ts[nt] = t,
                    offs[nt] = (long long)(o / (f32 ? 4 : 2));  // in elements
                    ++nt;
                }
            o += (size_t)g.Cp * std::max(f.T, 1) * kc * 2;
        }
        if (f32)
            launch_weight_transform_tf32(reinterpret_cast<const float *>(w), reinterpret_cast<float *>(pl->wt),
                                         (int)g.F, (int)g.Fp, (int)g.C, (int)g.Cp, g.K, nt, ka, kb, Ts, ts, offs, st);
        else
            launch_weight_transform_multi(reinterpret_cast<const __nv_bfloat16 *>(w), pl->wt, (int)g.F, (int)g.Fp,
                                          (int)g.C, (int)g.Cp, g.K, nt, ka, kb, Ts, ts, offs, st);
    }
    std::vector<GemmLaunch> L(ph.size());
    size_t off = 0;
    for (size_t i = 0; i < ph.size(); ++i) {
        Phase &f = ph[i];
        __nv_bfloat16 *wt = pl->wt + off / 2;
        off += (size_t)g.Cp * std::max(f.T, 1) * kc * 2;
        if (!f.active) continue;
        ConvGemmParams &p = L[i].p;
        std::memset(&p, 0, sizeof p);
        L[i].cin = kc;
        if (f32) L[i].kind = 1, L[i].a_seg = (int)(2 * g.Fp), L[i].a_cvirt = 4 * g.Fp, L[i].out_f32 = true;
        p.bkc = pick_bkc(kc);
        p.kc = (int)(kc / p.bkc);
        p.bn = pick_bn(g.Cp);
        p.stages = pick_stages(p.bkc, p.bn);
        p.T = f.T;
        std::memcpy(p.tap_h, f.tap_h, sizeof p.tap_h);
        std::memcpy(p.tap_w, f.tap_w, sizeof p.tap_w);
        p.s_in = 1;
        p.origin_h = f.origin_h, p.origin_w = f.origin_w;
        p.out = reinterpret_cast<__nv_bfloat16 *>(dx);
        p.out_sn = dxd.stride_n, p.out_sh = dxd.stride_h, p.out_sw = dxd.stride_w;
        p.out_h0 = f.out_h0, p.out_w0 = f.out_w0, p.out_dh = S, p.out_dw = S;
        p.nout_p = (int)g.Cp;
        L[i].nout_tiles = (int)ceil_div(g.Cp, p.bn);
        weight_map(&L[i].bmap, wt, g.Cp, (int64_t)std::max(f.T, 1) * kc, p.bkc, p.bn);
        L[i].w_base = wt, L[i].w_rows = g.Cp, L[i].w_kcols = (int64_t)std::max(f.T, 1) * kc;
        Split2D s{f.nt_h, f.nt_w, f.bl, f.bh, f.bwl, f.bwh};
        make_rects(s, L[i].interior, L[i].boundary);
        L[i].work_hint = ceil_div(g.N * ceil_div(ceil_div(g.H, S), kV2TH) * ceil_div(ceil_div(g.W, S), kV2TW) *
                                      L[i].nout_tiles,
                                  (int64_t)pl->splitk_world());
        L[i].ksplit = choose_ksplit(L[i].work_hint, kc);
        apply_scatter(pl, L[i]);
        L[i].flat = S == 1 && flat_ok(g, dyd) && L[i].interior.size() + L[i].boundary.size() == 1;
    }
    // one split-K workspace region per phase: the phases' interior and
    // boundary launches may run concurrently on two streams
    size_t ks_need = 0;
    std::vector<size_t> ks_off(ph.size(), 0);
    for (size_t i = 0; i < ph.size(); ++i)
        if (ph[i].active) {
            ks_off[i] = ks_need;
            ks_need += ksplit_bytes(L[i], (int)rp.nrange.size());
        }
    ensure_alloc(pl->grave, pl->ws2, pl->ws2_bytes, ks_need);
    for (size_t i = 0; i < ph.size(); ++i)
        if (ph[i].active && L[i].ksplit > 1) {
            const OutRect b = whole(L[i]);
            L[i].ws_h = b.nh, L[i].ws_w = b.nw, L[i].ws = pl->ws2 + ks_off[i] / sizeof(float);
        }
    if (run_bwd_data_sub2(pl, ph, L, dy, dyd, dxd, dx, kc, st)) return;
    const bool need_dy = (flags & DC_EXCHANGE) && (!rp.dy_send.empty() || !rp.dy_recv.empty());
    const bool overlap = need_dy && !(flags & DC_NO_OVERLAP) &&
                         ((flags & DC_FORCE_OVERLAP) || halo_recv_bytes(pl, 1) >= kOverlapMinHaloBytes);
    if (need_dy && !overlap) exchange(pl, 1, dy, flags, st);  // exchange, then compute
    if (overlap) {
        CK(cudaEventRecord(pl->ev[0], st));
        CK(cudaStreamWaitEvent(pl->s_comm, pl->ev[0], 0));
        exchange(pl, 1, dy, flags, pl->s_comm);
    }
    int nactive = 0;
    for (auto &f : ph) nactive += f.active ? 1 : 0;
    if (!overlap && nactive > 1 && pl->s_ph[0]) {
        // stride phases are independent GEMMs with disjoint outputs and split-K
        // workspaces: one stream each, so their ramp-up / tail / reduce overlap
        // (running them side by side on tap-proportional SM shares, so that
        // they would sweep dy together and share its L2 lines, was measured
        // slower in round 2: conv2_1 backward-data 0.68 -> 1.36 ms, conv3_1
        // 0.40 -> 0.56 ms, conv4_1 0.34 -> 0.46 ms)
        CK(cudaEventRecord(pl->ev_ph[0], st));
        int k = 0;
        for (size_t i = 0; i < ph.size(); ++i) {
            if (!ph[i].active) continue;
            cudaStream_t sp = pl->s_ph[k];
            CK(cudaStreamWaitEvent(sp, pl->ev_ph[0], 0));
            launch_rects(L[i], {whole(L[i])}, dy, dyd, kc, (int)rp.nrange.size(), sp);
            CK(cudaEventRecord(pl->ev_ph[1 + k], sp));
            ++k;
        }
        for (int j = 0; j < k; ++j) CK(cudaStreamWaitEvent(st, pl->ev_ph[1 + j], 0));
        return;
    }
    for (size_t i = 0; i < ph.size(); ++i) {
        if (!ph[i].active) continue;
        std::vector<OutRect> rects = overlap ? L[i].interior : std::vector<OutRect>{whole(L[i])};
        launch_rects(L[i], rects, dy, dyd, kc, (int)rp.nrange.size(), st);
    }
    if (overlap) {  // boundary tiles on the comm stream after the exchange, joined
        for (size_t i = 0; i < ph.size(); ++i)
            if (ph[i].active)
                launch_rects(L[i], L[i].boundary, dy, dyd, kc, (int)rp.nrange.size(), pl->s_comm);
        CK(cudaEventRecord(pl->ev[1], pl->s_comm));
        CK(cudaStreamWaitEvent(st, pl->ev[1], 0));
    }
}

// ---------------------------------------------------------------------------
// backward-filter
// ---------------------------------------------------------------------------
// Split-K factor of the tile-reuse wgrad kernel from a small cost model:
// a CTA spends max(MMA issue, TMA bytes at its share of L2 bandwidth) per
// 8x8 pixel block (MMA 128xNx16 ~ 27 + 0.41 N cycles, measured with
// tools/mbar_bench.cu), CTAs beyond one per SM run in further waves, and every
// split costs one more fp32 partial of dW written and read back by the reduce.
// Returns the split count; *atomic tells whether the splits should add into dW
// with fp32 reductions (allowed unless DC_DETERMINISTIC) rather than through
// partials + the fixed-order reduce launch, whichever the model finds cheaper.
int wgrad_splits(const WgradV2Params &q, int ctas, long long per_split, bool allow_atomic, bool *atomic) {
    const int sms = device_sm_count();
    const int nks = q.kind == 1 ? 8 : q.bw / 2;  // MMAs per block and M tile (K = 8 tf32 / 16 bf16)
    const double mma_ns = nks * q.G * (27.0 + 0.41 * q.bn) / 1.9;
    const double stage_bytes = q.x_stage_bytes + q.dy_stage_bytes;
    const double sm_gbs = 40.0;  // (re-swept in round 2: 25 / 60 / 100 no better, tools/gbs_sweep.sh)
    int best = 1;
    bool best_atomic = false;
    double best_t = 1e30;
    for (int s = 1; s <= std::min(q.nblocks, 256); ++s) {
        if ((size_t)s * per_split * 4 > ((size_t)1 << 30)) break;
        const long long active = std::min<long long>((long long)ctas * s, sms);
        // per-SM ingest: measured 45-60 GB/s on the TMA-fed wgrad_v2 (stride-2
        // conv2_1 at 64 CTAs: 1.66 GB in 577 us; conv1_1 at 80 CTAs: 3.49 GB in
        // 731 us, profiles/r1_wgrad_s2_n8.txt), so memory-heavy layers need all
        // SMs; the whole GPU caps at ~7 TB/s
        const double bw = std::min(sm_gbs, 7000.0 / (double)active);  // GB/s = bytes/ns per SM
        const double blk_ns = std::max(mma_ns, stage_bytes / bw);
        const long long waves = ceil_div((long long)ctas * s, (long long)sms);
        const double t0 = (double)waves * (double)ceil_div((long long)q.nblocks, (long long)s) * blk_ns;
        // partials written + read by the reduce launch (HBM), or fp32 reductions
        // in L2 (~1.5 TB/s effective, measured on 9.4 MB dW) after a memset
        const double t_red = s > 1 ? 2.0 * s * 4.0 * (double)per_split / 6500.0 + 3000.0 : 0.0;
        const double t_atm = s > 1 ? s * 4.0 * (double)per_split / 1500.0 + 1000.0 : 0.0;
        // measured: atomics win for small dW (conv1_2 129 -> 109 us, its quarter
        // shard 64 -> 50 us) and lose for the 9.4 MB dW of the 512-channel
        // layers (49 -> 56 us), where the model's two estimates are too close
        // to call -- decide by size, count splits with the reduce model
        const bool use_atm = allow_atomic && s > 1 && per_split < (1LL << 20);
        (void)t_atm;
        const double t = t0 + t_red;
        if (t < best_t * 0.97) best_t = t, best = s, best_atomic = use_atm;
    }
    *atomic = best_atomic;
    return best;
}

void run_bwd_filter(dc_plan_s *pl, const void *x, const void *dy, float *dw, cudaStream_t st,
                    bool allow_atomic) {
    const RankPlan &rp = pl->rp;
    const ConvGeom &g = rp.g;
    const dc_shard_desc_t xd = describe(rp, DC_X), dyd = describe(rp, DC_DY);
    const int64_t ho = rp.h.out.size(), wo = rp.w.out.size(), nl = rp.nrange.size();
    const bool f32 = g.dt == 1;
    const int esz = g.esz();
    // dy WITHOUT its halo: maps over the owned block only
    const void *dy_owned = reinterpret_cast<const uint8_t *>(dy) +
                           (size_t)(dyd.halo_n * dyd.wb + dyd.halo_w) * dyd.c_pad * esz;
    if (f32 || g.Fp % 64 == 0) {
        // tile-reuse kernel (wgrad_v2.cu)
        WgradV2Params q;
        std::memset(&q, 0, sizeof q);
        q.kind = f32 ? 1 : 0;
        q.s_in = g.S;
        q.origin_h = (int)(g.S * rp.h.out.lo - g.P - rp.h.xbuf.lo);
        q.origin_w = (int)(g.S * rp.w.out.lo - g.P - rp.w.xbuf.lo);
        q.kh = q.kw = g.K;
        q.T = g.K * g.K;
        q.F = (int)g.F, q.Fp = (int)g.Fp, q.cp = (int)g.Cp;
        q.pixels_hint = nl * ho * wo;
        if (wgrad_v2_configure(q, kV2SmemLimit)) {
            q.tiles_h = (int)ceil_div(ho, 8);
            q.tiles_w = (int)ceil_div(wo, (int64_t)q.bw);
            // 3xTF32: three passes over the pixel blocks, one accumulation
            // (x_hi dy_hi, x_hi dy_lo, x_lo dy_hi; the lo halves sit Cp / Fp
            // channels after the hi halves in the [hi | lo] buffers)
            q.passes = f32 ? 3 : 1;
            q.nblocks_pix = (int)(nl * q.tiles_h * q.tiles_w);
            q.nblocks = q.passes * q.nblocks_pix;
            q.x_lo = (int)g.Cp, q.dy_lo = (int)g.Fp;
            const int mgroups = wgrad_v2_mgroups(q), ntiles = (int)ceil_div(g.Fp, q.bn);
            const long long per_split = (long long)g.F * q.T * g.C;  // dW: [F][K][K][C]
            const long long split_stride = round_up(per_split, 4);
            q.C = (int)g.C;
            bool atomic = false;
            const int splits = wgrad_splits(q, mgroups * ntiles, split_stride, allow_atomic, &atomic);
            q.splits = splits;
            q.ws_split = split_stride;
            if (splits > 1 && atomic) {
                // splits accumulate into the zeroed dW (no partials, no reduce
                // launch); fp32 addition order varies run to run (DC_DW_ATOMIC)
                CK(cudaMemsetAsync(dw, 0, (size_t)per_split * 4, st));
                q.ws = dw, q.ws_split = 0, q.atomic_out = 1;
            } else if (splits > 1) {
                ensure_alloc(pl->grave, pl->ws, pl->ws_bytes, (size_t)splits * split_stride * 4);
                q.ws = pl->ws;
            } else {
                q.ws = dw;
            }
            CUtensorMap xmap, dymap;
            const int64_t xc = xd.c_pad, fc = dyd.c_pad;  // elements per pixel of the buffers
            const uint64_t xdims[4] = {(uint64_t)xc, (uint64_t)xd.wb, (uint64_t)xd.hb, (uint64_t)xd.n};
            const uint64_t xstr[3] = {(uint64_t)(xc * esz), (uint64_t)(xd.wb * xc * esz),
                                      (uint64_t)(xd.hb * xd.wb * xc * esz)};
            const uint32_t xbox[4] = {(uint32_t)q.cgw, (uint32_t)(q.pitch * g.S), (uint32_t)q.PH, 1};
            const uint32_t xes[4] = {1, (uint32_t)g.S, 1, 1};
            const uint64_t ddims[4] = {(uint64_t)fc, (uint64_t)wo, (uint64_t)ho, (uint64_t)nl};
            const uint64_t dstr[3] = {(uint64_t)(fc * esz), (uint64_t)(dyd.wb * fc * esz),
                                      (uint64_t)(dyd.hb * dyd.wb * fc * esz)};
            const uint32_t dbox[4] = {(uint32_t)(128 / esz), (uint32_t)q.bw, 8, 1};
            if (f32) {  // MN-major tf32 operands: 128-byte rows, 32-byte-granule swizzle
                make_tmap_ex(&xmap, x, 4, xdims, xstr, xbox, xes, CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                             CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
                make_tmap_ex(&dymap, dy_owned, 4, ddims, dstr, dbox, nullptr, CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                             CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
            } else {
                make_tmap(&xmap, x, 4, xdims, xstr, xbox, xes, q.cgw * 2);
                make_tmap(&dymap, dy_owned, 4, ddims, dstr, dbox, nullptr, 128);
            }
            launch_wgrad_v2(xmap, dymap, q, st);
            if (splits > 1 && !q.atomic_out) launch_splitk_reduce(pl->ws, splits, per_split, split_stride, dw, st);
            return;
        }
    }
    DC_REQUIRE(!f32, DC_ERR_UNSUPPORTED, "3xTF32 backward-filter: the tile-reuse kernel does not fit this layer");
    WgradParams p;
    std::memset(&p, 0, sizeof p);
    p.T = g.K * g.K;
    p.bkc = pick_bkc(g.Cp);
    p.kc = (int)(g.Cp / p.bkc);
    p.pairs_total = p.T * p.kc;
    p.bf = g.Fp % 64 == 0 ? 64 : g.Fp % 32 == 0 ? 32 : 16;
    p.bn = g.Fp <= 256 ? (int)g.Fp : 256;
    p.stages = 4;
    for (int a = 0; a < g.K; ++a)
        for (int b = 0; b < g.K; ++b) {
            p.tap_h[a * g.K + b] = (int8_t)a;
            p.tap_w[a * g.K + b] = (int8_t)b;
        }
    p.s_in = g.S;
    p.origin_h = (int)(g.S * rp.h.out.lo - g.P - rp.h.xbuf.lo);
    p.origin_w = (int)(g.S * rp.w.out.lo - g.P - rp.w.xbuf.lo);
    p.tw_log2 = pick_twl(ho, wo, 64);
    const int tw = 1 << p.tw_log2, th = 64 >> p.tw_log2;
    p.tiles_h = (int)ceil_div(ho, th);
    p.tiles_w = (int)ceil_div(wo, tw);
    p.nblocks = (int)(nl * p.tiles_h * p.tiles_w);
    const int ppm = 128 / p.bkc;
    const int m_tiles = (int)ceil_div(p.pairs_total, ppm);
    const int n_tiles = (int)ceil_div(g.F, p.bn);
    const long long per_split = (long long)g.F * p.T * g.C;  // dW: [F][K][K][C]
    const long long split_stride = round_up(per_split, 4);
    int splits = (int)ceil_div(296, (int64_t)m_tiles * n_tiles);
    splits = std::max(1, std::min(splits, std::max(1, p.nblocks / 4)));
    while (splits > 1 && (size_t)splits * split_stride * 4 > ((size_t)1 << 30)) --splits;
    p.splits = splits;
    p.F = (int)g.F;
    p.cp = (int)g.Cp;
    p.C = (int)g.C;
    p.ws_split = split_stride;
    if (splits > 1) {
        ensure_alloc(pl->grave, pl->ws, pl->ws_bytes, (size_t)splits * split_stride * 4);
        p.ws = pl->ws;
    } else {
        p.ws = dw;
    }
    CUtensorMap xmap, dymap;
    nhwc_map(&xmap, x, xd.n, xd.hb, xd.wb, g.Cp, xd.wb, xd.hb * xd.wb, p.bkc, tw, th, g.S);
    // dy WITHOUT its halo: a map over the owned block only
    nhwc_map(&dymap, dy_owned, nl, ho, wo, g.Fp, dyd.wb, dyd.hb * dyd.wb, p.bf, tw, th, 1);
    launch_wgrad(xmap, dymap, p, m_tiles, n_tiles, st);
    if (splits > 1) launch_splitk_reduce(pl->ws, splits, per_split, split_stride, dw, st);
}

// Early "ready" signal (P2P halo protocol): after the last consumer of a
// margined buffer (x: backward-filter, retention contract; dy: backward-data),
// tell the neighbours that send into it that the next epoch may be written, so
// the next exchange does not wait for a handshake. The exchange kernel also
// signals ready for its own epoch, so this is an optimisation, never required.
void signal_ready_next(dc_plan_s *pl, int which, const void *buf, cudaStream_t st) {
    if (pl->is_virtual || pl->world() <= 1 || g_dry_run) return;
    const BufState &B = pl->buf[which];
    if (B.ptr != buf) return;  // the P2P protocol applies to dc_buffer_alloc buffers only
    resolve_local_peers(pl);
    if (pl->peer_flags.empty()) return;
    const auto &recvs = which == 0 ? pl->rp.x_recv : pl->rp.dy_recv;
    if (recvs.empty()) return;
    std::vector<uint32_t *> fl;
    for (auto &m : recvs) fl.push_back(pl->flag(pl->peer_flags.at(m.peer), which, FLAG_READY, pl->rp.rank));
    launch_signal(fl.data(), (int)fl.size(), 0, B.dev_epoch, st);
}

void allreduce_dw(dc_plan_s *pl, float *dw, cudaStream_t st) {
    if (pl->world() <= 1) return;
    DC_REQUIRE(!is_local(pl), DC_ERR_UNSUPPORTED, "dW allreduce needs real ranks (loopback group: DC_ALLREDUCE off)");
    DC_REQUIRE(pl->nccl() != nullptr, DC_ERR_ARG, "allreduce needs a communicator");
    const ConvGeom &g = pl->rp.g;
    NK(ncclAllReduce(dw, dw, (size_t)g.F * g.K * g.K * g.C, ncclFloat32, ncclSum, pl->nccl(), st));
}

// DC_ALLREDUCE_ASYNC: the allreduce waits for the work queued on `st` so far
// (the filter gradient) and runs on the communicator's gradient stream; `st`
// does not wait for it (dc_comm_sync joins).
// Issue the collected bucket: s_grad waits for everything queued on `st` so
// far (those layers' filter gradients), then one grouped NCCL call.
void flush_bucket(dc_comm_s *c, cudaStream_t st) {
    if (c->bucket.empty()) return;
    CK(cudaEventRecord(c->ev_in, st));
    CK(cudaStreamWaitEvent(c->s_grad, c->ev_in, 0));
    NK(ncclGroupStart());
    for (auto &b : c->bucket) NK(ncclAllReduce(b.first, b.first, b.second, ncclFloat32, ncclSum, c->grad_nccl, c->s_grad));
    NK(ncclGroupEnd());
    c->bucket.clear();
    c->bucket_bytes = 0;
    c->grad_pending = true;
}

void allreduce_dw_async(dc_plan_s *pl, float *dw, cudaStream_t st) {
    if (pl->world() <= 1) return;
    DC_REQUIRE(!is_local(pl), DC_ERR_UNSUPPORTED, "dW allreduce needs real ranks (loopback group: DC_ALLREDUCE off)");
    dc_comm_s *c = pl->comm;
    DC_REQUIRE(c && c->grad_nccl, DC_ERR_ARG, "allreduce needs a communicator");
    const ConvGeom &g = pl->rp.g;
    const size_t n = (size_t)g.F * g.K * g.K * g.C;
    c->bucket.emplace_back(dw, n);
    c->bucket_bytes += n * 4;
    if (c->bucket_bytes >= c->bucket_cap) flush_bucket(c, st);
}

// Streams, events and small scratch of this rank (created lazily for virtual
// plans, which may compute when no exchange / allreduce is requested).
void ensure_local_resources(dc_plan_s *pl) {
    if (pl->s_comm) return;
    if (pl->comm && pl->comm->group) {
        // loopback: the rank's side stream, no phase streams (phases run one
        // after another): no extra hardware queues shared between ranks
        pl->s_comm = pl->comm->s_side;
        pl->s_comm_shared = true;
    } else if (pl->comm && pl->comm->s_side) {  // the communicator's shared set
        pl->s_comm = pl->comm->s_side;
        for (int k = 0; k < 4; ++k) pl->s_ph[k] = pl->comm->s_ph[k];
        pl->s_copy = pl->comm->s_copy;
        pl->s_comm_shared = true;
    } else {
        CK(cudaStreamCreateWithFlags(&pl->s_comm, cudaStreamNonBlocking));
        for (auto &sp : pl->s_ph) CK(cudaStreamCreateWithFlags(&sp, cudaStreamNonBlocking));
    }
    for (auto &e : pl->ev) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto &e : pl->ev_ph) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK(cudaMalloc(&pl->bn_sums, sizeof(double) * 4 * pl->rp.g.Fp));  // local sums, global sums
}

// Make `st` wait for a DC_IMPORT_ASYNC import into buffer `which` (0: x, 1: dy).
void join_import(dc_plan_s *pl, int which, cudaStream_t st) {
    if (!pl->import_pending[which]) return;
    CK(cudaStreamWaitEvent(st, pl->ev_copy_out[which], 0));
    pl->import_pending[which] = false;
}

// Size every workspace of a plan once at creation: a dry run of the host-side
// configuration of each compute call (g_dry_run: nothing is launched), so no
// compute call needs cudaMalloc later -- cudaMalloc can wait for the device,
// which must not happen while this rank's (or, in a loopback group, another
// virtual rank's) halo / BN kernels spin for a peer, nor in a timed step.
void presize(dc_plan_s *pl) {
    struct Scope {
        Scope() { g_dry_run = true; }
        ~Scope() { g_dry_run = false; }
    } dry;
    void *d = nullptr;  // any 16-byte aligned device address: TMA maps are encoded, never used
    CK(cudaMalloc(&d, 4096));
    cudaStream_t s = pl->s_comm;
    const dc_status_t r1 = dc_conv_fwd(pl, d, d, d, DC_BN_STATS, s);
    const dc_status_t r2 = dc_conv_bwd_data(pl, d, d, d, 0, s);
    const dc_status_t r3 = dc_conv_bwd_filter(pl, d, d, reinterpret_cast<float *>(d), 0, s);
    const dc_status_t r4 = dc_bn_spatial_stats(pl, d, reinterpret_cast<double *>(d), reinterpret_cast<double *>(d),
                                              DC_BN_LOCAL, s);
    double *dd = reinterpret_cast<double *>(d);
    float *df = reinterpret_cast<float *>(d);
    const dc_status_t r5 = dc_bn_backward(pl, d, d, dd, dd, df, df, 1e-5, nullptr, DC_BN_LOCAL, nullptr, nullptr,
                                          nullptr, d, s);
    CK(cudaFree(d));
    pl->fwd_epoch = 0, pl->bn_fused_epoch = 0, pl->bn_fused_y = nullptr, pl->bn_fused_slots = 0;
    DC_REQUIRE(r1 == DC_OK && r2 == DC_OK && r3 == DC_OK && r4 == DC_OK && r5 == DC_OK, DC_ERR_UNSUPPORTED,
               "layer not supported by the kernels (%d %d %d %d %d): %s", (int)r1, (int)r2, (int)r3, (int)r4,
               (int)r5, dc_last_error());
}

dc_plan_s *create_plan(const ConvGeom &g, Grid grid, int rank, dc_comm_s *comm, bool is_virtual) {
    auto *pl = new dc_plan_s();
    try {
        pl->rp = make_rank_plan(g, grid, rank);
        pl->comm = comm;
        pl->is_virtual = is_virtual;
        pl->bn_group = grid.ph * grid.pw;  // BN group: ranks with equal i_N
        if (!is_virtual) {
            pl->seq = comm ? comm->plan_seq++ : 0;
            ensure_local_resources(pl);
            if (grid.size() > 1) {
                const bool local = comm->group != nullptr;
                if (pl->bn_group > 1 && !local) {
                    if (grid.pn == 1) {
                        pl->bn_comm = comm->nccl;
                    } else {
                        NK(ncclCommSplit(comm->nccl, pl->rp.in, rank, &pl->bn_comm, nullptr));
                        pl->bn_comm_owned = true;
                    }
                }
                // P2P flags, mapped into the neighbours
                const size_t fb = sizeof(uint32_t) * 4 * grid.size();
                CK(cudaMalloc(&pl->flags, fb));
                CK(cudaMemset(pl->flags, 0, fb));
                CK(cudaMalloc(&pl->dev_epochs, sizeof(uint32_t) * 4));
                CK(cudaMemset(pl->dev_epochs, 0, sizeof(uint32_t) * 4));
                pl->buf[0].dev_epoch = pl->dev_epochs;
                pl->buf[1].dev_epoch = pl->dev_epochs + 2;
                // the BN group's one-shot NVLink mailbox (<= 8 members; NCCL beyond)
                const int gsz = pl->bn_group;
                if (gsz > 1 && gsz <= kMaxBnGroup) {
                    const size_t bytes = 256 + (size_t)2 * gsz * 2 * g.Fp * sizeof(double);
                    CK(cudaMalloc(&pl->bn_mail, bytes));
                    CK(cudaMemset(pl->bn_mail, 0, bytes));
                    CK(cudaMalloc(&pl->bn_epoch, sizeof(uint32_t)));
                    CK(cudaMemset(pl->bn_epoch, 0, sizeof(uint32_t)));
                    pl->bn_p2p = true;
                    pl->bn_peer_mail.assign(gsz, nullptr);
                    pl->bn_peer_mail[rank - pl->rp.in * gsz] = pl->bn_mail;
                }
                if (local) {
                    std::lock_guard<std::mutex> lk(comm->group->mu);
                    comm->group->plans[{pl->seq, rank}] = pl;
                } else {
                    struct Handles {
                        cudaIpcMemHandle_t flags, bn;
                    } h{};
                    CK(cudaIpcGetMemHandle(&h.flags, pl->flags));
                    if (pl->bn_p2p) CK(cudaIpcGetMemHandle(&h.bn, pl->bn_mail));
                    auto all = allgather_bytes(pl, &h, sizeof h);
                    auto at = [&](int r) {
                        Handles x;
                        std::memcpy(&x, all.data() + r * sizeof x, sizeof x);
                        return x;
                    };
                    std::vector<int> nb = neighbours(pl->rp, 0);
                    for (int p : neighbours(pl->rp, 1))
                        if (std::find(nb.begin(), nb.end(), p) == nb.end()) nb.push_back(p);
                    for (int p : nb) {
                        void *ptr = nullptr;
                        CK(cudaIpcOpenMemHandle(&ptr, at(p).flags, cudaIpcMemLazyEnablePeerAccess));
                        pl->peer_flags[p] = reinterpret_cast<uint32_t *>(ptr);
                    }
                    if (pl->bn_p2p) {
                        const int lo = pl->rp.in * gsz;
                        for (int k = 0; k < gsz; ++k) {
                            if (lo + k == rank) continue;
                            void *ptr = nullptr;
                            CK(cudaIpcOpenMemHandle(&ptr, at(lo + k).bn, cudaIpcMemLazyEnablePeerAccess));
                            pl->bn_peer_mail[k] = reinterpret_cast<uint8_t *>(ptr);
                        }
                    }
                }
                CK(cudaDeviceSynchronize());
            }
            presize(pl);
        }
    } catch (...) {
        delete pl;
        throw;
    }
    return pl;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================
extern "C" {

const char *dc_last_error(void) { return g_err.c_str(); }
uint64_t dc_kernel_launches(void) { return g_launches; }

dc_status_t dc_comm_unique_id(void *uid128) {
    DC_API_BEGIN
    DC_REQUIRE(uid128 != nullptr, DC_ERR_ARG, "null uid");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    NK(ncclGetUniqueId(&id));
    std::memcpy(uid128, &id, sizeof id);
    DC_API_END
}

dc_status_t dc_comm_create(int rank, int world, const void *uid128, int device, dc_comm_t *out) {
    DC_API_BEGIN
    DC_REQUIRE(out != nullptr && world >= 1 && rank >= 0 && rank < world, DC_ERR_ARG,
               "bad rank/world (%d/%d)", rank, world);
    CK(cudaSetDevice(device));
    preload_kernels();
    auto *c = new dc_comm_s();
    c->rank = rank, c->world = world, c->device = device;
    if (world > 1) {
        DC_REQUIRE(uid128 != nullptr, DC_ERR_ARG, "world > 1 needs an NCCL unique id");
        ncclUniqueId id;
        std::memcpy(&id, uid128, sizeof id);
        ncclResult_t r = ncclCommInitRank(&c->nccl, world, id, rank);
        if (r != ncclSuccess) {
            delete c;
            fail(DC_ERR_COMM, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
        }
        NK(ncclCommSplit(c->nccl, 0, rank, &c->grad_nccl, nullptr));
        CK(cudaStreamCreateWithFlags(&c->s_grad, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&c->ev_in, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&c->ev_out, cudaEventDisableTiming));
    }
    CK(cudaStreamCreateWithFlags(&c->s_side, cudaStreamNonBlocking));
    for (auto &sp : c->s_ph) CK(cudaStreamCreateWithFlags(&sp, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&c->s_copy, cudaStreamNonBlocking));
    *out = c;
    DC_API_END
}

dc_status_t dc_comm_create_local(int world, int device, dc_comm_t *comms) {
    DC_API_BEGIN
    DC_REQUIRE(comms != nullptr && world >= 1 && world <= 64, DC_ERR_ARG, "bad loopback world %d", world);
    CK(cudaSetDevice(device));
    preload_kernels();
    // Each virtual rank's kernels must be able to run while another rank's
    // protocol kernel spins: no two ranks' streams may share one of the
    // device's hardware queues (CUDA_DEVICE_MAX_CONNECTIONS, default 8; work of
    // streams aliased onto one queue runs in order). 2 streams per rank,
    // created back to back, map to distinct queues when 2 W <= connections.
    const char *mc = std::getenv("CUDA_DEVICE_MAX_CONNECTIONS");
    const int conns = mc ? std::atoi(mc) : 8;
    DC_REQUIRE(2 * world <= conns, DC_ERR_ARG,
               "a loopback group of %d ranks needs CUDA_DEVICE_MAX_CONNECTIONS >= %d (now %d), set before CUDA "
               "initializes",
               world, 2 * world, conns);
    auto G = std::make_shared<LocalGroup>();
    G->world = world;
    for (int r = 0; r < world; ++r) {
        auto *c = new dc_comm_s();
        c->rank = r, c->world = world, c->device = device;
        c->group = G;
        CK(cudaStreamCreateWithFlags(&c->s_main, cudaStreamNonBlocking));
        CK(cudaStreamCreateWithFlags(&c->s_side, cudaStreamNonBlocking));
        comms[r] = c;
    }
    DC_API_END
}

dc_status_t dc_comm_stream(dc_comm_t c, void **stream) {
    DC_API_BEGIN
    DC_REQUIRE(c && stream, DC_ERR_ARG, "null argument");
    DC_REQUIRE(c->group != nullptr, DC_ERR_ARG, "dc_comm_stream: loopback communicators only");
    *stream = c->s_main;
    DC_API_END
}

dc_status_t dc_comm_destroy(dc_comm_t c) {
    DC_API_BEGIN
    if (c) {
        if (c->s_grad) cudaStreamSynchronize(c->s_grad);
        cudaDeviceSynchronize();
        // (the device is idle here; ncclCommAbort frees the communicator
        // without the finalize handshake ncclCommDestroy runs with the other
        // ranks, which was measured to hang the 2- and 4-rank bench teardown)
        if (c->grad_nccl) ncclCommAbort(c->grad_nccl);
        if (c->nccl) ncclCommAbort(c->nccl);
        if (c->s_grad) cudaStreamDestroy(c->s_grad);
        if (c->s_main) cudaStreamDestroy(c->s_main);
        if (c->s_side) cudaStreamDestroy(c->s_side);
        for (auto sp : c->s_ph)
            if (sp) cudaStreamDestroy(sp);
        if (c->s_copy) cudaStreamDestroy(c->s_copy);
        if (c->ev_in) cudaEventDestroy(c->ev_in);
        if (c->ev_out) cudaEventDestroy(c->ev_out);
        delete c;
    }
    DC_API_END
}

dc_status_t dc_comm_set_bucket_bytes(dc_comm_t c, size_t bytes) {
    DC_API_BEGIN
    DC_REQUIRE(c != nullptr, DC_ERR_ARG, "null communicator");
    c->bucket_cap = bytes;
    DC_API_END
}

dc_status_t dc_comm_sync(dc_comm_t c, void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(c != nullptr, DC_ERR_ARG, "null communicator");
    if (c->s_grad) flush_bucket(c, (cudaStream_t)stream);
    if (c->s_grad && c->grad_pending) {  // (nothing queued: no-op, also inside a graph capture)
        CK(cudaEventRecord(c->ev_out, c->s_grad));
        CK(cudaStreamWaitEvent((cudaStream_t)stream, c->ev_out, 0));
        c->grad_pending = false;
    }
    DC_API_END
}

dc_status_t dc_plan_create(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int K,
                           int stride, int pad, dc_decomp_t decomp, dc_dtype_t dtype,
                           dc_comm_t comm, dc_plan_t *out) {
    DC_API_BEGIN
    DC_REQUIRE(out != nullptr, DC_ERR_ARG, "null out");
    DC_REQUIRE(dtype == DC_BF16 || dtype == DC_FP32_3XTF32, DC_ERR_ARG, "unknown dtype %d", (int)dtype);
    ConvGeom g = make_geom(N, C, H, W, F, K, stride, pad, dtype == DC_FP32_3XTF32 ? 1 : 0);
    const int world = comm ? comm->world : 1, rank = comm ? comm->rank : 0;
    Grid grid{decomp.pn, decomp.ph, decomp.pw};
    double pred = 0;
    DC_REQUIRE(decomp.pn >= 0 && decomp.ph >= 0 && decomp.pw >= 0, DC_ERR_ARG, "negative grid entry");
    if (decomp.pn == 0 || decomp.ph == 0 || decomp.pw == 0) {  // zeros: the model's choice
        DC_REQUIRE(model_choose(g, world, grid, pred, grid), DC_ERR_PARTITION,
                   "no valid decomposition of %d ranks with (%d,%d,%d) fixed", world, decomp.pn, decomp.ph,
                   decomp.pw);
        // every rank ran the model on its own process-local state (cost table,
        // comm terms): check that they agree before building neighbour lists
        if (world > 1) {
            const std::array<int, 3> mine{grid.pn, grid.ph, grid.pw};
            if (comm->group) {
                std::lock_guard<std::mutex> lk(comm->group->mu);
                auto it = comm->group->grids.emplace(comm->plan_seq, mine).first;
                DC_REQUIRE(it->second == mine, DC_ERR_PARTITION,
                           "ranks chose different grids: (%d,%d,%d) here, (%d,%d,%d) on the first rank", grid.pn,
                           grid.ph, grid.pw, it->second[0], it->second[1], it->second[2]);
            } else {
                const auto all = comm_allgather(comm, mine.data(), sizeof mine);
                for (int r = 0; r < world; ++r)
                    DC_REQUIRE(std::memcmp(all.data() + r * sizeof mine, mine.data(), sizeof mine) == 0,
                               DC_ERR_PARTITION, "ranks chose different grids (rank %d differs from rank %d)", r,
                               rank);
            }
        }
    } else {
        DC_REQUIRE(grid.size() == world, DC_ERR_PARTITION, "grid (%d,%d,%d) has %d ranks, world is %d",
                   grid.pn, grid.ph, grid.pw, grid.size(), world);
    }
    dc_plan_s *pl = create_plan(g, grid, rank, comm, false);
    pl->predicted = model_layer_cost(g, grid, true);
    *out = pl;
    DC_API_END
}

dc_status_t dc_plan_create_virtual(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int K,
                                   int stride, int pad, dc_decomp_t decomp, dc_dtype_t dtype,
                                   int rank, dc_plan_t *out) {
    DC_API_BEGIN
    DC_REQUIRE(out != nullptr, DC_ERR_ARG, "null out");
    DC_REQUIRE(dtype == DC_BF16 || dtype == DC_FP32_3XTF32, DC_ERR_ARG, "unknown dtype %d", (int)dtype);
    ConvGeom g = make_geom(N, C, H, W, F, K, stride, pad, dtype == DC_FP32_3XTF32 ? 1 : 0);
    Grid grid{decomp.pn, decomp.ph, decomp.pw};
    dc_plan_s *pl = create_plan(g, grid, rank, nullptr, true);
    pl->predicted = model_layer_cost(g, grid, true);
    *out = pl;
    DC_API_END
}

dc_status_t dc_plan_query(dc_plan_t plan, dc_tensor_t t, dc_shard_desc_t *desc) {
    DC_API_BEGIN
    DC_REQUIRE(plan && desc, DC_ERR_ARG, "null argument");
    *desc = describe(plan->rp, t);
    DC_API_END
}

dc_status_t dc_plan_halo_msgs(dc_plan_t plan, dc_tensor_t t, dc_halo_msg_t *msgs, int *count) {
    DC_API_BEGIN
    DC_REQUIRE(plan && count && (t == DC_X || t == DC_DY), DC_ERR_ARG, "bad argument");
    const auto &S = t == DC_X ? plan->rp.x_send : plan->rp.dy_send;
    const auto &R = t == DC_X ? plan->rp.x_recv : plan->rp.dy_recv;
    const int n = (int)(S.size() + R.size());
    if (msgs) {
        DC_REQUIRE(*count >= n, DC_ERR_ARG, "capacity %d < %d messages", *count, n);
        int k = 0;
        for (int pass = 0; pass < 2; ++pass)
            for (auto &m : pass == 0 ? S : R)
                msgs[k++] = dc_halo_msg_t{m.peer, pass == 0 ? 1 : 0, m.rows.lo, m.rows.size(),
                                          m.cols.lo, m.cols.size()};
    }
    *count = n;
    DC_API_END
}

dc_status_t dc_plan_decomp(dc_plan_t plan, dc_decomp_t *chosen, double *predicted) {
    DC_API_BEGIN
    DC_REQUIRE(plan && chosen, DC_ERR_ARG, "null argument");
    *chosen = dc_decomp_t{plan->rp.grid.pn, plan->rp.grid.ph, plan->rp.grid.pw};
    if (predicted) *predicted = plan->predicted;
    DC_API_END
}

dc_status_t dc_plan_set_splitk_world(dc_plan_t plan, int world) {
    DC_API_BEGIN
    DC_REQUIRE(plan && world >= 0, DC_ERR_ARG, "bad argument");
    plan->ks_world = world;
    DC_API_END
}

dc_status_t dc_plan_destroy(dc_plan_t plan) {
    DC_API_BEGIN
    delete plan;
    DC_API_END
}

dc_status_t dc_buffer_alloc(dc_plan_t pl, dc_tensor_t t, void **dev_ptr) {
    DC_API_BEGIN
    DC_REQUIRE(pl && dev_ptr && (t == DC_X || t == DC_DY || t == DC_Y || t == DC_DX), DC_ERR_ARG, "bad argument");
    DC_REQUIRE(!pl->is_virtual, DC_ERR_ARG, "virtual plan has no device buffers");
    if (t == DC_Y || t == DC_DX) {  // dense: a redistribution target (mapped by dc_redist_create)
        BufState &D = pl->dense[t == DC_Y ? 0 : 1];
        DC_REQUIRE(D.ptr == nullptr, DC_ERR_ARG, "buffer already allocated for this tensor");
        const dc_shard_desc_t d = describe(pl->rp, t);
        cudaError_t e = cudaMalloc(&D.ptr, std::max<size_t>(d.bytes, 256));
        DC_REQUIRE(e == cudaSuccess, DC_ERR_OOM, "cudaMalloc(%zu): %s", d.bytes, cudaGetErrorString(e));
        D.owned = true;
        D.bytes = d.bytes;
        CK(cudaMemset(D.ptr, 0, std::max<size_t>(d.bytes, 256)));
        CK(cudaDeviceSynchronize());
        *dev_ptr = D.ptr;
        return DC_OK;
    }
    const int which = t == DC_X ? 0 : 1;
    BufState &B = pl->buf[which];
    const dc_shard_desc_t d = describe(pl->rp, t);
    DC_REQUIRE(B.ptr == nullptr, DC_ERR_ARG, "buffer already allocated for this tensor");
    cudaError_t e = cudaMalloc(&B.ptr, std::max<size_t>(d.bytes, 256));
    DC_REQUIRE(e == cudaSuccess, DC_ERR_OOM, "cudaMalloc(%zu): %s", d.bytes, cudaGetErrorString(e));
    B.owned = true;
    B.bytes = d.bytes;
    CK(cudaMemset(B.ptr, 0, std::max<size_t>(d.bytes, 256)));
    if (pl->world() > 1 && !is_local(pl)) {  // (loopback: peers resolve it from the registry)
        cudaIpcMemHandle_t h;
        CK(cudaIpcGetMemHandle(&h, B.ptr));
        auto all = allgather_bytes(pl, &h, sizeof h);
        for (int p : neighbours(pl->rp, which)) {
            cudaIpcMemHandle_t ph;
            std::memcpy(&ph, all.data() + p * sizeof ph, sizeof ph);
            void *ptr = nullptr;
            CK(cudaIpcOpenMemHandle(&ptr, ph, cudaIpcMemLazyEnablePeerAccess));
            B.peer[p] = ptr;
        }
    }
    CK(cudaDeviceSynchronize());
    *dev_ptr = B.ptr;
    DC_API_END
}

dc_status_t dc_tensor_import(dc_plan_t pl, dc_tensor_t t, const void *src, void *dst, unsigned flags,
                             void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(pl && src && dst && (t == DC_X || t == DC_DY), DC_ERR_ARG, "bad argument");
    DC_REQUIRE((flags & ~(DC_IMPORT_ASYNC | DC_SRC_BF16)) == 0, DC_ERR_ARG, "unknown import flags 0x%x", flags);
    const ConvGeom &g = pl->rp.g;
    DC_REQUIRE(!((flags & DC_SRC_BF16) && g.dt), DC_ERR_ARG, "DC_SRC_BF16 needs a DC_BF16 plan");
    NoPdlScope no_pdl(is_local(pl));
    ensure_local_resources(pl);
    const int which = t == DC_X ? 0 : 1;
    const dc_shard_desc_t d = describe(pl->rp, t);
    const int cp = (int)(g.dt ? d.c_pad / 2 : d.c_pad);
    const bool bf16_src = (flags & DC_SRC_BF16) != 0;
    const size_t src_bytes = (size_t)d.n * d.h * d.w * d.c * (bf16_src ? 2 : 4);
    cudaPointerAttributes pa{};
    CK(cudaPointerGetAttributes(&pa, src));
    const bool host = pa.type != cudaMemoryTypeDevice && pa.type != cudaMemoryTypeManaged;
    cudaStream_t st = (cudaStream_t)stream, cs = st;
    if (is_local(pl)) flags &= ~DC_IMPORT_ASYNC;  // (loopback: no extra streams)
    if (flags & DC_IMPORT_ASYNC) {  // on the copy stream, after the caller's work so far
        ensure_local_resources(pl);
        if (!pl->ev_copy_in[0]) {
            if (!pl->s_copy) CK(cudaStreamCreateWithFlags(&pl->s_copy, cudaStreamNonBlocking));
            for (int i = 0; i < 2; ++i) {
                CK(cudaEventCreateWithFlags(&pl->ev_copy_in[i], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&pl->ev_copy_out[i], cudaEventDisableTiming));
            }
        }
        cs = pl->s_copy;
        CK(cudaEventRecord(pl->ev_copy_in[which], st));
        CK(cudaStreamWaitEvent(cs, pl->ev_copy_in[which], 0));
    }
    const void *dsrc = src;
    if (host) {  // host buffer: one H2D copy into the plan's staging, then the layout kernel
        uint8_t *&sp = reinterpret_cast<uint8_t *&>(pl->stage[which]);
        ensure_alloc(pl->grave, sp, pl->stage_bytes[which], std::max<size_t>(src_bytes, 16));
        CK(cudaMemcpyAsync(sp, src, src_bytes, cudaMemcpyHostToDevice, cs));
        dsrc = sp;
    }
    launch_import(dsrc, bf16_src, dst, (int)d.n, (int)d.h, (int)d.w, (int)d.c, cp, (int)d.hb, (int)d.wb, d.halo_n,
                  d.halo_w, g.dt, cs);
    if (flags & DC_IMPORT_ASYNC) {
        CK(cudaEventRecord(pl->ev_copy_out[which], cs));
        pl->import_pending[which] = true;
    }
    DC_API_END
}

dc_status_t dc_halo_exchange(dc_plan_t pl, dc_tensor_t t, void *buf, unsigned flags, void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(pl && buf && (t == DC_X || t == DC_DY), DC_ERR_ARG, "bad argument");
    NoPdlScope no_pdl(is_local(pl));  // (loopback: ranks share the SMs)
    join_import(pl, t == DC_X ? 0 : 1, (cudaStream_t)stream);
    exchange(pl, t == DC_X ? 0 : 1, buf, flags, (cudaStream_t)stream);
    DC_API_END
}

dc_status_t dc_conv_fwd(dc_plan_t pl, void *x, const void *w, void *y, unsigned flags,
                        void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(pl && x && w && y, DC_ERR_ARG, "null argument");
    NoPdlScope no_pdl(is_local(pl));  // (loopback: ranks share the SMs)
    ensure_local_resources(pl);
    cudaStream_t st = (cudaStream_t)stream;
    join_import(pl, 0, st);
    GemmLaunch L;
    prepare_fwd(pl, x, w, y, L, st);
    pl->bn_fused_y = nullptr;
    pl->bn_fused_epoch = 0;
    ++pl->fwd_epoch;
    if (flags & DC_BN_STATS) {
        L.bn_slot_cap = 8 * device_sm_count();
        ensure_alloc(pl->grave, pl->bn_fpart, pl->bn_fpart_bytes, sizeof(double) * L.bn_slot_cap * 2 * pl->rp.g.Fp);
        L.bn_part = pl->bn_fpart;
    }
    const dc_shard_desc_t xd = describe(pl->rp, DC_X);
    const int nl = (int)pl->rp.nrange.size();
    const bool need_x = (flags & DC_EXCHANGE) && (!pl->rp.x_send.empty() || !pl->rp.x_recv.empty());
    const bool overlap = need_x && !(flags & DC_NO_OVERLAP) &&
                         ((flags & DC_FORCE_OVERLAP) || halo_recv_bytes(pl, 0) >= kOverlapMinHaloBytes);
    if (need_x && !overlap) {  // exchange, then one launch over the whole shard
        exchange(pl, 0, x, flags, st);
        launch_rects(L, {whole(L)}, x, xd, L.cin, nl, st);
    } else if (overlap) {
        CK(cudaEventRecord(pl->ev[0], st));
        CK(cudaStreamWaitEvent(pl->s_comm, pl->ev[0], 0));
        exchange(pl, 0, x, flags, pl->s_comm);
        // interior tiles on the caller's stream, concurrently with the exchange;
        // the halo-dependent boundary tiles right after it on the comm stream
        // (disjoint outputs, and disjoint split-K workspace pixels), joined below.
        // (capping the interior grid to leave SMs to the exchange measured
        // neutral at 4 GPUs with 8 or 16 reserved SMs)
        launch_rects(L, L.interior, x, xd, L.cin, nl, st);
        launch_rects(L, L.boundary, x, xd, L.cin, nl, pl->s_comm);
        CK(cudaEventRecord(pl->ev[1], pl->s_comm));
        CK(cudaStreamWaitEvent(st, pl->ev[1], 0));
    } else if (sub2_ok(pl, L, xd)) {
        // 1x1 stride 2: the pixels the filter reads gathered into a dense
        // buffer, then the flattened GEMM over them (the stride-2 tiles of the
        // tile-reuse kernel leave most rows of a 16 x 8 tile empty on 7^2-28^2
        // images and re-read every weight stage per tile)
        const dc_shard_desc_t yd = describe(pl->rp, DC_Y);
        ensure_alloc(pl->grave, pl->xsub, pl->xsub_bytes, (size_t)(yd.n * yd.h * yd.w * L.cin * 2));
        launch_subsample2(x, xd.n, xd.hb, xd.wb, (int)(L.cin * 2), L.p.origin_h, L.p.origin_w, yd.h, yd.w, pl->xsub,
                          st);
        dc_shard_desc_t f = xd;
        f.h = f.hb = yd.h, f.w = f.wb = yd.w;
        f.halo_n = f.halo_s = f.halo_w = f.halo_e = 0;
        L.p.s_in = 1, L.p.origin_h = 0, L.p.origin_w = 0;
        L.flat = true;
        launch_rects(L, {whole(L)}, pl->xsub, f, L.cin, nl, st);
    } else {
        launch_rects(L, {whole(L)}, x, xd, L.cin, nl, st);
    }
    if (L.bn_part && L.bn_ok && L.bn_slot > 0) {  // dc_bn_spatial_stats(y) reduces these
        pl->bn_fused_y = y;
        pl->bn_fused_slots = L.bn_slot;
        pl->bn_fused_epoch = pl->fwd_epoch;
    }
    DC_API_END
}

dc_status_t dc_conv_bwd_data(dc_plan_t pl, void *dy, const void *w, void *dx, unsigned flags,
                             void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(pl && dy && w && dx, DC_ERR_ARG, "null argument");
    NoPdlScope no_pdl(is_local(pl));  // (loopback: ranks share the SMs)
    ensure_local_resources(pl);
    join_import(pl, 1, (cudaStream_t)stream);
    run_bwd_data(pl, dy, w, dx, flags, (cudaStream_t)stream);
    signal_ready_next(pl, 1, dy, (cudaStream_t)stream);
    DC_API_END
}

dc_status_t dc_conv_bwd_filter(dc_plan_t pl, const void *x, const void *dy, float *dw,
                               unsigned flags, void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(pl && x && dy && dw, DC_ERR_ARG, "null argument");
    NoPdlScope no_pdl(is_local(pl));  // (loopback: ranks share the SMs)
    ensure_local_resources(pl);
    cudaStream_t st = (cudaStream_t)stream;
    join_import(pl, 0, st);
    join_import(pl, 1, st);
    run_bwd_filter(pl, x, dy, dw, st, (flags & DC_DW_ATOMIC) != 0);
    signal_ready_next(pl, 0, x, st);
    if ((flags & DC_ALLREDUCE) && (flags & DC_ALLREDUCE_ASYNC)) allreduce_dw_async(pl, dw, st);
    else if (flags & DC_ALLREDUCE) allreduce_dw(pl, dw, st);
    DC_API_END
}

dc_status_t dc_conv_bwd(dc_plan_t pl, const void *x, void *dy, const void *w, void *dx, float *dw,
                        unsigned flags, void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(pl && x && dy && w && dx && dw, DC_ERR_ARG, "null argument");
    NoPdlScope no_pdl(is_local(pl));  // (loopback: ranks share the SMs)
    ensure_local_resources(pl);
    cudaStream_t st = (cudaStream_t)stream;
    join_import(pl, 0, st);
    join_import(pl, 1, st);
    const bool halo = (flags & DC_EXCHANGE) && (!pl->rp.dy_send.empty() || !pl->rp.dy_recv.empty());
    const bool ar_async = (flags & DC_ALLREDUCE) && (flags & DC_ALLREDUCE_ASYNC) && pl->world() > 1;
    const bool ar = (flags & DC_ALLREDUCE) && pl->world() > 1 && !ar_async;
    if (halo) {  // dy halo on the comm stream, concurrent with the filter gradient
        CK(cudaEventRecord(pl->ev[0], st));
        CK(cudaStreamWaitEvent(pl->s_comm, pl->ev[0], 0));
        exchange(pl, 1, dy, flags, pl->s_comm);
        CK(cudaEventRecord(pl->ev[1], pl->s_comm));
    }
    run_bwd_filter(pl, x, dy, dw, st, (flags & DC_DW_ATOMIC) != 0);
    signal_ready_next(pl, 0, x, st);
    if (ar_async) allreduce_dw_async(pl, dw, st);
    if (ar) {  // dW allreduce on the comm stream, concurrent with the data gradient
        CK(cudaEventRecord(pl->ev[2], st));
        CK(cudaStreamWaitEvent(pl->s_comm, pl->ev[2], 0));
        allreduce_dw(pl, dw, pl->s_comm);
        CK(cudaEventRecord(pl->ev[3], pl->s_comm));
    }
    if (halo) CK(cudaStreamWaitEvent(st, pl->ev[1], 0));
    run_bwd_data(pl, dy, w, dx, flags & ~DC_EXCHANGE, st);
    signal_ready_next(pl, 1, dy, st);
    if (ar) CK(cudaStreamWaitEvent(st, pl->ev[3], 0));
    DC_API_END
}

dc_status_t dc_bn_spatial_stats(dc_plan_t pl, const void *t, double *mean, double *var, unsigned flags,
                                void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(pl && t && mean && var, DC_ERR_ARG, "null argument");
    NoPdlScope no_pdl(is_local(pl));  // (loopback: ranks share the SMs)
    DC_REQUIRE((flags & ~(DC_BN_LOCAL | DC_BN_FROM_FWD)) == 0, DC_ERR_ARG, "unknown BN flags 0x%x", flags);
    ensure_local_resources(pl);
    cudaStream_t st = (cudaStream_t)stream;
    const RankPlan &rp = pl->rp;
    const ConvGeom &g = rp.g;
    const long long npix = rp.nrange.size() * rp.h.out.size() * rp.w.out.size();
    const int nblk = g.dt ? bn_partial_blocks_f32(npix, (int)g.Fp) : bn_stats_blocks(npix, (int)g.Fp);
    ensure_alloc(pl->grave, pl->bn_part, pl->bn_part_bytes, sizeof(double) * 2 * g.Fp * nblk);
    const bool global = !(flags & DC_BN_LOCAL) && pl->bn_group > 1;
    // the partials of this plan's latest forward, if it ran with DC_BN_STATS
    // on this tensor and the caller states t is unchanged since (DC_BN_FROM_FWD);
    // consumed once. Otherwise t is read (bn.cu, bn_staged_kernel<kBnStats>).
    const bool fused = (flags & DC_BN_FROM_FWD) && pl->bn_fused_y == t && pl->bn_fused_epoch != 0 &&
                       pl->bn_fused_epoch == pl->fwd_epoch && pl->bn_fused_slots > 0;
    // single group: the reduce kernel also finalises mean/var (no allreduce between)
    if (fused) {
        launch_bn_reduce(pl->bn_fpart, pl->bn_fused_slots, (int)g.Fp, pl->bn_sums, (int)g.F, (double)npix,
                         global ? nullptr : mean, global ? nullptr : var, st);
    } else if (g.dt) {  // fp32 y (3xTF32 plans): fp64 partials per block, the same reduction
        launch_bn_partials_f32(reinterpret_cast<const float *>(t), npix, (int)g.Fp, pl->bn_part, st);
        launch_bn_reduce(pl->bn_part, nblk, (int)g.Fp, pl->bn_sums, (int)g.F, (double)npix, global ? nullptr : mean,
                         global ? nullptr : var, st);
    } else {  // bf16 y: the staged pass (bn.cu), the same reduction
        launch_bn_stats(t, npix, (int)g.Fp, pl->bn_part, nblk, st);
        launch_bn_reduce(pl->bn_part, nblk, (int)g.Fp, pl->bn_sums, (int)g.F, (double)npix, global ? nullptr : mean,
                         global ? nullptr : var, st);
    }
    pl->bn_fused_y = nullptr;
    pl->bn_fused_epoch = 0;
    if (global && pl->bn_p2p) {
        // one-shot NVLink allreduce among the ranks with this rank's i_N
        resolve_local_peers(pl);
        BnP2P b{};
        b.gsize = pl->bn_group;
        for (int k = 0; k < b.gsize; ++k) {
            DC_REQUIRE(pl->bn_peer_mail[k] != nullptr, DC_ERR_ARG, "BN mailbox of group member %d not mapped", k);
            b.peer_box[k] = reinterpret_cast<double *>(pl->bn_peer_mail[k] + 256);
            b.peer_flags[k] = reinterpret_cast<uint32_t *>(pl->bn_peer_mail[k]);
        }
        b.my_box = reinterpret_cast<const double *>(pl->bn_mail + 256);
        b.my_flags = reinterpret_cast<const uint32_t *>(pl->bn_mail);
        b.my_idx = rp.rank - rp.in * pl->bn_group;
        b.epoch = pl->bn_epoch;
        b.local = pl->bn_sums;
        b.cpad = (int)g.Fp, b.c = (int)g.F;
        b.count = (double)rp.nrange.size() * g.Ho * g.Wo;
        b.sums = pl->bn_sums + 2 * g.Fp;
        b.mean = mean, b.var = var;
        launch_bn_allreduce_p2p(b, st);
    } else if (global) {
        DC_REQUIRE(pl->bn_comm != nullptr, DC_ERR_ARG, "spatial BN statistics need a communicator");
        NK(ncclAllReduce(pl->bn_sums, pl->bn_sums, 2 * g.Fp, ncclFloat64, ncclSum, pl->bn_comm, st));
        launch_bn_finalize(pl->bn_sums, (int)g.Fp, (int)g.F, (double)rp.nrange.size() * g.Ho * g.Wo, mean,
                           var, st);
    }
    DC_API_END
}

namespace {
// Sum 2 * Fp per-channel doubles (local at `local`) over this plan's BN group
// (the ranks with this rank's i_N): the plan's NVLink mailbox,
// or NCCL; returns the device pointer of the group sums. mean / var of the
// mailbox kernel go to `mean`, `var` (scratch when the caller needs none).
const double *bn_group_sum(dc_plan_s *pl, double *local, double *mean, double *var, cudaStream_t st) {
    const RankPlan &rp = pl->rp;
    const ConvGeom &g = rp.g;
    if (pl->bn_p2p) {
        resolve_local_peers(pl);
        BnP2P b{};
        b.gsize = pl->bn_group;
        for (int k = 0; k < b.gsize; ++k) {
            DC_REQUIRE(pl->bn_peer_mail[k] != nullptr, DC_ERR_ARG, "BN mailbox of group member %d not mapped", k);
            b.peer_box[k] = reinterpret_cast<double *>(pl->bn_peer_mail[k] + 256);
            b.peer_flags[k] = reinterpret_cast<uint32_t *>(pl->bn_peer_mail[k]);
        }
        b.my_box = reinterpret_cast<const double *>(pl->bn_mail + 256);
        b.my_flags = reinterpret_cast<const uint32_t *>(pl->bn_mail);
        b.my_idx = rp.rank - rp.in * pl->bn_group;
        b.epoch = pl->bn_epoch;
        b.local = local;
        b.cpad = (int)g.Fp, b.c = (int)g.F;
        b.count = (double)rp.nrange.size() * g.Ho * g.Wo;
        b.sums = local + 2 * g.Fp;
        b.mean = mean, b.var = var;
        launch_bn_allreduce_p2p(b, st);
        return local + 2 * g.Fp;
    }
    DC_REQUIRE(pl->bn_comm != nullptr, DC_ERR_ARG, "spatial BN needs a communicator");
    NK(ncclAllReduce(local, local, 2 * g.Fp, ncclFloat64, ncclSum, pl->bn_comm, st));
    return local;
}

BnArgs bn_args(dc_plan_s *pl, const void *y, const void *res, const void *dout, bool relu) {
    const RankPlan &rp = pl->rp;
    const ConvGeom &g = rp.g;
    BnArgs a{};
    a.y = y, a.res = res, a.dout = dout, a.coef = pl->bn_coef;
    a.esz = g.esz(), a.relu = relu ? 1 : 0;
    a.n = (int)rp.nrange.size(), a.h = (int)rp.h.out.size(), a.w = (int)rp.w.out.size();
    a.npix = (long long)a.n * a.h * a.w;
    a.cpad = (int)g.Fp, a.c = (int)g.F;
    return a;
}
}  // namespace

dc_status_t dc_bn_apply(dc_plan_t pl, const void *y, const double *mean, const double *var, const float *gamma,
                        const float *beta, double eps, const void *residual, unsigned flags, dc_plan_t dst_plan,
                        void *dst, void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(pl && y && mean && var && gamma && beta && dst, DC_ERR_ARG, "null argument");
    DC_REQUIRE((flags & ~DC_RELU) == 0, DC_ERR_ARG, "unknown BN apply flags 0x%x", flags);
    NoPdlScope no_pdl(is_local(pl));
    ensure_local_resources(pl);
    cudaStream_t st = (cudaStream_t)stream;
    const ConvGeom &g = pl->rp.g;
    ensure_alloc(pl->grave, pl->bn_coef, pl->bn_coef_bytes, sizeof(float) * 4 * g.Fp);
    launch_bn_coeff(mean, var, gamma, beta, eps, (int)g.F, (int)g.Fp, pl->bn_coef, st);
    BnArgs a = bn_args(pl, y, residual, nullptr, (flags & DC_RELU) != 0);
    a.dst = dst;
    if (dst_plan) {  // the next layer's margined input: the same block of the activation
        const dc_shard_desc_t yd = describe(pl->rp, DC_Y), xd = describe(dst_plan->rp, DC_X);
        DC_REQUIRE(dst_plan->rp.g.dt == g.dt && xd.c == yd.c && xd.n0 == yd.n0 && xd.n == yd.n && xd.h0 == yd.h0 &&
                       xd.h == yd.h && xd.w0 == yd.w0 && xd.w == yd.w,
                   DC_ERR_PARTITION,
                   "dc_bn_apply: the next layer's input block differs from this layer's output block "
                   "(a different decomposition needs a redistribution)");
        a.hb = (int)xd.hb, a.wb = (int)xd.wb, a.r0 = xd.halo_n, a.c0 = xd.halo_w, a.dcp = (int)xd.c_pad;
        a.split = g.dt;
    } else {
        a.hb = a.h, a.wb = a.w, a.r0 = 0, a.c0 = 0, a.dcp = a.cpad, a.split = 0;
    }
    launch_bn_apply(a, st);
    DC_API_END
}

dc_status_t dc_bn_backward(dc_plan_t pl, const void *dout, const void *y, const double *mean, const double *var,
                           const float *gamma, const float *beta, double eps, const void *residual, unsigned flags,
                           float *dgamma, float *dbeta, void *dresidual, void *dy_margined, void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(pl && dout && y && mean && var && gamma && beta && dy_margined, DC_ERR_ARG, "null argument");
    DC_REQUIRE((flags & ~(DC_RELU | DC_BN_LOCAL)) == 0, DC_ERR_ARG, "unknown BN backward flags 0x%x", flags);
    NoPdlScope no_pdl(is_local(pl));
    ensure_local_resources(pl);
    cudaStream_t st = (cudaStream_t)stream;
    const RankPlan &rp = pl->rp;
    const ConvGeom &g = rp.g;
    ensure_alloc(pl->grave, pl->bn_coef, pl->bn_coef_bytes, sizeof(float) * 4 * g.Fp);
    ensure_alloc(pl->grave, pl->bn_scratch, pl->bn_scratch_bytes, sizeof(double) * 2 * g.Fp);
    launch_bn_coeff(mean, var, gamma, beta, eps, (int)g.F, (int)g.Fp, pl->bn_coef, st);
    BnArgs a = bn_args(pl, y, residual, dout, (flags & DC_RELU) != 0);
    const int blocks = bn_bwd_blocks(a);
    ensure_alloc(pl->grave, pl->bnb_part, pl->bnb_part_bytes, sizeof(double) * 2 * g.Fp * blocks);
    launch_bn_bwd_partials(a, pl->bnb_part, blocks, st);
    launch_bn_reduce(pl->bnb_part, blocks, (int)g.Fp, pl->bn_sums, (int)g.F, (double)a.npix, nullptr, nullptr, st);
    const bool global = !(flags & DC_BN_LOCAL) && pl->bn_group > 1;
    const double *sums = global ? bn_group_sum(pl, pl->bn_sums, pl->bn_scratch, pl->bn_scratch + g.Fp, st)
                                : pl->bn_sums;
    const double count = global ? (double)rp.nrange.size() * g.Ho * g.Wo : (double)a.npix;
    const dc_shard_desc_t dyd = describe(rp, DC_DY);
    a.dst = dy_margined;
    a.hb = (int)dyd.hb, a.wb = (int)dyd.wb, a.r0 = dyd.halo_n, a.c0 = dyd.halo_w, a.dcp = (int)dyd.c_pad;
    a.split = g.dt;
    launch_bn_bwd_apply(a, sums, count, gamma, dgamma, dbeta, dresidual, st);
    DC_API_END
}

}  // extern "C"

// ===========================================================================
// Redistribution between decompositions (Shuffle(D_i, D_j))
// ===========================================================================
struct dc_redist_s {
    dc_plan_s *from = nullptr, *to = nullptr;
    dc_tensor_t tf = DC_Y, tt = DC_X;
    dc_comm_s *comm = nullptr;
    bool is_virtual = false;
    int rank = 0, world = 1, which = 0, seq = -1;
    int esz = 2;
    // global block (samples, rows, cols) moving between this rank and `peer`
    struct Piece {
        int peer;
        int64_t n0, n, h0, h, w0, w;
    };
    std::vector<Piece> sends, recvs;  // ascending peer order
    dc_shard_desc_t src_d{};              // my source shard
    std::vector<dc_shard_desc_t> dst_all; // every rank's destination shard
    uint32_t *flags = nullptr;  // [2][world]: ready flag of rank p at p, data counter from p at world + p
    uint32_t *epoch = nullptr;  // {epoch, blocks done}
    std::map<int, uint32_t *> peer_flags;  // peer -> its flag array mapped here
    std::map<int, void *> peer_dst;        // receiver -> its destination buffer mapped here
    void *stage = nullptr;                 // NCCL transport: [send | recv]
    size_t stage_bytes = 0;
    std::vector<void *> grave;

    ~dc_redist_s() {
        const bool local = comm && comm->group;
        if (local) {
            std::lock_guard<std::mutex> lk(comm->group->mu);
            comm->group->redists.erase({seq, rank});
        } else {
            for (auto &kv : peer_flags)
                if (kv.first != rank) cudaIpcCloseMemHandle(kv.second);
            for (auto &kv : peer_dst)
                if (kv.first != rank) cudaIpcCloseMemHandle(kv.second);
        }
        for (void *q : grave) cudaFree(q);
        if (stage) cudaFree(stage);
        if (flags) cudaFree(flags);
        if (epoch) cudaFree(epoch);
    }
};

namespace {

// The global extents (N, H, W, channels) of a plan's tensor.
std::array<int64_t, 4> global_extent(const ConvGeom &g, dc_tensor_t t) {
    if (t == DC_X || t == DC_DX) return {g.N, g.H, g.W, g.C};
    return {g.N, g.Ho, g.Wo, g.F};
}

// The dc_buffer_alloc buffer of tensor t of a plan (margined X / DY, dense Y / DX).
void *alloc_buffer(const dc_plan_s *pl, dc_tensor_t t) {
    switch (t) {
    case DC_X: return pl->buf[0].ptr;
    case DC_DY: return pl->buf[1].ptr;
    case DC_Y: return pl->dense[0].ptr;
    case DC_DX: return pl->dense[1].ptr;
    default: return nullptr;
    }
}

Range isect(int64_t a0, int64_t an, int64_t b0, int64_t bn) {
    return Range{std::max(a0, b0), std::min(a0 + an, b0 + bn)};
}

// One piece as a copy: rows of `run` 16-byte vectors from the block at its
// place in shard `a` (pointer pa) to its place in shard `b` (pb); pass a
// null shard for a contiguous staging block [n][h][w] at pa / pb.
RedistPiece make_piece(const dc_redist_s::Piece &p, const dc_shard_desc_t *a, const void *pa,
                       const dc_shard_desc_t *b, void *pb, int esz) {
    const int64_t px = (a ? a->c_pad : b->c_pad) * esz / 16;  // vectors per pixel
    RedistPiece c{};
    auto place = [&](const dc_shard_desc_t *d, int64_t &sn, int64_t &sh) -> int64_t {
        if (!d) {
            sh = p.w * px, sn = p.h * sh;
            return 0;
        }
        sn = d->stride_n * esz / 16, sh = d->stride_h * esz / 16;
        return (p.n0 - d->n0) * sn + (p.h0 - d->h0 + d->halo_n) * sh + (p.w0 - d->w0 + d->halo_w) * px;
    };
    int64_t sn, sh, dn, dh;
    const int64_t so = place(a, sn, sh), dof = place(b, dn, dh);
    c.src = reinterpret_cast<const uint4 *>(pa) + so;
    c.dst = reinterpret_cast<uint4 *>(pb) + dof;
    c.s_sn = sn, c.s_sh = sh, c.d_sn = dn, c.d_sh = dh;
    c.nn = (int)p.n, c.rows = (int)p.h, c.run = (int)(p.w * px);
    return c;
}

int64_t piece_bytes(const dc_redist_s::Piece &p, int64_t pixel_bytes) { return p.n * p.h * p.w * pixel_bytes; }

void resolve_redist_peers(dc_redist_s *r) {
    if (!(r->comm && r->comm->group)) return;
    LocalGroup &G = *r->comm->group;
    for (int pass = 0; pass < 2; ++pass)
        for (auto &p : pass ? r->recvs : r->sends) {
            dc_redist_s *q = nullptr;
            {
                std::lock_guard<std::mutex> lk(G.mu);
                auto it = G.redists.find({r->seq, p.peer});
                DC_REQUIRE(it != G.redists.end(), DC_ERR_ARG,
                           "loopback group: rank %d has not created redistribution #%d", p.peer, r->seq);
                q = it->second;
            }
            r->peer_flags[p.peer] = q->flags;
            if (!pass) {
                void *d = alloc_buffer(local_peer(r->to, p.peer), r->tt);
                DC_REQUIRE(d != nullptr, DC_ERR_ARG, "redistribution: rank %d has no dc_buffer_alloc buffer",
                           p.peer);
                r->peer_dst[p.peer] = d;
            }
        }
}

// One P2P all-to-all (redist.cuh). Real ranks: the one-kernel protocol.
// Loopback group: the same flags in four launches -- a one-block ready
// handshake, the piece copies, the data flags, a one-block wait -- because the
// virtual ranks share the SMs: many spinning blocks of one rank could leave
// no room for the GEMM another rank must finish before it joins.
void run_redist_p2p(const RedistP2P &x, bool local, cudaStream_t st) {
    if (!local) {
        launch_redist_p2p(x, st);
        return;
    }
    CfFlags rdy{};
    for (int k = 0; k < x.n_ready_out; ++k) rdy.out[k] = x.ready_out[k];
    for (int k = 0; k < x.n_ready_in; ++k) rdy.in[k] = x.ready_in[k];
    rdy.n = x.n_ready_out, rdy.n_in = x.n_ready_in, rdy.epoch = x.epoch_ctr;
    launch_cf_handshake(rdy, st);
    launch_redist_copy(x.piece, x.npiece, st);
    launch_signal(const_cast<uint32_t *const *>(x.data_out), x.n_data_out, 0, x.epoch_ctr, st);
    CfFlags dat{};
    for (int k = 0; k < x.n_data_in; ++k) dat.in[k] = x.data_in[k];
    dat.n = 0, dat.n_in = x.n_data_in, dat.epoch = x.epoch_ctr, dat.publish = 1;
    launch_cf_wait(dat, st);
}

void redist_p2p(dc_redist_s *r, const void *src, cudaStream_t st) {
    resolve_redist_peers(r);
    DC_REQUIRE((int)r->sends.size() <= kRedistMaxPeers && (int)r->recvs.size() <= kRedistMaxPeers,
               DC_ERR_UNSUPPORTED, "P2P redistribution: more than %d peers (use DC_HALO_NCCL)", kRedistMaxPeers);
    RedistP2P x{};
    x.epoch_ctr = r->epoch;
    // blocks per launch, equal on all ranks of the group; a loopback group's
    // ranks share one GPU, and all of their blocks must be resident at once
    // (each waits for the others' flags): at most 4 blocks per SM in total
    x.nblocks = kRedistBlocks;
    if (r->comm->group) x.nblocks = std::max(8, std::min(kRedistBlocks, 4 * device_sm_count() / r->world));
    const int W = r->world;
    for (auto &p : r->sends) {
        x.piece[x.npiece++] = make_piece(p, &r->src_d, src, &r->dst_all[p.peer], r->peer_dst.at(p.peer), r->esz);
        x.ready_in[x.n_ready_in++] = r->flags + p.peer;
        x.data_out[x.n_data_out++] = r->peer_flags.at(p.peer) + W + r->rank;
    }
    for (auto &p : r->recvs) {
        x.ready_out[x.n_ready_out++] = r->peer_flags.at(p.peer) + r->rank;
        x.data_in[x.n_data_in++] = r->flags + W + p.peer;
    }
    run_redist_p2p(x, r->comm->group != nullptr, st);
}

void redist_nccl(dc_redist_s *r, const void *src, void *dst, cudaStream_t st) {
    const int64_t pxb = r->src_d.c_pad * r->esz;
    size_t sb = 0, rb = 0;
    for (auto &p : r->sends)
        if (p.peer != r->rank) sb += piece_bytes(p, pxb);
    for (auto &p : r->recvs)
        if (p.peer != r->rank) rb += piece_bytes(p, pxb);
    ensure_alloc(r->grave, reinterpret_cast<uint8_t *&>(r->stage), r->stage_bytes, sb + rb);
    uint8_t *sbuf = reinterpret_cast<uint8_t *>(r->stage), *rbuf = sbuf + sb;
    const dc_shard_desc_t &me = r->dst_all[r->rank];
    std::vector<RedistPiece> pack, unpack;
    size_t off = 0;
    for (auto &p : r->sends) {
        if (p.peer == r->rank) {
            pack.push_back(make_piece(p, &r->src_d, src, &me, dst, r->esz));  // the piece I keep
            continue;
        }
        pack.push_back(make_piece(p, &r->src_d, src, nullptr, sbuf + off, r->esz));
        off += piece_bytes(p, pxb);
    }
    launch_redist_copy(pack.data(), (int)pack.size(), st);
    NK(ncclGroupStart());
    off = 0;
    for (auto &p : r->sends)
        if (p.peer != r->rank) {
            NK(ncclSend(sbuf + off, piece_bytes(p, pxb), ncclUint8, p.peer, r->comm->nccl, st));
            off += piece_bytes(p, pxb);
        }
    off = 0;
    for (auto &p : r->recvs)
        if (p.peer != r->rank) {
            NK(ncclRecv(rbuf + off, piece_bytes(p, pxb), ncclUint8, p.peer, r->comm->nccl, st));
            off += piece_bytes(p, pxb);
        }
    NK(ncclGroupEnd());
    off = 0;
    for (auto &p : r->recvs)
        if (p.peer != r->rank) {
            unpack.push_back(make_piece(p, nullptr, rbuf + off, &me, dst, r->esz));
            off += piece_bytes(p, pxb);
        }
    launch_redist_copy(unpack.data(), (int)unpack.size(), st);
}

}  // namespace

extern "C" {

dc_status_t dc_redist_create(dc_plan_t from, dc_tensor_t tf, dc_plan_t to, dc_tensor_t tt, dc_redist_t *out) {
    DC_API_BEGIN
    DC_REQUIRE(from && to && out, DC_ERR_ARG, "null argument");
    DC_REQUIRE(tf == DC_X || tf == DC_Y || tf == DC_DX || tf == DC_DY, DC_ERR_ARG, "bad source tensor");
    DC_REQUIRE(tt == DC_X || tt == DC_Y || tt == DC_DX || tt == DC_DY, DC_ERR_ARG, "bad destination tensor");
    DC_REQUIRE(from->is_virtual == to->is_virtual, DC_ERR_ARG, "both plans virtual, or neither");
    DC_REQUIRE(from->rp.rank == to->rp.rank && from->world() == to->world(), DC_ERR_ARG,
               "plans of different ranks / world sizes");
    DC_REQUIRE(from->is_virtual || from->comm == to->comm, DC_ERR_ARG, "plans on different communicators");
    const ConvGeom &gf = from->rp.g, &gt = to->rp.g;
    DC_REQUIRE(gf.dt == gt.dt, DC_ERR_ARG, "plans of different dtypes");
    const auto ef = global_extent(gf, tf), et = global_extent(gt, tt);
    DC_REQUIRE(ef == et, DC_ERR_SHAPE, "tensors differ: (%lld,%lld,%lld,%lld) vs (%lld,%lld,%lld,%lld)",
               (long long)ef[0], (long long)ef[1], (long long)ef[2], (long long)ef[3], (long long)et[0],
               (long long)et[1], (long long)et[2], (long long)et[3]);
    std::unique_ptr<dc_redist_s> r(new dc_redist_s());
    r->from = from, r->to = to, r->tf = tf, r->tt = tt;
    r->comm = from->comm, r->is_virtual = from->is_virtual;
    r->rank = from->rp.rank, r->world = from->world();
    r->which = tt == DC_X ? 0 : 1;
    r->esz = gf.esz();
    r->src_d = describe(from->rp, tf);
    DC_REQUIRE(r->src_d.c_pad == describe(to->rp, tt).c_pad, DC_ERR_UNSUPPORTED,
               "pixel layouts differ (fp32 plans: the source must be a margined x / dy, whose pixels are "
               "already split into tf32 [hi | lo])");
    // every rank's owned blocks under both decompositions (host integer math)
    std::vector<dc_shard_desc_t> src_all(r->world);
    r->dst_all.resize(r->world);
    for (int q = 0; q < r->world; ++q) {
        src_all[q] = q == r->rank ? r->src_d : describe(make_rank_plan(gf, from->rp.grid, q), tf);
        r->dst_all[q] = describe(q == r->rank ? to->rp : make_rank_plan(gt, to->rp.grid, q), tt);
    }
    auto piece = [&](int peer, const dc_shard_desc_t &a, const dc_shard_desc_t &b, std::vector<dc_redist_s::Piece> &v) {
        const Range n = isect(a.n0, a.n, b.n0, b.n), h = isect(a.h0, a.h, b.h0, b.h), w = isect(a.w0, a.w, b.w0, b.w);
        if (!n.empty() && !h.empty() && !w.empty())
            v.push_back({peer, n.lo, n.size(), h.lo, h.size(), w.lo, w.size()});
    };
    for (int q = 0; q < r->world; ++q) {
        piece(q, r->src_d, r->dst_all[q], r->sends);
        piece(q, src_all[q], r->dst_all[r->rank], r->recvs);
    }
    if (!r->is_virtual && r->world > 1) {
        dc_comm_s *c = r->comm;
        DC_REQUIRE(c && (c->nccl || c->group), DC_ERR_ARG, "redistribution needs a communicator");
        void *dst = alloc_buffer(to, tt);
        DC_REQUIRE(dst != nullptr, DC_ERR_ARG,
                   "redistribution: allocate the destination with dc_buffer_alloc (on every rank) first");
        r->seq = c->redist_seq++;
        CK(cudaMalloc(&r->flags, sizeof(uint32_t) * 2 * r->world));
        CK(cudaMemset(r->flags, 0, sizeof(uint32_t) * 2 * r->world));
        CK(cudaMalloc(&r->epoch, sizeof(uint32_t) * 2));
        CK(cudaMemset(r->epoch, 0, sizeof(uint32_t) * 2));
        if (c->group) {
            std::lock_guard<std::mutex> lk(c->group->mu);
            c->group->redists[{r->seq, r->rank}] = r.get();
        } else {
            struct Handles {
                cudaIpcMemHandle_t flags, dst;
            } h{};
            CK(cudaIpcGetMemHandle(&h.flags, r->flags));
            CK(cudaIpcGetMemHandle(&h.dst, dst));
            auto all = comm_allgather(c, &h, sizeof h);
            auto at = [&](int q) {
                Handles x;
                std::memcpy(&x, all.data() + q * sizeof x, sizeof x);
                return x;
            };
            for (int pass = 0; pass < 2; ++pass)
                for (auto &p : pass ? r->recvs : r->sends) {
                    if (p.peer == r->rank) {
                        r->peer_flags[p.peer] = r->flags;
                        if (!pass) r->peer_dst[p.peer] = dst;
                        continue;
                    }
                    if (!r->peer_flags.count(p.peer)) {
                        void *ptr = nullptr;
                        CK(cudaIpcOpenMemHandle(&ptr, at(p.peer).flags, cudaIpcMemLazyEnablePeerAccess));
                        r->peer_flags[p.peer] = reinterpret_cast<uint32_t *>(ptr);
                    }
                    if (!pass) {
                        void *ptr = nullptr;
                        CK(cudaIpcOpenMemHandle(&ptr, at(p.peer).dst, cudaIpcMemLazyEnablePeerAccess));
                        r->peer_dst[p.peer] = ptr;
                    }
                }
        }
        CK(cudaDeviceSynchronize());
    }
    *out = r.release();
    DC_API_END
}

dc_status_t dc_redist_bytes(dc_redist_t r, int64_t *send_bytes, int64_t *recv_bytes) {
    DC_API_BEGIN
    DC_REQUIRE(r && send_bytes && recv_bytes, DC_ERR_ARG, "null argument");
    const int64_t pxb = r->src_d.c_pad * r->esz;
    for (int q = 0; q < r->world; ++q) send_bytes[q] = recv_bytes[q] = 0;
    for (auto &p : r->sends) send_bytes[p.peer] = piece_bytes(p, pxb);
    for (auto &p : r->recvs) recv_bytes[p.peer] = piece_bytes(p, pxb);
    DC_API_END
}

dc_status_t dc_redistribute(dc_redist_t r, const void *src, void *dst, unsigned flags, void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(r && src && dst, DC_ERR_ARG, "null argument");
    DC_REQUIRE(!r->is_virtual, DC_ERR_ARG, "virtual plans have no data");
    DC_REQUIRE((flags & ~DC_HALO_NCCL) == 0, DC_ERR_ARG, "unknown redistribution flags 0x%x", flags);
    DC_REQUIRE(src != dst, DC_ERR_ARG, "redistribution is not in place");
    cudaStream_t st = (cudaStream_t)stream;
    const bool local = r->comm && r->comm->group;
    NoPdlScope no_pdl(local);  // (loopback: ranks share the SMs)
    if (r->tt == DC_X || r->tt == DC_DY) join_import(r->to, r->which, st);
    if (r->tf == DC_X || r->tf == DC_DY) join_import(r->from, r->tf == DC_X ? 0 : 1, st);
    if (r->world == 1) {
        const dc_shard_desc_t &me = r->dst_all[0];
        std::vector<RedistPiece> one;
        for (auto &p : r->sends) one.push_back(make_piece(p, &r->src_d, src, &me, dst, r->esz));
        launch_redist_copy(one.data(), (int)one.size(), st);
    } else if (flags & DC_HALO_NCCL) {
        DC_REQUIRE(!local, DC_ERR_UNSUPPORTED, "DC_HALO_NCCL needs real ranks (loopback group)");
        redist_nccl(r, src, dst, st);
    } else {
        DC_REQUIRE(dst == alloc_buffer(r->to, r->tt), DC_ERR_ARG,
                   "P2P redistribution writes the destination plan's dc_buffer_alloc buffer");
        redist_p2p(r, src, st);
    }
    DC_API_END
}

dc_status_t dc_redist_destroy(dc_redist_t r) {
    DC_API_BEGIN
    delete r;
    DC_API_END
}

}  // extern "C"

// ===========================================================================
// Channel / filter parallelism
// ===========================================================================
// Ranks form a pN x pC grid (rank = i_N pC + i_C). Rank (i_N, i_C) owns the
// samples block i_N, the input channels block i_C (x, dx, its columns of w and
// dW) and the filters block i_C (y, dy): "if the input x to a layer is
// partitioned on its C dimension, the output y is partitioned on its F
// dimension". Forward: every rank of a channel group computes
// the partial y of ALL filters over its channels and the sum over channels
// is a reduce-scatter over F; backward-data likewise over F
// with a reduce-scatter over C; backward-filter gathers dy over the group
// ("may require data to be gathered") and computes its dW
// columns, summed over the sample groups (DC_ALLREDUCE). The reduce-scatter
// runs inside the conv GEMM: its epilogue stores each fp32 partial tile
// straight into the receive slot of the block's owner over peer memory, the
// owner sums the p slots in rank order.
struct dc_cplan_s {
    ConvGeom g;
    int pn = 1, pc = 1, rank = 0, in = 0, ic = 0;
    Range nr, cr, fr;  // my samples, input channels, filters (global)
    bool is_virtual = false;
    dc_comm_s *comm = nullptr;
    int seq = -1;
    dc_plan_s *fwd = nullptr;  // (N_l, C_r, H, W, F): forward, backward-filter
    dc_plan_s *bwd = nullptr;  // (N_l, C, H, W, F_r): backward-data
    __nv_bfloat16 *wslice = nullptr;  // w[:, C_r] as [F][K][K][C_r]
    size_t wslice_bytes = 0;
    float *slots = nullptr;          // [pc][slot_elems] fp32 partials received
    int64_t slot_elems = 0;
    __nv_bfloat16 *dyfull = nullptr; // [N_l][Ho][Wo][F]: dy gathered over the group
    uint32_t *flags = nullptr;       // [4][pc]: conv ready, conv data, gather ready, gather data
    uint32_t *epochs = nullptr;      // [2][2]: conv exchange {epoch, count}, gather {epoch, count}
    float *peer_slots[kCfMaxGroup] = {};
    uint32_t *peer_flags[kCfMaxGroup] = {};
    __nv_bfloat16 *peer_dyfull[kCfMaxGroup] = {};
    bool resolved = false;
    ncclComm_t sample_comm = nullptr;  // ranks with my i_C (dW allreduce over the samples)

    int64_t npix_y() const { return nr.size() * g.Ho * g.Wo; }
    int64_t npix_x() const { return nr.size() * g.H * g.W; }
    int member(int k) const { return in * pc + k; }
    ~dc_cplan_s() {
        const bool local = comm && comm->group;
        if (local) {
            std::lock_guard<std::mutex> lk(comm->group->mu);
            comm->group->cplans.erase({seq, rank});
        } else {
            for (int k = 0; k < pc; ++k) {
                if (k == ic) continue;
                if (peer_slots[k]) cudaIpcCloseMemHandle(peer_slots[k]);
                if (peer_flags[k]) cudaIpcCloseMemHandle(peer_flags[k]);
                if (peer_dyfull[k]) cudaIpcCloseMemHandle(peer_dyfull[k]);
            }
        }
        if (sample_comm) ncclCommAbort(sample_comm);  // (see dc_comm_destroy)
        delete fwd;
        delete bwd;
        if (wslice) cudaFree(wslice);
        if (slots) cudaFree(slots);
        if (dyfull) cudaFree(dyfull);
        if (flags) cudaFree(flags);
        if (epochs) cudaFree(epochs);
    }
};

namespace {

dc_cplan_s *create_cplan(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int K, int S, int P, int pn, int pc,
                         int rank, dc_comm_s *comm, bool is_virtual) {
    DC_REQUIRE(pn >= 1 && pc >= 1 && pc <= kCfMaxGroup, DC_ERR_ARG, "bad channel grid (%d, %d)", pn, pc);
    std::unique_ptr<dc_cplan_s> c(new dc_cplan_s());
    c->g = make_geom(N, C, H, W, F, K, S, P, 0);
    DC_REQUIRE(C % (16 * pc) == 0 && F % (16 * pc) == 0, DC_ERR_UNSUPPORTED,
               "channel / filter parallelism: C and F must be multiples of 16 x p_C (C=%lld F=%lld p_C=%d)",
               (long long)C, (long long)F, pc);
    DC_REQUIRE(pn <= N, DC_ERR_PARTITION, "p_N = %d > N = %lld", pn, (long long)N);
    c->pn = pn, c->pc = pc, c->rank = rank, c->in = rank / pc, c->ic = rank % pc;
    c->nr = blocked(N, pn, c->in);
    c->cr = blocked(C, pc, c->ic);
    c->fr = blocked(F, pc, c->ic);
    c->is_virtual = is_virtual;
    c->comm = comm;
    const int64_t nl = c->nr.size();
    c->fwd = create_plan(make_geom(nl, c->cr.size(), H, W, F, K, S, P, 0), Grid{1, 1, 1}, 0, comm, is_virtual);
    c->bwd = create_plan(make_geom(nl, C, H, W, c->fr.size(), K, S, P, 0), Grid{1, 1, 1}, 0, comm, is_virtual);
    if (is_virtual) return c.release();
    const ConvGeom &g = c->g;
    c->slot_elems = std::max(c->npix_y() * c->fr.size(), c->npix_x() * c->cr.size());
    CK(cudaMalloc(&c->wslice, (size_t)F * K * K * c->cr.size() * 2));
    CK(cudaMalloc(&c->slots, (size_t)pc * c->slot_elems * 4));
    CK(cudaMalloc(&c->dyfull, (size_t)c->npix_y() * F * 2));
    CK(cudaMemset(c->dyfull, 0, (size_t)c->npix_y() * F * 2));
    CK(cudaMalloc(&c->flags, sizeof(uint32_t) * 4 * pc));
    CK(cudaMemset(c->flags, 0, sizeof(uint32_t) * 4 * pc));
    CK(cudaMalloc(&c->epochs, sizeof(uint32_t) * 4));
    CK(cudaMemset(c->epochs, 0, sizeof(uint32_t) * 4));
    (void)g;
    const int world = pn * pc;
    if (world > 1) {
        DC_REQUIRE(comm && comm->world == world && comm->rank == rank, DC_ERR_ARG,
                   "channel grid (%d, %d) needs a communicator of %d ranks", pn, pc, world);
        c->seq = comm->cplan_seq++;
        if (comm->group) {
            std::lock_guard<std::mutex> lk(comm->group->mu);
            comm->group->cplans[{c->seq, rank}] = c.get();
        } else {
            if (pn > 1) NK(ncclCommSplit(comm->nccl, c->ic, rank, &c->sample_comm, nullptr));
            struct Handles {
                cudaIpcMemHandle_t slots, flags, dyfull;
            } h{};
            CK(cudaIpcGetMemHandle(&h.slots, c->slots));
            CK(cudaIpcGetMemHandle(&h.flags, c->flags));
            CK(cudaIpcGetMemHandle(&h.dyfull, c->dyfull));
            auto all = comm_allgather(comm, &h, sizeof h);
            for (int k = 0; k < pc; ++k) {
                if (k == c->ic) continue;
                Handles x;
                std::memcpy(&x, all.data() + c->member(k) * sizeof x, sizeof x);
                void *p = nullptr;
                CK(cudaIpcOpenMemHandle(&p, x.slots, cudaIpcMemLazyEnablePeerAccess));
                c->peer_slots[k] = reinterpret_cast<float *>(p);
                CK(cudaIpcOpenMemHandle(&p, x.flags, cudaIpcMemLazyEnablePeerAccess));
                c->peer_flags[k] = reinterpret_cast<uint32_t *>(p);
                CK(cudaIpcOpenMemHandle(&p, x.dyfull, cudaIpcMemLazyEnablePeerAccess));
                c->peer_dyfull[k] = reinterpret_cast<__nv_bfloat16 *>(p);
            }
            c->resolved = true;
        }
    }
    c->peer_slots[c->ic] = c->slots, c->peer_flags[c->ic] = c->flags, c->peer_dyfull[c->ic] = c->dyfull;
    if (world == 1) c->resolved = true;
    CK(cudaDeviceSynchronize());
    return c.release();
}

void resolve_cplan(dc_cplan_s *c) {
    if (c->resolved) return;
    LocalGroup &G = *c->comm->group;
    std::lock_guard<std::mutex> lk(G.mu);
    for (int k = 0; k < c->pc; ++k) {
        auto it = G.cplans.find({c->seq, c->member(k)});
        DC_REQUIRE(it != G.cplans.end(), DC_ERR_ARG, "loopback group: rank %d has not created channel plan #%d",
                   c->member(k), c->seq);
        c->peer_slots[k] = it->second->slots;
        c->peer_flags[k] = it->second->flags;
        c->peer_dyfull[k] = it->second->dyfull;
    }
    c->resolved = true;
}

// flags kind: 0 conv ready, 1 conv data, 2 gather ready, 3 gather data
CfFlags cf_flags(const dc_cplan_s *c, int kind) {
    CfFlags f{};
    f.n = c->pc;
    for (int k = 0; k < c->pc; ++k) {
        f.out[k] = c->peer_flags[k] + kind * c->pc + c->ic;
        f.in[k] = c->flags + kind * c->pc + k;
    }
    f.epoch = c->epochs;
    return f;
}

// The reduce-scatter half of a channel-parallel conv call: the partial of
// block k goes to member k's slot [my index]; after the GEMM (queued by
// `gemm`), wait for every member's partial and sum them into `out`.
template <class Gemm>
void cf_reduce_scatter(dc_cplan_s *c, dc_plan_s *sub, int64_t seg, int64_t npix, void *out, cudaStream_t st,
                       Gemm &&gemm) {
    resolve_cplan(c);
    launch_cf_handshake(cf_flags(c, 0), st);  // every owner's slots are free
    for (int k = 0; k < c->pc; ++k) sub->scat[k] = c->peer_slots[k] + (int64_t)c->ic * c->slot_elems;
    sub->scat_seg = (int)seg;
    try {
        gemm();
    } catch (...) {
        sub->scat_seg = 0;
        throw;
    }
    sub->scat_seg = 0;
    const CfFlags d = cf_flags(c, 1);
    launch_signal(const_cast<uint32_t *const *>(d.out), d.n, 0, c->epochs, st);
    launch_cf_wait(d, st);
    launch_cf_reduce(c->slots, c->pc, c->slot_elems, npix, (int)seg, out, (int)seg, c->epochs, st);
}

}  // namespace

extern "C" {

dc_status_t dc_cplan_create(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int K, int stride, int pad,
                            int pn, int pc, dc_dtype_t dtype, dc_comm_t comm, dc_cplan_t *out) {
    DC_API_BEGIN
    DC_REQUIRE(out != nullptr, DC_ERR_ARG, "null out");
    DC_REQUIRE(dtype == DC_BF16, DC_ERR_UNSUPPORTED, "channel / filter parallelism: bf16 plans only");
    const int rank = comm ? comm->rank : 0;
    if (comm) CK(cudaSetDevice(comm->device));
    *out = create_cplan(N, C, H, W, F, K, stride, pad, pn, pc, rank, comm, false);
    DC_API_END
}

dc_status_t dc_cplan_create_virtual(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int K, int stride,
                                    int pad, int pn, int pc, int rank, dc_cplan_t *out) {
    DC_API_BEGIN
    DC_REQUIRE(out != nullptr && rank >= 0 && rank < pn * pc, DC_ERR_ARG, "bad argument");
    *out = create_cplan(N, C, H, W, F, K, stride, pad, pn, pc, rank, nullptr, true);
    DC_API_END
}

dc_status_t dc_cplan_query(dc_cplan_t c, dc_tensor_t t, dc_shard_desc_t *desc, int64_t *c0) {
    DC_API_BEGIN
    DC_REQUIRE(c && desc, DC_ERR_ARG, "null argument");
    int64_t first = 0;
    switch (t) {
    case DC_X:
    case DC_DX:
        *desc = describe(c->fwd->rp, t);
        first = c->cr.lo;
        break;
    case DC_Y:
    case DC_DY:
        *desc = describe(c->bwd->rp, t);
        first = c->fr.lo;
        break;
    case DC_W: {  // replicated: the whole [F][K][K][C] bf16 filter bank
        const ConvGeom &g = c->g;
        dc_shard_desc_t d{};
        d.n = g.F, d.h = g.K, d.w = g.K, d.c = g.C, d.c_pad = g.C, d.hb = g.K, d.wb = g.K;
        d.stride_w = g.C, d.stride_h = g.K * g.C, d.stride_n = g.K * g.K * g.C;
        d.bytes = (size_t)g.F * g.K * g.K * g.C * 2;
        *desc = d;
        break;
    }
    case DC_DW:
        *desc = describe(c->fwd->rp, DC_DW);
        first = c->cr.lo;
        break;
    default:
        fail(DC_ERR_ARG, "unknown tensor kind");
    }
    desc->n0 = t == DC_W || t == DC_DW ? 0 : c->nr.lo;
    if (c0) *c0 = first;
    DC_API_END
}

dc_status_t dc_cconv_fwd(dc_cplan_t c, const void *x, const void *w, void *y, unsigned flags, void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(c && x && w && y, DC_ERR_ARG, "null argument");
    DC_REQUIRE(!c->is_virtual, DC_ERR_ARG, "virtual plans have no data");
    DC_REQUIRE(flags == 0, DC_ERR_ARG, "unknown flags 0x%x", flags);
    const bool local = c->comm && c->comm->group;
    NoPdlScope no_pdl(local);
    cudaStream_t st = (cudaStream_t)stream;
    const ConvGeom &g = c->g;
    const int64_t cl = c->cr.size();
    // my columns of the replicated filter bank: w[:, :, :, C_r]
    RedistPiece wp{};
    wp.src = reinterpret_cast<const uint4 *>(reinterpret_cast<const __nv_bfloat16 *>(w) + c->cr.lo);
    wp.dst = reinterpret_cast<uint4 *>(c->wslice);
    wp.nn = 1, wp.rows = (int)(g.F * g.K * g.K), wp.run = (int)(cl * 2 / 16);
    wp.s_sh = g.C * 2 / 16, wp.d_sh = cl * 2 / 16;
    launch_redist_copy(&wp, 1, st);
    dc_plan_s *sub = c->fwd;
    ensure_local_resources(sub);
    cf_reduce_scatter(c, sub, c->fr.size(), c->npix_y(), y, st, [&] {
        GemmLaunch L;
        prepare_fwd(sub, x, c->wslice, y, L, st);
        launch_rects(L, {whole(L)}, x, describe(sub->rp, DC_X), L.cin, (int)sub->rp.nrange.size(), st);
    });
    DC_API_END
}

dc_status_t dc_cconv_bwd_data(dc_cplan_t c, const void *dy, const void *w, void *dx, unsigned flags,
                              void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(c && dy && w && dx, DC_ERR_ARG, "null argument");
    DC_REQUIRE(!c->is_virtual, DC_ERR_ARG, "virtual plans have no data");
    DC_REQUIRE(flags == 0, DC_ERR_ARG, "unknown flags 0x%x", flags);
    const bool local = c->comm && c->comm->group;
    NoPdlScope no_pdl(local);
    cudaStream_t st = (cudaStream_t)stream;
    const ConvGeom &g = c->g;
    dc_plan_s *sub = c->bwd;
    ensure_local_resources(sub);
    // my filters' rows of the replicated bank: w[F_r, :, :, :]
    const __nv_bfloat16 *wf = reinterpret_cast<const __nv_bfloat16 *>(w) + c->fr.lo * g.K * g.K * g.C;
    cf_reduce_scatter(c, sub, c->cr.size(), c->npix_x(), dx, st,
                      [&] { run_bwd_data(sub, const_cast<void *>(dy), wf, dx, 0, st); });
    DC_API_END
}

dc_status_t dc_cconv_bwd_filter(dc_cplan_t c, const void *x, const void *dy, float *dw, unsigned flags,
                                void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(c && x && dy && dw, DC_ERR_ARG, "null argument");
    DC_REQUIRE(!c->is_virtual, DC_ERR_ARG, "virtual plans have no data");
    DC_REQUIRE((flags & ~DC_ALLREDUCE) == 0, DC_ERR_ARG, "unknown flags 0x%x", flags);
    const bool local = c->comm && c->comm->group;
    NoPdlScope no_pdl(local);
    cudaStream_t st = (cudaStream_t)stream;
    const ConvGeom &g = c->g;
    resolve_cplan(c);
    // gather dy over the channel group: my filters' block of every pixel into
    // every member's [N_l][Ho][Wo][F] (one P2P all-to-all launch)
    const int64_t fl = c->fr.size();
    RedistP2P x2{};
    x2.epoch_ctr = c->epochs + 2;
    x2.nblocks = local ? std::max(8, std::min(kRedistBlocks, 4 * device_sm_count() / (c->pn * c->pc)))
                       : kRedistBlocks;
    for (int k = 0; k < c->pc; ++k) {
        RedistPiece &p = x2.piece[x2.npiece++];
        p.src = reinterpret_cast<const uint4 *>(dy);
        p.dst = reinterpret_cast<uint4 *>(c->peer_dyfull[k] + c->fr.lo);
        p.nn = 1, p.rows = (int)c->npix_y(), p.run = (int)(fl * 2 / 16);
        p.s_sh = fl * 2 / 16, p.d_sh = g.F * 2 / 16;
        x2.ready_out[x2.n_ready_out++] = c->peer_flags[k] + 2 * c->pc + c->ic;
        x2.ready_in[x2.n_ready_in++] = c->flags + 2 * c->pc + k;
        x2.data_out[x2.n_data_out++] = c->peer_flags[k] + 3 * c->pc + c->ic;
        x2.data_in[x2.n_data_in++] = c->flags + 3 * c->pc + k;
    }
    run_redist_p2p(x2, local, st);
    dc_plan_s *sub = c->fwd;
    ensure_local_resources(sub);
    run_bwd_filter(sub, x, c->dyfull, dw, st, false);
    if ((flags & DC_ALLREDUCE) && c->pn > 1) {
        DC_REQUIRE(!local, DC_ERR_UNSUPPORTED, "dW allreduce needs real ranks (loopback group: DC_ALLREDUCE off)");
        NK(ncclAllReduce(dw, dw, (size_t)g.F * g.K * g.K * c->cr.size(), ncclFloat32, ncclSum, c->sample_comm, st));
    }
    DC_API_END
}

dc_status_t dc_cplan_destroy(dc_cplan_t c) {
    DC_API_BEGIN
    delete c;
    DC_API_END
}

}  // extern "C"

// ===========================================================================
// Max pooling on the decomposition ("Pooling layers are
// parallelized similarly"; "halo exchanges before ... pooling")
// ===========================================================================
// Two plans of one grid: the OUTPUT plan has the pooling window's geometry
// (K, S, P: y / dy ownership, the dy halo of the backward); the INPUT plan's
// x buffer carries a halo of K - 1 on every side (a K' = 2K - 1, S' = 1,
// P' = K - 1 geometry), wide enough that the backward can recompute the first
// maximum of every window that touches an owned input -- including windows
// of outputs owned by a neighbour -- from x (no argmax tensor to store or
// exchange).
struct dc_pool_s {
    dc_plan_s *in = nullptr, *out = nullptr;
    PoolGeom pg{};
    ~dc_pool_s() {
        delete out;
        delete in;
    }
};

extern "C" {

dc_status_t dc_pool_create(int64_t N, int64_t C, int64_t H, int64_t W, int K, int stride, int pad, dc_decomp_t decomp,
                           dc_dtype_t dtype, dc_comm_t comm, dc_pool_t *out) {
    DC_API_BEGIN
    DC_REQUIRE(out != nullptr, DC_ERR_ARG, "null out");
    DC_REQUIRE(dtype == DC_BF16, DC_ERR_UNSUPPORTED, "pooling: bf16 plans only");
    DC_REQUIRE(decomp.pn > 0 && decomp.ph > 0 && decomp.pw > 0, DC_ERR_ARG, "pooling needs an explicit grid");
    DC_REQUIRE(K >= 1 && K % 2 == 1, DC_ERR_SHAPE, "pooling window K=%d: odd (PAPER.md:57)", K);
    DC_REQUIRE(2 * K - 1 <= 15 && pad < K, DC_ERR_UNSUPPORTED, "pooling window K=%d pad=%d", K, pad);
    const Grid grid{decomp.pn, decomp.ph, decomp.pw};
    const int rank = comm ? comm->rank : 0;
    DC_REQUIRE(grid.size() == 1 || (comm && comm->world == grid.size()), DC_ERR_ARG,
               "grid of %d ranks needs a communicator of that size", grid.size());
    if (comm) CK(cudaSetDevice(comm->device));
    std::unique_ptr<dc_pool_s> p(new dc_pool_s());
    p->in = create_plan(make_geom(N, C, H, W, C, 2 * K - 1, 1, K - 1, 0), grid, rank, comm, false);
    p->out = create_plan(make_geom(N, C, H, W, C, K, stride, pad, 0), grid, rank, comm, false);
    const RankPlan &ri = p->in->rp, &ro = p->out->rp;
    const ConvGeom &g = ro.g;
    // every window the forward (owned outputs) and the backward (outputs in
    // the dy buffer) evaluate lies inside the wide x buffer
    auto covered = [&](const DimSplit &o, const DimSplit &x, int64_t X) {
        for (const Range &r : {o.out, o.dbuf}) {
            if (r.empty()) continue;
            const int64_t lo = std::max<int64_t>(0, stride * r.lo - pad);
            const int64_t hi = std::min<int64_t>(X, stride * (r.hi - 1) - pad + K);
            if (lo < x.xbuf.lo || hi > x.xbuf.hi) return false;
        }
        return x.in.lo == o.in.lo && x.in.hi == o.in.hi;
    };
    DC_REQUIRE(covered(ro.h, ri.h, H) && covered(ro.w, ri.w, W), DC_ERR_PARTITION,
               "pooling: the windows of this rank's outputs reach past the neighbouring input blocks");
    PoolGeom &q = p->pg;
    q.K = K, q.S = stride, q.P = pad, q.H = (int)H, q.W = (int)W;
    q.n = (int)ro.nrange.size(), q.cpad = (int)g.Cp;
    q.xr0 = (int)ri.h.xbuf.lo, q.xc0 = (int)ri.w.xbuf.lo;
    q.xhb = (int)ri.h.xbuf.size(), q.xwb = (int)ri.w.xbuf.size();
    q.oh0 = (int)ro.h.out.lo, q.ow0 = (int)ro.w.out.lo, q.oh = (int)ro.h.out.size(), q.ow = (int)ro.w.out.size();
    q.gi0 = (int)ro.h.in.lo, q.gj0 = (int)ro.w.in.lo, q.ih = (int)ro.h.in.size(), q.iw = (int)ro.w.in.size();
    q.dr0 = (int)ro.h.dbuf.lo, q.dc0 = (int)ro.w.dbuf.lo;
    q.dhb = (int)ro.h.dbuf.size(), q.dwb = (int)ro.w.dbuf.size();
    q.Ho = (int)g.Ho, q.Wo = (int)g.Wo;
    *out = p.release();
    DC_API_END
}

dc_status_t dc_pool_plans(dc_pool_t p, dc_plan_t *in_plan, dc_plan_t *out_plan) {
    DC_API_BEGIN
    DC_REQUIRE(p, DC_ERR_ARG, "null pool");
    if (in_plan) *in_plan = p->in;
    if (out_plan) *out_plan = p->out;
    DC_API_END
}

dc_status_t dc_pool_fwd(dc_pool_t p, void *x, void *y, unsigned flags, void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(p && x && y, DC_ERR_ARG, "null argument");
    DC_REQUIRE((flags & ~(DC_EXCHANGE | DC_HALO_NCCL)) == 0, DC_ERR_ARG, "unknown pooling flags 0x%x", flags);
    NoPdlScope no_pdl(is_local(p->in));
    cudaStream_t st = (cudaStream_t)stream;
    join_import(p->in, 0, st);
    if (flags & DC_EXCHANGE) exchange(p->in, 0, x, flags & DC_HALO_NCCL, st);
    launch_maxpool_fwd(p->pg, x, y, st);
    DC_API_END
}

dc_status_t dc_pool_bwd(dc_pool_t p, const void *x, void *dy, void *dx, unsigned flags, void *stream) {
    DC_API_BEGIN
    DC_REQUIRE(p && x && dy && dx, DC_ERR_ARG, "null argument");
    DC_REQUIRE((flags & ~(DC_EXCHANGE | DC_HALO_NCCL)) == 0, DC_ERR_ARG, "unknown pooling flags 0x%x", flags);
    NoPdlScope no_pdl(is_local(p->out));
    cudaStream_t st = (cudaStream_t)stream;
    join_import(p->out, 1, st);
    if (flags & DC_EXCHANGE) exchange(p->out, 1, dy, flags & DC_HALO_NCCL, st);
    launch_maxpool_bwd(p->pg, x, dy, dx, st);
    DC_API_END
}

dc_status_t dc_pool_destroy(dc_pool_t p) {
    DC_API_BEGIN
    delete p;
    DC_API_END
}

}  // extern "C"


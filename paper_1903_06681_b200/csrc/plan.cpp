// plan.cpp -- L1 index math (see plan.hpp for the paper passages).
#include "plan.hpp"

#include <algorithm>
#include <string>

namespace dc {

Range blocked(int64_t extent, int parts, int idx) {
    const int64_t base = extent / parts, rem = extent % parts;
    Range r;
    r.lo = idx * base + std::min<int64_t>(idx, rem);
    r.hi = r.lo + base + (idx < rem ? 1 : 0);
    return r;
}

ConvGeom make_geom(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int K, int S, int P, int dt) {
    DC_REQUIRE(N > 0 && C > 0 && H > 0 && W > 0 && F > 0, DC_ERR_SHAPE,
               "non-positive extent (N=%lld C=%lld H=%lld W=%lld F=%lld)", (long long)N,
               (long long)C, (long long)H, (long long)W, (long long)F);
    DC_REQUIRE(K > 0 && K % 2 == 1, DC_ERR_SHAPE, "K must be odd and positive (K=%d; PAPER.md:57)", K);
    DC_REQUIRE(P >= 0 && P <= K / 2, DC_ERR_SHAPE, "need 0 <= P <= K/2 (P=%d, K=%d)", P, K);
    DC_REQUIRE(S >= 1, DC_ERR_SHAPE, "stride must be >= 1");
    DC_REQUIRE(S <= 2, DC_ERR_UNSUPPORTED, "stride %d not supported (1 or 2)", S);
    ConvGeom g{N, C, H, W, F, K, S, P, 0, 0, 0, 0, dt};
    DC_REQUIRE(H + 2 * P >= K && W + 2 * P >= K, DC_ERR_SHAPE, "input smaller than the kernel");
    g.Ho = (H + 2 * P - K) / S + 1;
    g.Wo = (W + 2 * P - K) / S + 1;
    // 32-byte channel granules: 16 bf16 or 8 fp32 (one MMA K step either way);
    // fp32 channel counts above 8 go to multiples of 32, so the 3xTF32 K
    // segments (6 x C_pad 16-bit units per tap) fill 128-byte (64-unit) stages
    // (C = 18: 24 channels gave 16-unit stages, measured 6x slower)
    auto pad = [&](int64_t c) { return dt ? (c <= 8 ? 8 : round_up(c, 32)) : round_up(c, 16); };
    g.Cp = pad(C);
    g.Fp = pad(F);
    return g;
}

// Input rows read by owned output rows [oq, or) through Eq. 1
// (index S*i + a - P), clipped to [0, X): [S oq - P, S (or-1) - P + K).
static Range fwd_window(Range out, int64_t X, int K, int S, int P) {
    Range r;
    if (out.empty()) return r;
    r.lo = std::max<int64_t>(0, S * out.lo - P);
    r.hi = std::min<int64_t>(X, S * (out.hi - 1) - P + K);
    return r;
}

// dy rows read by owned input rows [q, r) through Eq. 3 (strided adjoint,
// reading R4): i in [ceil((q + P - K + 1)/S), floor((r - 1 + P)/S)] n [0, Xo).
static Range bwd_window(Range in, int64_t Xo, int K, int S, int P) {
    Range r;
    if (in.empty()) return r;
    r.lo = std::max<int64_t>(0, -floor_div(-(in.lo + P - K + 1), S));
    r.hi = std::min<int64_t>(Xo, floor_div(in.hi - 1 + P, S) + 1);
    return r;
}

static DimSplit split_nocheck(int64_t X, int K, int S, int P, int parts, int idx) {
    DimSplit d;
    d.X = X;
    d.Xo = (X + 2 * P - K) / S + 1;
    d.parts = parts;
    d.idx = idx;
    d.in = blocked(X, parts, idx);
    d.out = blocked(d.Xo, parts, idx);
    Range fw = fwd_window(d.out, X, K, S, P);
    d.xbuf.lo = fw.empty() ? d.in.lo : std::min(d.in.lo, fw.lo);
    d.xbuf.hi = fw.empty() ? d.in.hi : std::max(d.in.hi, fw.hi);
    Range bw = bwd_window(d.in, d.Xo, K, S, P);
    d.dbuf.lo = bw.empty() ? d.out.lo : std::min(d.out.lo, bw.lo);
    d.dbuf.hi = bw.empty() ? d.out.hi : std::max(d.out.hi, bw.hi);
    return d;
}

DimSplit make_split(int64_t X, int K, int S, int P, int parts, int idx) {
    DC_REQUIRE(parts >= 1 && idx >= 0 && idx < parts, DC_ERR_ARG, "bad part index");
    DimSplit d = split_nocheck(X, K, S, P, parts, idx);
    DC_REQUIRE(!d.in.empty() && !d.out.empty(), DC_ERR_PARTITION,
               "%d-way split of extent %lld (output %lld) leaves part %d empty", parts,
               (long long)X, (long long)d.Xo, idx);
    // Halos must come from the adjacent part only (PAPER.md:145 degenerate case).
    if (idx > 0) {
        Range nb_in = blocked(X, parts, idx - 1), nb_out = blocked(d.Xo, parts, idx - 1);
        DC_REQUIRE(d.xbuf.lo >= nb_in.lo && d.dbuf.lo >= nb_out.lo, DC_ERR_PARTITION,
                   "part %d of a %d-way split of %lld needs a halo wider than its neighbour "
                   "(PAPER.md:145: spatial extent ~ kernel size)", idx, parts, (long long)X);
    }
    if (idx + 1 < parts) {
        Range nb_in = blocked(X, parts, idx + 1), nb_out = blocked(d.Xo, parts, idx + 1);
        DC_REQUIRE(d.xbuf.hi <= nb_in.hi && d.dbuf.hi <= nb_out.hi, DC_ERR_PARTITION,
                   "part %d of a %d-way split of %lld needs a halo wider than its neighbour "
                   "(PAPER.md:145: spatial extent ~ kernel size)", idx, parts, (long long)X);
    }
    return d;
}

bool grid_valid(const ConvGeom &g, Grid grid, std::string *why) {
    try {
        DC_REQUIRE(grid.pn >= 1 && grid.ph >= 1 && grid.pw >= 1, DC_ERR_PARTITION, "bad grid");
        DC_REQUIRE(grid.pn <= g.N, DC_ERR_PARTITION, "p_N=%d > N=%lld", grid.pn, (long long)g.N);
        for (int i = 0; i < grid.ph; ++i) make_split(g.H, g.K, g.S, g.P, grid.ph, i);
        for (int i = 0; i < grid.pw; ++i) make_split(g.W, g.K, g.S, g.P, grid.pw, i);
    } catch (const Error &e) {
        if (why) *why = e.what();
        return false;
    }
    return true;
}

// Block (dh, dw) of the receiver's buffer (dh, dw in {-1,0,1}, not both 0).
static void recv_block(const DimSplit &h, const DimSplit &w, bool dy, int dh, int dw, Range &rows,
                       Range &cols) {
    const Range &hb = dy ? h.dbuf : h.xbuf, &ho = dy ? h.out : h.in;
    const Range &wb = dy ? w.dbuf : w.xbuf, &wo = dy ? w.out : w.in;
    rows = dh < 0 ? Range{hb.lo, ho.lo} : dh == 0 ? ho : Range{ho.hi, hb.hi};
    cols = dw < 0 ? Range{wb.lo, wo.lo} : dw == 0 ? wo : Range{wo.hi, wb.hi};
}

static void build_msgs(RankPlan &p, bool dy) {
    const ConvGeom &g = p.g;
    auto &send = dy ? p.dy_send : p.x_send;
    auto &recv = dy ? p.dy_recv : p.x_recv;
    for (int dh = -1; dh <= 1; ++dh)
        for (int dw = -1; dw <= 1; ++dw) {
            if (dh == 0 && dw == 0) continue;
            const int dir = (dh + 1) * 3 + (dw + 1) - ((dh + 1) * 3 + (dw + 1) > 4 ? 1 : 0);
            // (a) I receive block (dh, dw) of my buffer from rank (ih+dh, iw+dw).
            {
                const int sh = p.ih + dh, sw = p.iw + dw;
                if (sh >= 0 && sh < p.grid.ph && sw >= 0 && sw < p.grid.pw) {
                    HaloMsg m;
                    recv_block(p.h, p.w, dy, dh, dw, m.rows, m.cols);
                    if (!m.rows.empty() && !m.cols.empty()) {
                        DimSplit shs = split_nocheck(g.H, g.K, g.S, g.P, p.grid.ph, sh);
                        DimSplit sws = split_nocheck(g.W, g.K, g.S, g.P, p.grid.pw, sw);
                        m.peer = p.grid.rank_of(p.in, sh, sw);
                        m.dir = dir;
                        const Range &sbh = dy ? shs.dbuf : shs.xbuf, &sbw = dy ? sws.dbuf : sws.xbuf;
                        const Range &rbh = dy ? p.h.dbuf : p.h.xbuf, &rbw = dy ? p.w.dbuf : p.w.xbuf;
                        m.src_row0 = m.rows.lo - sbh.lo;
                        m.src_col0 = m.cols.lo - sbw.lo;
                        m.dst_row0 = m.rows.lo - rbh.lo;
                        m.dst_col0 = m.cols.lo - rbw.lo;
                        m.src_hb = sbh.size(); m.src_wb = sbw.size();
                        m.dst_hb = rbh.size(); m.dst_wb = rbw.size();
                        recv.push_back(m);
                    }
                }
            }
            // (b) I send block (dh, dw) of the buffer of rank (ih-dh, iw-dw).
            {
                const int rh = p.ih - dh, rw = p.iw - dw;
                if (rh >= 0 && rh < p.grid.ph && rw >= 0 && rw < p.grid.pw) {
                    DimSplit rhs = split_nocheck(g.H, g.K, g.S, g.P, p.grid.ph, rh);
                    DimSplit rws = split_nocheck(g.W, g.K, g.S, g.P, p.grid.pw, rw);
                    HaloMsg m;
                    recv_block(rhs, rws, dy, dh, dw, m.rows, m.cols);
                    if (!m.rows.empty() && !m.cols.empty()) {
                        m.peer = p.grid.rank_of(p.in, rh, rw);
                        m.dir = dir;
                        const Range &sbh = dy ? p.h.dbuf : p.h.xbuf, &sbw = dy ? p.w.dbuf : p.w.xbuf;
                        const Range &rbh = dy ? rhs.dbuf : rhs.xbuf, &rbw = dy ? rws.dbuf : rws.xbuf;
                        m.src_row0 = m.rows.lo - sbh.lo;
                        m.src_col0 = m.cols.lo - sbw.lo;
                        m.dst_row0 = m.rows.lo - rbh.lo;
                        m.dst_col0 = m.cols.lo - rbw.lo;
                        m.src_hb = sbh.size(); m.src_wb = sbw.size();
                        m.dst_hb = rbh.size(); m.dst_wb = rbw.size();
                        send.push_back(m);
                    }
                }
            }
        }
}

RankPlan make_rank_plan(const ConvGeom &g, Grid grid, int rank) {
    std::string why;
    DC_REQUIRE(grid_valid(g, grid, &why), DC_ERR_PARTITION, "invalid grid (%d,%d,%d): %s",
               grid.pn, grid.ph, grid.pw, why.c_str());
    DC_REQUIRE(rank >= 0 && rank < grid.size(), DC_ERR_ARG, "rank %d outside grid of %d", rank,
               grid.size());
    RankPlan p;
    p.g = g;
    p.grid = grid;
    p.rank = rank;
    grid.coords(rank, p.in, p.ih, p.iw);
    p.nrange = blocked(g.N, grid.pn, p.in);
    p.h = make_split(g.H, g.K, g.S, g.P, grid.ph, p.ih);
    p.w = make_split(g.W, g.K, g.S, g.P, grid.pw, p.iw);
    build_msgs(p, false);
    build_msgs(p, true);
    return p;
}

}  // namespace dc

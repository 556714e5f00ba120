// plan.hpp -- L1: blocked sample/spatial decomposition and halo index math.
//
// Everything here is host integer arithmetic, once per plan
// (SURVEY.md 8(a) a1). Sources:
//   blocked spatial distribution            PAPER.md:112, 91 (reading R8)
//   owned indices q = min ind, r = max ind
//   halo of x / dy
//   stride-adjusted halos                   PAPER.md:145 (reading R5)
//   degenerate partitions rejected          PAPER.md:145 (reading R22)
#pragma once
#include <array>
#include <cstdint>
#include <vector>

#include "common.hpp"

namespace dc {

struct Range {  // half-open [lo, hi)
    int64_t lo = 0, hi = 0;
    int64_t size() const { return hi > lo ? hi - lo : 0; }
    bool empty() const { return hi <= lo; }
};

// Blocked split of [0, extent) into `parts`, remainder to the lowest blocks.
Range blocked(int64_t extent, int parts, int idx);

// One spatial dimension (H or W) of one rank.
struct DimSplit {
    int64_t X = 0, Xo = 0;  // global input / output extent
    int parts = 1, idx = 0;
    Range in;    // owned input indices  [q, r)
    Range out;   // owned output indices [oq, or)
    Range xbuf;  // rows held in the x buffer (owned inputs + fwd halo)
    Range dbuf;  // rows held in the dy buffer (owned outputs + bwd-data halo)
    int64_t x_halo_lo() const { return in.lo - xbuf.lo; }
    int64_t x_halo_hi() const { return xbuf.hi - in.hi; }
    int64_t d_halo_lo() const { return out.lo - dbuf.lo; }
    int64_t d_halo_hi() const { return dbuf.hi - out.hi; }
};

struct ConvGeom {
    int64_t N, C, H, W, F;
    int K, S, P;
    int64_t Ho, Wo;
    int64_t Cp, Fp;  // padded channel counts: multiples of 16 (bf16) / 8 (fp32, 3xTF32)
    int dt = 0;      // 0: bf16 (DC_BF16), 1: fp32 via 3xTF32 (DC_FP32_3XTF32)
    int esz() const { return dt ? 4 : 2; }
};

// Validates and fills Ho/Wo/Cp/Fp. Throws DC_ERR_SHAPE / DC_ERR_UNSUPPORTED.
ConvGeom make_geom(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F, int K, int S, int P, int dt = 0);

// Computes the split of one dimension; throws DC_ERR_PARTITION if the
// partition is invalid for this rank (no output rows, or a halo wider than
// the adjacent rank's block).
DimSplit make_split(int64_t X, int K, int S, int P, int parts, int idx);

// One halo message: a block of global rows x cols (all local samples and
// channels) moving from `src_rank` to `dst_rank`.
struct HaloMsg {
    int peer = -1;                 // the other rank
    int dir = 0;                   // 0..7: (dh+1)*3+(dw+1) skipping 4, from the receiver's view
    Range rows, cols;              // global indices
    int64_t src_row0, src_col0;    // first row/col inside the sender's buffer
    int64_t dst_row0, dst_col0;    // first row/col inside the receiver's buffer
    int64_t src_hb, src_wb;        // sender's buffer extents (rows, cols)
    int64_t dst_hb, dst_wb;        // receiver's buffer extents (rows, cols)
};

struct Grid {
    int pn = 1, ph = 1, pw = 1;
    int size() const { return pn * ph * pw; }
    int rank_of(int in, int ih, int iw) const { return (in * ph + ih) * pw + iw; }
    void coords(int rank, int &in, int &ih, int &iw) const {
        in = rank / (ph * pw);
        ih = (rank / pw) % ph;
        iw = rank % pw;
    }
};

struct RankPlan {
    ConvGeom g;
    Grid grid;
    int rank = 0, in = 0, ih = 0, iw = 0;
    Range nrange;     // owned samples
    DimSplit h, w;
    // Halo traffic of this rank for tensor x (fwd) and dy (bwd-data).
    std::vector<HaloMsg> x_send, x_recv, dy_send, dy_recv;
};

// Full plan of one rank of a grid (validates every rank's split, so that all
// ranks agree on validity). Throws DC_ERR_PARTITION on an invalid grid.
RankPlan make_rank_plan(const ConvGeom &g, Grid grid, int rank);

// True iff the grid is valid for the geometry (no throw).
bool grid_valid(const ConvGeom &g, Grid grid, std::string *why = nullptr);

}  // namespace dc

// perfmodel.cpp -- L4: the paper's performance model and
// the per-layer decomposition choice, host only.
//
//   SR(n)   = alpha + beta n
//   AR(p,n) = min(recursive doubling, ring)           PAPER.md:82 (Thakur; reading R15)
//   FP_l    = C(local) + 2SR(O N C H) + 2SR(O N C W) + 4SR(O^2 N C)
//   BPx_l   = Cx(local) + the same halo terms with F channels          PAPER.md:198-203 (R13)
//   BPw_l   = Cw(local);  BPa_l = AR(P, F C K^2)
//   Cost    = FP + BPx + BPw + BPa adjusted for overlap                PAPER.md:206 (R16)
//   candidates: every (pN,pH,pW) with product P that is valid; ties to
//   sample parallelism first                                           PAPER.md:222 (R17)
// C, Cx, Cw come from an empirical table measured on B200
// with this library's own kernels (bench.py --cost-table); shapes missing
// from the table use a roofline estimate.
#include <cmath>
#include <cstdio>
#include <fstream>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <tuple>
#include <algorithm>
#include <array>
#include <vector>

#include "plan.hpp"

namespace dc {

namespace {
struct Model {
    double alpha = 5e-6;          // s (NVLink P2P latency incl. launch)
    double beta = 1.0 / 700e9;    // s/byte (measured-class NVLink 5 per direction)
    double peak_flops = 1.36e15;  // sustained bf16 dense, MEASURED_PEAKS.json
    double peak_bw = 6.55e12;     // HBM copy, MEASURED_PEAKS.json
    double launch = 4e-6;         // fixed per-kernel overhead
    bool overlap = true;          // reading R16; false: plain sums (halo and allreduce exposed)
    double alpha_w = 0.0;         // extra latency of a strided (east/west, corner) halo message
    std::map<std::tuple<int, int64_t, int64_t, int64_t, int64_t, int64_t, int, int, int>, double> table;
    std::mutex mu;
};
Model &model() {
    static Model m;
    return m;
}

int op_id(const std::string &s) { return s == "fp" ? 0 : s == "bpx" ? 1 : s == "bpw" ? 2 : -1; }

double sr(double words, int word_bytes) {
    Model &m = model();
    return m.alpha + m.beta * words * word_bytes;
}

double ar(int p, double words, int word_bytes) {
    if (p <= 1) return 0.0;
    Model &m = model();
    const double bp = m.beta * word_bytes;
    const double rd = std::ceil(std::log2((double)p)) * (m.alpha + words * bp);
    const double ring = 2.0 * (p - 1) * m.alpha + 2.0 * ((double)(p - 1) / p) * words * bp;
    return std::min(rd, ring);
}

// Local conv time: table entry if present, else roofline estimate.
double conv_time(int op, int64_t n, int64_t c, int64_t h, int64_t w, int64_t f, int K, int S, int P) {
    Model &m = model();
    {
        std::lock_guard<std::mutex> lk(m.mu);
        auto it = m.table.find(std::make_tuple(op, n, c, h, w, f, K, S, P));
        if (it != m.table.end()) return it->second;
    }
    const int64_t ho = (h + 2 * P - K) / S + 1, wo = (w + 2 * P - K) / S + 1;
    // the kernels compute whole 16 x 8 output tiles (conv_v2; 8 x 16 pixel
    // blocks in wgrad_v2): a 4-row shard costs a 16-row tile
    const double tiled = (double)(16 * ((std::max<int64_t>(ho, 1) + 15) / 16)) *
                         (double)(8 * ((std::max<int64_t>(wo, 1) + 7) / 8));
    const double flops = 2.0 * n * f * c * K * K * tiled;
    const double bytes = 2.0 * ((double)n * h * w * c + (double)n * ho * wo * f) + 2.0 * f * c * K * K;
    return m.launch + std::max(flops / m.peak_flops, bytes / m.peak_bw);
}

double halo_terms(int64_t Nl, int64_t Ch, int64_t Hl, int64_t Wl, int O, bool hs, bool ws) {
    if (O == 0) return 0.0;
    const double aw = model().alpha_w;  // NHWC: e/w and corner slabs are strided runs
    double t = 0.0;
    if (ws) t += 2 * (sr((double)O * Nl * Ch * Hl, 2) + aw);
    if (hs) t += 2 * sr((double)O * Nl * Ch * Wl, 2);
    if (hs && ws) t += 4 * (sr((double)O * O * Nl * Ch, 2) + aw);
    return t;
}
}  // namespace

double model_layer_cost(const ConvGeom &g, Grid d, bool include_allreduce) {
    const int64_t Nl = blocked(g.N, d.pn, 0).size();
    const int64_t Hl = blocked(g.H, d.ph, 0).size(), Wl = blocked(g.W, d.pw, 0).size();
    const int O = g.K / 2;
    const double c_fp = conv_time(0, Nl, g.C, Hl, Wl, g.F, g.K, g.S, g.P);
    const double c_bx = conv_time(1, Nl, g.C, Hl, Wl, g.F, g.K, g.S, g.P);
    const double c_bw = conv_time(2, Nl, g.C, Hl, Wl, g.F, g.K, g.S, g.P);
    const double hx = halo_terms(Nl, g.C, Hl, Wl, O, d.ph > 1, d.pw > 1);
    const double hdy = halo_terms(Nl, g.F, Hl, Wl, O, d.ph > 1, d.pw > 1);
    const double bpa = include_allreduce ? ar(d.size(), (double)g.F * g.C * g.K * g.K, 4) : 0.0;
    if (!model().overlap) return c_fp + hx + c_bw + hdy + c_bx + bpa;
    const double fp = std::max(c_fp, hx);
    const double bp = std::max(c_bw, hdy) + std::max(c_bx, bpa);
    return fp + bp;
}

// fix: entries > 0 pin that grid dimension (e.g. {1,0,0}: pure spatial, the
// model picks p_H x p_W); {0,0,0} searches every factorisation of world
bool model_choose(const ConvGeom &g, int world, Grid &best, double &best_t, Grid fix) {
    bool found = false;
    for (int pn = world; pn >= 1; --pn) {
        if (world % pn || (fix.pn > 0 && pn != fix.pn)) continue;
        const int rest = world / pn;
        for (int ph = rest; ph >= 1; --ph) {
            if (rest % ph || (fix.ph > 0 && ph != fix.ph) || (fix.pw > 0 && rest / ph != fix.pw)) continue;
            Grid d{pn, ph, rest / ph};
            if (!grid_valid(g, d)) continue;
            const double t = model_layer_cost(g, d, true);
            // strict '<': enumeration order (larger pN, then larger pH first) is the tie-break
            if (!found || t < best_t) {
                best = d;
                best_t = t;
                found = true;
            }
        }
    }
    return found;
}

// ---------------------------------------------------------------------------
// Parallel execution strategies (PAPER.md:151-153,
// 216-228): Shuffle(D_i, D_j) and the shortest path over per-layer candidates
// ---------------------------------------------------------------------------
namespace {
int64_t overlap(Range a, Range b) { return std::max<int64_t>(0, std::min(a.hi, b.hi) - std::max(a.lo, b.lo)); }
}  // namespace

// Pairwise-exchange all-to-all moving an N x Ch x H x W activation (2-byte
// words) from the blocked distribution of grid A to that of grid B
// (each rank sends the indices it no longer owns): the max
// over ranks of the sum over its peers of SR(words sent to that peer); 0 when
// A == B.
double model_shuffle_cost(int64_t N, int64_t Ch, int64_t H, int64_t W, Grid A, Grid B) {
    if (A.pn == B.pn && A.ph == B.ph && A.pw == B.pw) return 0.0;
    const int P = A.size();
    double worst = 0.0;
    for (int r = 0; r < P; ++r) {
        int an, ah, aw;
        A.coords(r, an, ah, aw);
        const Range rn = blocked(N, A.pn, an), rh = blocked(H, A.ph, ah), rw = blocked(W, A.pw, aw);
        double t = 0.0;
        for (int q = 0; q < P; ++q) {
            if (q == r) continue;
            int bn, bh, bw;
            B.coords(q, bn, bh, bw);
            const double words = (double)overlap(rn, blocked(N, B.pn, bn)) * overlap(rh, blocked(H, B.ph, bh)) *
                                 overlap(rw, blocked(W, B.pw, bw)) * Ch;
            if (words > 0) t += sr(words, 2);
        }
        worst = std::max(worst, t);
    }
    return worst;
}

namespace {
// the activation between parent p and child c: p's output (N, F_p, Ho_p, Wo_p)
double edge_cost(const ConvGeom &p, Grid dp, Grid dc_) {
    // forward (activation) and backward (its gradient) both move
    return model_shuffle_cost(p.N, p.F, p.Ho, p.Wo, dp, dc_) + model_shuffle_cost(p.N, p.F, p.Ho, p.Wo, dc_, dp);
}
}  // namespace

// Strategy over a network given as layers with up to two parents each (-1:
// the network input, provided in the first layer's distribution).
// A line network is solved exactly as a shortest path; with
// branches, the longest remaining path (by the layers' 1-GPU cost, counting
// only unassigned layers) is solved first with the already assigned layers
// fixed, repeated until every layer is assigned. Returns the
// strategy's total: sum of Cost_D(l) + the shuffles on every edge.
double model_strategy(const std::vector<ConvGeom> &L, const std::vector<std::array<int, 2>> &par, int world,
                      int fix_pn, std::vector<Grid> &out) {
    const int n = (int)L.size();
    std::vector<std::vector<Grid>> cand(n);
    std::vector<std::vector<double>> cost(n);
    for (int i = 0; i < n; ++i) {
        for (int pn = world; pn >= 1; --pn) {
            if (world % pn || (fix_pn > 0 && pn != fix_pn)) continue;
            const int rest = world / pn;
            for (int ph = rest; ph >= 1; --ph) {
                if (rest % ph) continue;
                Grid d{pn, ph, rest / ph};
                if (!grid_valid(L[i], d)) continue;
                cand[i].push_back(d);
                cost[i].push_back(model_layer_cost(L[i], d, true));
            }
        }
        DC_REQUIRE(!cand[i].empty(), DC_ERR_PARTITION, "layer %d has no valid grid of %d ranks", i, world);
    }
    std::vector<std::vector<int>> kids(n);
    for (int i = 0; i < n; ++i)
        for (int p : par[i])
            if (p >= 0) {
                DC_REQUIRE(p < i, DC_ERR_ARG, "layer %d: parent %d must come earlier", i, p);
                kids[p].push_back(i);
            }
    std::vector<double> weight(n);
    for (int i = 0; i < n; ++i) weight[i] = model_layer_cost(L[i], Grid{1, 1, 1}, false);
    std::vector<int> assigned(n, -1);  // candidate index
    for (;;) {
        // longest path over unassigned weight (DAG in index order)
        std::vector<double> best(n, -1.0);
        std::vector<int> from(n, -1);
        int end = -1;
        for (int i = 0; i < n; ++i) {
            const double w = assigned[i] < 0 ? weight[i] : 0.0;
            best[i] = w;
            for (int p : par[i])
                if (p >= 0 && best[p] + w > best[i]) best[i] = best[p] + w, from[i] = p;
        }
        for (int i = 0; i < n; ++i)
            if (kids[i].empty() && (end < 0 || best[i] > best[end])) end = i;
        std::vector<int> path;
        for (int i = end; i >= 0; i = from[i]) path.push_back(i);
        std::reverse(path.begin(), path.end());
        bool any = false;
        for (int i : path) any = any || assigned[i] < 0;
        if (!any) {  // every sink path assigned: remaining layers (if any) start new paths
            int u = -1;
            for (int i = 0; i < n && u < 0; ++i)
                if (assigned[i] < 0) u = i;
            if (u < 0) break;
            path.clear();  // a chain down from u through unassigned first children
            for (int i = u; i >= 0;) {
                path.push_back(i);
                int nx = -1;
                for (int k : kids[i])
                    if (assigned[k] < 0) {
                        nx = k;
                        break;
                    }
                i = nx;
            }
        }
        // shortest path along `path`, assigned layers restricted to their grid
        const int m = (int)path.size();
        std::vector<std::vector<double>> dist(m);
        std::vector<std::vector<int>> back(m);
        for (int k = 0; k < m; ++k) {
            const int i = path[k];
            const int nc = (int)cand[i].size();
            dist[k].assign(nc, 1e300);
            back[k].assign(nc, -1);
            for (int a = 0; a < nc; ++a) {
                if (assigned[i] >= 0 && assigned[i] != a) continue;
                if (k == 0) {
                    dist[k][a] = cost[i][a];
                    continue;
                }
                const int ip = path[k - 1];
                for (int b = 0; b < (int)cand[ip].size(); ++b) {
                    if (dist[k - 1][b] >= 1e299) continue;
                    const double t = dist[k - 1][b] + edge_cost(L[ip], cand[ip][b], cand[i][a]) + cost[i][a];
                    if (t < dist[k][a]) dist[k][a] = t, back[k][a] = b;  // strict: first candidate on ties
                }
            }
        }
        int a = 0;
        for (int c = 1; c < (int)dist[m - 1].size(); ++c)
            if (dist[m - 1][c] < dist[m - 1][a]) a = c;
        for (int k = m - 1; k >= 0; --k) {
            assigned[path[k]] = a;
            a = back[k][a];
        }
    }
    out.resize(n);
    double total = 0.0;
    for (int i = 0; i < n; ++i) {
        out[i] = cand[i][assigned[i]];
        total += cost[i][assigned[i]];
        for (int p : par[i])
            if (p >= 0) total += edge_cost(L[p], out[p], out[i]);
    }
    return total;
}

}  // namespace dc

using namespace dc;

extern "C" dc_status_t dc_model_shuffle_cost(int64_t N, int64_t Ch, int64_t H, int64_t W, dc_decomp_t from,
                                             dc_decomp_t to, double *seconds) {
    DC_API_BEGIN
    DC_REQUIRE(seconds && N > 0 && Ch > 0 && H > 0 && W > 0, DC_ERR_ARG, "bad arguments");
    Grid A{from.pn, from.ph, from.pw}, B{to.pn, to.ph, to.pw};
    DC_REQUIRE(A.size() == B.size() && A.size() > 0, DC_ERR_ARG, "grids of different sizes");
    *seconds = model_shuffle_cost(N, Ch, H, W, A, B);
    DC_API_END
}

extern "C" dc_status_t dc_model_strategy(const dc_layer_t *layers, int n, int world, int fix_pn, dc_decomp_t *grids,
                                         double *total_seconds) {
    DC_API_BEGIN
    DC_REQUIRE(layers && grids && n > 0 && world >= 1 && fix_pn >= 0, DC_ERR_ARG, "bad arguments");
    std::vector<ConvGeom> L;
    std::vector<std::array<int, 2>> par;
    for (int i = 0; i < n; ++i) {
        const dc_layer_t &l = layers[i];
        L.push_back(make_geom(l.N, l.C, l.H, l.W, l.F, l.K, l.stride, l.pad));
        par.push_back({l.parent, l.parent2});
        for (int p : par.back())
            if (p >= 0) {
                DC_REQUIRE(p < i, DC_ERR_ARG, "layer %d: parent %d must come earlier", i, p);
                DC_REQUIRE(L[p].N == L[i].N && L[p].F == L[i].C && L[p].Ho == L[i].H && L[p].Wo == L[i].W,
                           DC_ERR_SHAPE, "layer %d does not read layer %d's output shape", i, p);
            }
    }
    std::vector<Grid> out;
    const double t = model_strategy(L, par, world, fix_pn, out);
    for (int i = 0; i < n; ++i) grids[i] = dc_decomp_t{out[i].pn, out[i].ph, out[i].pw};
    if (total_seconds) *total_seconds = t;
    DC_API_END
}

extern "C" dc_status_t dc_model_set_comm(double alpha, double beta) {
    DC_API_BEGIN
    DC_REQUIRE(alpha >= 0 && beta >= 0, DC_ERR_ARG, "alpha, beta must be >= 0");
    model().alpha = alpha;
    model().beta = beta;
    DC_API_END
}

extern "C" dc_status_t dc_model_set_strided_latency(double alpha_w) {
    DC_API_BEGIN
    DC_REQUIRE(alpha_w >= 0, DC_ERR_ARG, "alpha_w must be >= 0");
    model().alpha_w = alpha_w;
    DC_API_END
}

extern "C" dc_status_t dc_model_set_overlap(int overlap) {
    DC_API_BEGIN
    model().overlap = overlap != 0;
    DC_API_END
}

extern "C" dc_status_t dc_model_load_table(const char *path) {
    DC_API_BEGIN
    DC_REQUIRE(path != nullptr, DC_ERR_ARG, "null path");
    std::ifstream f(path);
    DC_REQUIRE(f.good(), DC_ERR_ARG, "cannot open cost table %s", path);
    std::string line;
    std::getline(f, line);
    DC_REQUIRE(line.rfind("op,n,c,h,w,f,k,s,pad,seconds", 0) == 0, DC_ERR_ARG,
               "cost table header must be op,n,c,h,w,f,k,s,pad,seconds (SPEC.md:418)");
    Model &m = model();
    std::lock_guard<std::mutex> lk(m.mu);
    while (std::getline(f, line)) {
        if (line.empty()) continue;
        std::stringstream ss(line);
        std::string op, tok;
        std::getline(ss, op, ',');
        long long v[8];
        for (int i = 0; i < 8; ++i) {
            std::getline(ss, tok, ',');
            v[i] = std::stoll(tok);
        }
        std::getline(ss, tok, ',');
        const int id = op_id(op);
        DC_REQUIRE(id >= 0, DC_ERR_ARG, "unknown op '%s' in cost table", op.c_str());
        m.table[std::make_tuple(id, (int64_t)v[0], (int64_t)v[1], (int64_t)v[2], (int64_t)v[3],
                                (int64_t)v[4], (int)v[5], (int)v[6], (int)v[7])] = std::stod(tok);
    }
    DC_API_END
}

extern "C" dc_status_t dc_model_layer_cost(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F,
                                           int K, int stride, int pad, dc_decomp_t d,
                                           int include_allreduce, double *seconds) {
    DC_API_BEGIN
    DC_REQUIRE(seconds != nullptr, DC_ERR_ARG, "null output");
    ConvGeom g = make_geom(N, C, H, W, F, K, stride, pad);
    Grid grid{d.pn, d.ph, d.pw};
    std::string why;
    DC_REQUIRE(grid_valid(g, grid, &why), DC_ERR_PARTITION, "%s", why.c_str());
    *seconds = model_layer_cost(g, grid, include_allreduce != 0);
    DC_API_END
}

extern "C" dc_status_t dc_model_choose(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F,
                                       int K, int stride, int pad, int world, dc_decomp_t *best,
                                       double *seconds) {
    DC_API_BEGIN
    DC_REQUIRE(best != nullptr && world >= 1, DC_ERR_ARG, "bad arguments");
    ConvGeom g = make_geom(N, C, H, W, F, K, stride, pad);
    Grid b;
    double t = 0;
    DC_REQUIRE(model_choose(g, world, b, t, Grid{0, 0, 0}), DC_ERR_PARTITION, "no valid grid of %d ranks", world);
    *best = dc_decomp_t{b.pn, b.ph, b.pw};
    if (seconds) *seconds = t;
    DC_API_END
}

extern "C" dc_status_t dc_model_choose_fixed(int64_t N, int64_t C, int64_t H, int64_t W, int64_t F,
                                             int K, int stride, int pad, int world, dc_decomp_t fix,
                                             dc_decomp_t *best, double *seconds) {
    DC_API_BEGIN
    DC_REQUIRE(best != nullptr && world >= 1 && fix.pn >= 0 && fix.ph >= 0 && fix.pw >= 0, DC_ERR_ARG,
               "bad arguments");
    ConvGeom g = make_geom(N, C, H, W, F, K, stride, pad);
    Grid b;
    double t = 0;
    DC_REQUIRE(model_choose(g, world, b, t, Grid{fix.pn, fix.ph, fix.pw}), DC_ERR_PARTITION,
               "no valid grid of %d ranks with (%d,%d,%d) fixed", world, fix.pn, fix.ph, fix.pw);
    *best = dc_decomp_t{b.pn, b.ph, b.pw};
    if (seconds) *seconds = t;
    DC_API_END
}

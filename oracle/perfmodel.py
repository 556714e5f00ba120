"""oracle.perfmodel -- TEST INFRASTRUCTURE ONLY.

Direct evaluation of the performance model of arXiv:1903.06681 §V
 in fp64, plus exhaustive enumeration of
(p_N, p_H, p_W) decompositions for the argmin. The product's C++ model
(paper_1903_06681_b200/csrc/perfmodel.cpp) is checked against this.

Readings: R13 (dy halos carry F channels), R15 (collective
model = min(recursive doubling, ring) as SPEC.md:356), R16 (overlap
accounting), R17 (tie-break), R22 (degenerate partitions rejected).
"""
from __future__ import annotations

import functools
import math

from . import out_extent
from .partition import blocked, halo_rows


def sr(n_words: float, alpha: float, beta: float, word_bytes: int = 4) -> float:
    """SR(n) = alpha + beta * n ("the cost to send a message
    between two nodes is alpha + beta n"); beta in s/byte."""
    return alpha + beta * n_words * word_bytes


def ar(p: int, n_words: float, alpha: float, beta: float, word_bytes: int = 4) -> float:
    """AR(p, n) (Thakur et al.; reading R15):
    p = 1 -> 0; else min(recursive doubling ceil(log2 p)(alpha + n beta'),
    ring 2(p-1) alpha + 2 (p-1)/p n beta') with beta' = beta * word_bytes."""
    if p <= 1:
        return 0.0
    bp = beta * word_bytes
    rd = math.ceil(math.log2(p)) * (alpha + n_words * bp)
    ring = 2 * (p - 1) * alpha + 2 * ((p - 1) / p) * n_words * bp
    return min(rd, ring)


def halo_terms(Nl: int, Ch: int, Hl: int, Wl: int, O: int, h_split: bool, w_split: bool,
               alpha: float, beta: float, word_bytes: int, alpha_w: float = 0.0) -> float:
    """The halo part of FP_l / BPx_l:
    2 SR(O N C H) [east/west] + 2 SR(O N C W) [north/south] + 4 SR(O^2 N C)
    [corners]; e/w and corners omitted if W is undivided, n/s and corners if
    H is undivided ("can be omitted"). alpha_w: extra latency of each
    east/west and corner message (strided slabs in NHWC; 0 = the paper's
    model)."""
    t = 0.0
    if O == 0:
        return 0.0
    if w_split:
        t += 2 * (sr(O * Nl * Ch * Hl, alpha, beta, word_bytes) + alpha_w)
    if h_split:
        t += 2 * sr(O * Nl * Ch * Wl, alpha, beta, word_bytes)
    if h_split and w_split:
        t += 4 * (sr(O * O * Nl * Ch, alpha, beta, word_bytes) + alpha_w)
    return t


def layer_cost(layer: dict, grid: tuple[int, int, int], cost, alpha: float, beta: float,
               word_bytes: int = 2, overlap: bool = True, include_allreduce: bool = True,
               alpha_w: float = 0.0) -> dict:
    """Cost_D(l) = FP + BPx + BPw + BPa, local extents of
    the largest (rank 0) block. `cost(op, n, c, h, w, f)` returns the
    empirical local time of op in {"fp", "bpx", "bpw"}.
    Overlap (reading R16): FP = max(C, halo_x); BP = max(Cw, halo_dy) +
    max(Cx, BPa); without overlap the plain sums."""
    N, C, H, W, F, K = (layer[k] for k in ("N", "C", "H", "W", "F", "K"))
    S, P = layer.get("S", 1), layer.get("P", K // 2)
    pn, ph, pw = grid
    Nl = blocked(N, pn, 0)[1]
    Hl, Wl = blocked(H, ph, 0)[1], blocked(W, pw, 0)[1]
    O = K // 2
    c_fp = cost("fp", Nl, C, Hl, Wl, F)
    c_bx = cost("bpx", Nl, C, Hl, Wl, F)
    c_bw = cost("bpw", Nl, C, Hl, Wl, F)
    hx = halo_terms(Nl, C, Hl, Wl, O, ph > 1, pw > 1, alpha, beta, word_bytes, alpha_w)
    hdy = halo_terms(Nl, F, Hl, Wl, O, ph > 1, pw > 1, alpha, beta, word_bytes, alpha_w)
    bpa = ar(pn * ph * pw, F * C * K * K, alpha, beta, 4) if include_allreduce else 0.0
    if overlap:
        fp = max(c_fp, hx)
        bp = max(c_bw, hdy) + max(c_bx, bpa)
    else:
        fp = c_fp + hx
        bp = c_bw + hdy + c_bx + bpa
    return {"fp": fp, "bp": bp, "total": fp + bp, "halo_x": hx, "halo_dy": hdy, "bpa": bpa}


def valid(layer: dict, grid: tuple[int, int, int]) -> bool:
    """Candidate validity (reading R22): p_N <= N, every rank
    owns >= 1 output row/col, and every halo comes from the adjacent rank
    only (halo width <= that neighbour's owned extent), for x and for dy."""
    N, H, W, K = layer["N"], layer["H"], layer["W"], layer["K"]
    S, P = layer.get("S", 1), layer.get("P", K // 2)
    pn, ph, pw = grid
    if pn > N:
        return False
    for ext, parts in ((H, ph), (W, pw)):
        Ho = out_extent(ext, K, S, P)
        if parts > Ho or parts > ext:
            return False
        for idx in range(parts):
            for tensor, full in (("x", ext), ("dy", Ho)):
                lo, hi = halo_rows(parts, idx, ext, K, S, P, tensor)
                if lo:
                    nb = blocked(full, parts, idx - 1) if idx > 0 else (0, 0)
                    if idx == 0 or min(lo) < nb[0]:
                        return False
                if hi:
                    nb = blocked(full, parts, idx + 1) if idx + 1 < parts else (0, 0)
                    if idx + 1 == parts or max(hi) >= nb[1]:
                        return False
    return True


def candidates(P_tot: int) -> list[tuple[int, int, int]]:
    """All (p_N, p_H, p_W) with product P_tot."""
    out = []
    for pn in range(1, P_tot + 1):
        if P_tot % pn:
            continue
        rest = P_tot // pn
        for ph in range(1, rest + 1):
            if rest % ph == 0:
                out.append((pn, ph, rest // ph))
    return out


def choose(layer: dict, P_tot: int, cost, alpha: float, beta: float, **kw):
    """Argmin of Cost over valid candidates by exhaustive enumeration; ties
    -> larger p_N, then larger p_H, then larger p_W ("prefer
    ... sample over spatial parallelism"; reading R17)."""
    best = None
    for g in candidates(P_tot):
        if not valid(layer, g):
            continue
        t = layer_cost(layer, g, cost, alpha, beta, **kw)["total"]
        key = (t, -g[0], -g[1], -g[2])
        if best is None or key < best[0]:
            best = (key, g, t)
    return None if best is None else (best[1], best[2])


# ---------------------------------------------------------------------------
# Parallel execution strategies (SURVEY.md 8(f)
# NEXT-3), written from the definitions: brute-force index ownership for the
# shuffle volumes, exhaustive enumeration for the best strategy.
# ---------------------------------------------------------------------------
def owner(N: int, H: int, W: int, grid, n: int, h: int, w: int) -> int:
    """Rank owning element (n, h, w) under the blocked distribution of grid
    (rank = (i_N p_H + i_H) p_W + i_W, reading R8)."""
    pn, ph, pw = grid

    def idx(x, X, p):
        for i in range(p):
            lo, hi = blocked(X, p, i)
            if lo <= x < hi:
                return i
        raise AssertionError
    return (idx(n, N, pn) * ph + idx(h, H, ph)) * pw + idx(w, W, pw)


@functools.lru_cache(maxsize=None)
def _shuffle_words(N: int, Ch: int, H: int, W: int, A: tuple, B: tuple) -> tuple:
    out = {}
    for n in range(N):
        for h in range(H):
            for w in range(W):
                r, q = owner(N, H, W, A, n, h, w), owner(N, H, W, B, n, h, w)
                if r != q:
                    out[(r, q)] = out.get((r, q), 0) + Ch
    return tuple(sorted(out.items()))


def shuffle_words(N: int, Ch: int, H: int, W: int, A, B) -> dict:
    """{(r, q): words} moved from rank r (owner under A) to rank q (owner
    under B), r != q: every element counted one by one (a
    processor sends the indices it no longer owns). (Memoised: a pure
    function of its arguments.)"""
    return dict(_shuffle_words(N, Ch, H, W, tuple(A), tuple(B)))


def shuffle_cost(N: int, Ch: int, H: int, W: int, A, B, alpha: float, beta: float) -> float:
    """Shuffle(D_i, D_j) as a pairwise-exchange all-to-all: the
    max over ranks of the sum over its peers of SR(words to that peer), 2-byte
    words; 0 when nothing moves."""
    per = {}
    for (r, q), n in shuffle_words(N, Ch, H, W, A, B).items():
        per[r] = per.get(r, 0.0) + sr(n, alpha, beta, 2)
    return max(per.values()) if per else 0.0


def strategy_total(layers: list, parents: list, grids: list, cost, alpha: float, beta: float, **kw) -> float:
    """Model time of a strategy: sum of Cost_D(l) (layer_cost) + on every
    parent -> child edge the shuffle of the parent's output forward and of its
    gradient backward (reading R28)."""
    t = 0.0
    for i, (l, g) in enumerate(zip(layers, grids)):
        t += layer_cost(l, g, cost, alpha, beta, **kw)["total"]
        for p in parents[i]:
            if p >= 0:
                lp = layers[p]
                Ho = out_extent(lp["H"], lp["K"], lp.get("S", 1), lp.get("P", lp["K"] // 2))
                Wo = out_extent(lp["W"], lp["K"], lp.get("S", 1), lp.get("P", lp["K"] // 2))
                t += shuffle_cost(lp["N"], lp["F"], Ho, Wo, grids[p], g, alpha, beta)
                t += shuffle_cost(lp["N"], lp["F"], Ho, Wo, g, grids[p], alpha, beta)
    return t


def strategy_exhaustive(layers: list, parents: list, P_tot: int, cost, alpha: float, beta: float, **kw):
    """The best strategy by enumerating every assignment of valid grids
    (the quantity the paper's shortest path minimises)."""
    import itertools
    cands = [[g for g in candidates(P_tot) if valid(l, g)] for l in layers]
    best = None
    for combo in itertools.product(*cands):
        t = strategy_total(layers, parents, list(combo), cost, alpha, beta, **kw)
        if best is None or t < best[1] - 1e-15:
            best = (list(combo), t)
    return best

"""oracle.partition -- TEST INFRASTRUCTURE ONLY.

Blocked sample/spatial distributions, brute-force halo dependence sets and
the explicitly halo-sliced partitioned convolution of arXiv:1903.06681 §III-A
(PAPER.md:112, 131-145). Pure Python loops over index sets (small cases
only); the arithmetic is delegated to the fp64 Eq. 1-3 oracle on masked
tensors, so a partition that reads outside its halo window changes the
result and fails the partition-invariance pin.
"""
from __future__ import annotations

import numpy as np

from . import conv_bwd_data, conv_bwd_filter, conv_fwd, bn_stats, out_extent


def blocked(extent: int, parts: int, idx: int) -> tuple[int, int]:
    """Blocked distribution of [0, extent) into `parts` contiguous blocks
    ("spatial dimensions are distributed in a blocked manner";
    PAPER.md:91 "minor imbalances due to divisibility"); remainder to the
    lowest indices (reading R8). Half-open [lo, hi)."""
    base, rem = divmod(extent, parts)
    lo = idx * base + min(idx, rem)
    return lo, lo + base + (1 if idx < rem else 0)


def rank_coords(rank: int, grid: tuple[int, int, int]) -> tuple[int, int, int]:
    """Row-major rank -> (i_N, i_H, i_W) (reading R8)."""
    pn, ph, pw = grid
    return rank // (ph * pw), (rank // pw) % ph, rank % pw


def fwd_needed(oq: int, or_: int, K: int, S: int, P: int, H: int) -> set[int]:
    """Brute-force dependence set: every input row h in [0,H) that some owned
    output row i in [oq, or_) reads through Eq. 1 (index S*i + a - P)."""
    return {S * i + a - P for i in range(oq, or_) for a in range(K) if 0 <= S * i + a - P < H}


def bwd_data_needed(q: int, r: int, K: int, S: int, P: int, Ho: int) -> set[int]:
    """Brute-force dependence set of Eq. 3: every dy row i that some owned
    input row u in [q, r) reads ((u + P - a) = S*i exactly, 0 <= i < Ho)."""
    out = set()
    for u in range(q, r):
        for a in range(K):
            t = u + P - a
            if t >= 0 and t % S == 0 and t // S < Ho:
                out.add(t // S)
    return out


def halo_rows(grid_parts: int, idx: int, H: int, K: int, S: int, P: int, tensor: str = "x") -> tuple[set, set]:
    """Halo of one rank along one dimension ("the non-local
    data that processor p requires"): (rows needed from the lower
    neighbour side, rows needed from the upper side), brute force."""
    Ho = out_extent(H, K, S, P)
    if tensor == "x":
        q, r = blocked(H, grid_parts, idx)
        oq, or_ = blocked(Ho, grid_parts, idx)
        need = fwd_needed(oq, or_, K, S, P, H)
    else:  # dy for backward-data: owned dy rows are the owned outputs
        xq, xr = blocked(H, grid_parts, idx)
        q, r = blocked(Ho, grid_parts, idx)
        need = bwd_data_needed(xq, xr, K, S, P, Ho)
    lo = {h for h in need if h < q}
    hi = {h for h in need if h >= r}
    return lo, hi


def _mask_rows_cols(t: np.ndarray, rows: set, cols: set) -> np.ndarray:
    """Copy of t that keeps only the given rows x cols (zero elsewhere)."""
    m = np.zeros_like(t)
    rr = np.array(sorted(rows), dtype=np.int64)
    cc = np.array(sorted(cols), dtype=np.int64)
    if rr.size and cc.size:
        m[:, :, rr[:, None], cc[None, :]] = t[:, :, rr[:, None], cc[None, :]]
    return m


def partitioned_fwd(x, w, S, P, grid):
    """Forward on a (p_N, p_H, p_W) grid by explicit halo slicing
    (PAPER.md:139): each rank sees only x on (its samples) x (owned rows and
    cols + halo), zero elsewhere, and computes its owned output block."""
    N, C, H, W = x.shape
    F, _, K, _ = w.shape
    Ho, Wo = out_extent(H, K, S, P), out_extent(W, K, S, P)
    y = np.zeros((N, F, Ho, Wo))
    pn, ph, pw = grid
    for rank in range(pn * ph * pw):
        iN, iH, iW = rank_coords(rank, grid)
        n0, n1 = blocked(N, pn, iN)
        oh0, oh1 = blocked(Ho, ph, iH)
        ow0, ow1 = blocked(Wo, pw, iW)
        rows = fwd_needed(oh0, oh1, K, S, P, H)
        cols = fwd_needed(ow0, ow1, K, S, P, W)
        xs = _mask_rows_cols(x[n0:n1], rows, cols)
        ys = conv_fwd(xs, w, S, P)
        y[n0:n1, :, oh0:oh1, ow0:ow1] = ys[:, :, oh0:oh1, ow0:ow1]
    return y


def partitioned_bwd_data(dy, w, H, W, S, P, grid):
    """Backward-data on a grid: each rank sees dy only on its owned output
    block plus the dy halo and computes dx on its owned inputs."""
    N, F, Ho, Wo = dy.shape
    _, C, K, _ = w.shape
    dx = np.zeros((N, C, H, W))
    pn, ph, pw = grid
    for rank in range(pn * ph * pw):
        iN, iH, iW = rank_coords(rank, grid)
        n0, n1 = blocked(N, pn, iN)
        h0, h1 = blocked(H, ph, iH)
        w0, w1 = blocked(W, pw, iW)
        rows = bwd_data_needed(h0, h1, K, S, P, Ho)
        cols = bwd_data_needed(w0, w1, K, S, P, Wo)
        dys = _mask_rows_cols(dy[n0:n1], rows, cols)
        dxs = conv_bwd_data(dys, w, H, W, S, P)
        dx[n0:n1, :, h0:h1, w0:w1] = dxs[:, :, h0:h1, w0:w1]
    return dx


def partitioned_bwd_filter(x, dy, K, S, P, grid):
    """Backward-filter on a grid: each rank's partial dW from
    its owned outputs (dy unhaloed) and its x window, then the
    allreduce "over all processors" as a sum in rank order (reading R10)."""
    N, C, H, W = x.shape
    _, F, Ho, Wo = dy.shape
    pn, ph, pw = grid
    dw = np.zeros((F, C, K, K))
    for rank in range(pn * ph * pw):
        iN, iH, iW = rank_coords(rank, grid)
        n0, n1 = blocked(N, pn, iN)
        oh0, oh1 = blocked(Ho, ph, iH)
        ow0, ow1 = blocked(Wo, pw, iW)
        rows = fwd_needed(oh0, oh1, K, S, P, H)
        cols = fwd_needed(ow0, ow1, K, S, P, W)
        xs = _mask_rows_cols(x[n0:n1], rows, cols)
        dys = np.zeros_like(dy[n0:n1])
        dys[:, :, oh0:oh1, ow0:ow1] = dy[n0:n1, :, oh0:oh1, ow0:ow1]
        dw = dw + conv_bwd_filter(xs, dys, K, S, P)
    return dw


def spatial_bn_stats(t, grid):
    """BN statistics aggregated over the ranks holding one sample group's
    spatial shards (reading R11): returns per-i_N (mean, var),
    computed from the owned blocks only, as (count, sum, sum of squared
    deviations) merged in rank order."""
    N, C, H, W = t.shape
    pn, ph, pw = grid
    out = []
    for iN in range(pn):
        n0, n1 = blocked(N, pn, iN)
        parts = []
        for iH in range(ph):
            for iW in range(pw):
                h0, h1 = blocked(H, ph, iH)
                w0, w1 = blocked(W, pw, iW)
                parts.append(t[n0:n1, :, h0:h1, w0:w1])
        cnt = sum(p.shape[0] * p.shape[2] * p.shape[3] for p in parts)
        s = sum(p.sum(axis=(0, 2, 3)) for p in parts)
        mu = s / cnt
        q = sum(((p - mu[None, :, None, None]) ** 2).sum(axis=(0, 2, 3)) for p in parts)
        out.append((mu, q / cnt))
    return out


__all__ = ["blocked", "rank_coords", "fwd_needed", "bwd_data_needed", "halo_rows",
           "partitioned_fwd", "partitioned_bwd_data", "partitioned_bwd_filter",
           "spatial_bn_stats", "bn_stats"]

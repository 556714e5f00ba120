"""Parity at BASELINE.json's full sizes (the bench's mesh2k_n8 layers, N = 8,
and the ResNet-50 layers of configs[1], N = 32; 1 GPU, the kernels and flags
bench.py times) on SAMPLED outputs.

The GPU runs each whole layer (forward with the fused BN statistics,
backward-data, backward-filter); the fp64 oracle then computes, one by one:
  * whole output rows of y (Eq. 1) for the first, a middle and
    the last output row of the first and last sample, from the x rows those
    outputs read (the halo-slicing reading of SURVEY.md §8(c) item 4: a row
    window of the global input, same column padding);
  * whole rows of dx (Eq. 3; strided adjoint, reading R4) from
    the dy rows that reach them;
  * dW entries (Eq. 2) at the corners and the middle of
    (f, c, a, b) from one channel of x and one of dy over all samples;
and the BN statistics of the whole stored y are checked against fp64 sums of
that same y (a property that holds at any size).

Sampling: every row on either side of the 2/4/8-way shard
boundaries plus first / middle / last rows of y and dx (first and last
sample); 4096 random interior points of y (and of dx for the stride-1 "same"
layers), all channels each; all K x K taps of up to 8 x 16 (c, f) pairs of dW
(>= 1024 entries where the layer has them).

Tolerances: element by element within the derived bound of DESIGN.md §7
(tests/gpu_util.py elementwise_bound: bf16 output rounding 2^-9 |o| plus the
fp32 accumulation term over |terms|), which also implies north_star's norms.
"""
from __future__ import annotations

import os
import zlib
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle  # noqa: E402

pytestmark = pytest.mark.gpu

# (name, N, C, H, W, F, K, S, P): a cross-section of bench.py's mesh2k_n8
# stack (reading R20) covering every kernel mode the step uses
LAYERS = [
    ("conv1_1", 8, 18, 2048, 2048, 64, 3, 2, 1),    # 18 -> 32 padded channels, sub-pixel backward-data
    ("conv1_2", 8, 64, 1024, 1024, 64, 3, 1, 1),    # register-accumulated fused BN, resident weights
    ("conv2_1", 8, 64, 1024, 1024, 128, 3, 2, 1),   # stride 2: four phase GEMMs
    ("conv3_2", 8, 256, 256, 256, 256, 3, 1, 1),    # 256-wide N tiles: two epilogue warp groups
    ("conv4_2", 8, 512, 128, 128, 512, 3, 1, 1),    # streamed weights, two N tiles
    ("conv6_2", 8, 512, 32, 32, 512, 3, 1, 1),      # small spatial extent: split-K
    ("pred", 8, 512, 32, 32, 2, 1, 1, 0),           # 1x1, F = 2
    # BASELINE.json configs[1]: the paper's ResNet-50 layers at N = 32
    ("resnet_conv1", 32, 3, 224, 224, 64, 7, 2, 3),
    ("res2a_branch2b", 32, 64, 56, 56, 64, 3, 1, 1),
    ("res3b_branch2a", 32, 512, 28, 28, 128, 1, 1, 0),
]


@pytest.fixture(scope="module")
def dc():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_1903_06681_b200 as dc
    torch.cuda.init()
    return dc


def _fwd_window(i, H, K, S, P):
    """Global input rows [r0, r0 + L) and the local output row i' such that
    the oracle's Eq. 1 on that window (same P) gives global output row i."""
    ip = min(i, -(-P // S))  # local row whose window starts at or after local row 0
    r0 = S * (i - ip)
    L = min(S * ip - P + K, H - r0)
    return r0, L, ip


def _bwd_window(u, Ho, H, K, S, P):
    """dy rows [i0, i1) reaching dx row u, the local dx height Hl and row u'
    such that the oracle's Eq. 3 on that window gives global dx row u."""
    i0 = max(0, -((K - 1 - P - u) // S))           # ceil((u + P - K + 1) / S), clamped
    i1 = min(Ho, (u + P) // S + 1)
    L = i1 - i0
    up = u - S * i0
    for Hl in range(max(1, S * (L - 1) + K - 2 * P), S * (L - 1) + K - 2 * P + S + up + 2):
        if Hl > up and oracle.out_extent(Hl, K, S, P) == L:
            return i0, i1, Hl, up
    raise AssertionError("no window")


def edge_rows(X):
    """Rows 0, X/2, X-1 and both sides of every block boundary of the 2-, 4-
    and 8-way blocked splits of X (where the shards of the bench's spatial
    decompositions meet)."""
    rows = {0, X // 2, X - 1}
    for parts in (2, 4, 8):
        base, rem = divmod(X, parts)
        lo = 0
        for k in range(parts - 1):
            lo += base + (1 if k < rem else 0)
            rows.update({lo - 1, lo})
    return sorted(r for r in rows if 0 <= r < X)


def _rel_l2(g, o):
    return float(np.linalg.norm((g - o).ravel()) / max(np.linalg.norm(o.ravel()), 1e-300))


@pytest.mark.parametrize("layer", LAYERS, ids=[l[0] for l in LAYERS])
def test_full_size_sampled_parity(dc, layer):
    import torch
    from tests.gpu_util import assert_elementwise, elementwise_bound, empty_dense

    name, N, C, H, W, F, K, S, P = layer
    Ho, Wo = oracle.out_extent(H, K, S, P), oracle.out_extent(W, K, S, P)
    plan = dc.dc_plan_create_virtual(N, C, H, W, F, K, S, P, (1, 1, 1), 0)
    try:
        xd, yd = dc.dc_plan_query(plan, dc.DC_X), dc.dc_plan_query(plan, dc.DC_Y)
        dyd, dxd = dc.dc_plan_query(plan, dc.DC_DY), dc.dc_plan_query(plan, dc.DC_DX)
        assert (xd["halo_n"], xd["halo_s"], xd["halo_w"], xd["halo_e"]) == (0, 0, 0, 0)
        gen = dict(c_pad=xd["c_pad"], dtype=torch.bfloat16, device="cuda")
        xb = datagen.gen_block_nhwc_torch((N, C, H, W), datagen.SEED, datagen.TID_X, **gen).contiguous()
        dyb = datagen.gen_block_nhwc_torch((N, F, Ho, Wo), datagen.SEED, datagen.TID_DY,
                                           c_pad=dyd["c_pad"], dtype=torch.bfloat16, device="cuda").contiguous()
        w = datagen.gen_w(F, C, K)
        wnp = np.zeros((F, K, K, xd["c_pad"]))
        wnp[..., :C] = w.transpose(0, 2, 3, 1)
        wb = torch.tensor(wnp, dtype=torch.bfloat16, device="cuda").contiguous()
        y, dx = empty_dense(yd), empty_dense(dxd)
        assert y.shape[:3] == (N, Ho, Wo) and dx.shape[:3] == (N, H, W)
        dw = torch.full((F, K, K, C), float("nan"), dtype=torch.float32, device="cuda")
        mean = torch.zeros(F, dtype=torch.float64, device="cuda")
        var = torch.zeros(F, dtype=torch.float64, device="cuda")
        dc.dc_conv_fwd(plan, xb, wb, y, dc.DC_BN_STATS)
        dc.dc_bn_spatial_stats(plan, y, mean, var, dc.DC_BN_LOCAL | dc.DC_BN_FROM_FWD)
        dc.dc_conv_bwd_data(plan, dyb, wb, dx, 0)
        dc.dc_conv_bwd_filter(plan, xb, dyb, dw, 0)
        torch.cuda.synchronize()
        del xb, dyb

        # BN statistics of the whole stored y (property at any size)
        y64 = y[..., :F].double()
        m_ref = y64.mean(dim=(0, 1, 2))
        v_ref = ((y64 - m_ref) ** 2).mean(dim=(0, 1, 2))
        yabs = y64.abs().mean(dim=(0, 1, 2)).cpu().numpy()
        y2 = (y64 ** 2).mean(dim=(0, 1, 2)).cpu().numpy()
        u = 2.0 ** -24
        d = 40  # fused-path depth
        tm = d * u * yabs
        tv = d * u * y2 + 2 * np.abs(m_ref.cpu().numpy()) * tm
        assert (np.abs(mean.cpu().numpy() - m_ref.cpu().numpy()) <= tm + 1e-12).all(), f"{name}: BN mean"
        assert (np.abs(var.cpu().numpy() - v_ref.cpu().numpy()) <= tv + 1e-12).all(), f"{name}: BN var"
        del y64

        # ---- rows: every shard-edge row of the 2/4/8-way H splits, first /
        # middle / last, of the first and last sample, element-wise ----
        aw = np.abs(w)
        for n in (0, N - 1):
            for i in edge_rows(Ho):
                r0, L, ip = _fwd_window(i, H, K, S, P)
                xw = datagen.gen_x(N, C, H, W, n=(n, n + 1), h=(r0, r0 + L))
                ref = oracle.conv_fwd(xw, w, S, P, rows=(ip, ip + 1))[0, :, ip, :]        # F x Wo
                Sb = oracle.conv_fwd(np.abs(xw), aw, S, P, rows=(ip, ip + 1))[0, :, ip, :]
                got = y[n, i, :, :F].double().cpu().numpy().T
                assert_elementwise(f"{name}: y[{n}, :, {i}, :]", got, ref,
                                   elementwise_bound(ref, Sb, C * K * K, 16, True))
            for uu in edge_rows(H):
                i0, i1, Hl, up = _bwd_window(uu, Ho, H, K, S, P)
                dyw = datagen.gen_dy(N, F, Ho, Wo, n=(n, n + 1), h=(i0, i1))
                ref = oracle.conv_bwd_data(dyw, w, Hl, W, S, P, rows=(up, up + 1))[0, :, up, :]  # C x W
                Sb = oracle.conv_bwd_data(np.abs(dyw), aw, Hl, W, S, P, rows=(up, up + 1))[0, :, up, :]
                got = dx[n, uu, :, :C].double().cpu().numpy().T
                assert_elementwise(f"{name}: dx[{n}, :, {uu}, :]", got, ref,
                                   elementwise_bound(ref, Sb, F * K * K, 16, True))

        # ---- 4096 random interior points of y (and of dx for stride 1):
        # all channels of each, from the K x K window the point reads ----
        rng = np.random.default_rng(zlib.crc32(name.encode()))
        npts = 4096
        pts = [(int(rng.integers(N)), int(rng.integers(K, max(K + 1, Ho - K))), int(rng.integers(K, max(K + 1, Wo - K))))
               for _ in range(npts)]
        win = np.stack([datagen.gen_x(N, C, H, W, n=(n, n + 1), h=(S * i - P, S * i - P + K),
                                      w=(S * j - P, S * j - P + K))[0] for n, i, j in pts])   # pts x C x K x K
        ref = oracle.conv_fwd(win, w, 1, 0)[:, :, 0, 0]                                      # pts x F
        Sb = oracle.conv_fwd(np.abs(win), aw, 1, 0)[:, :, 0, 0]
        idx = torch.tensor(pts, device="cuda")
        got = y[idx[:, 0], idx[:, 1], idx[:, 2], :F].double().cpu().numpy()
        assert_elementwise(f"{name}: y at {npts} interior points", got, ref,
                           elementwise_bound(ref, Sb, C * K * K, 16, True))
        del win
        if S == 1 and P == K // 2:
            pts = [(int(rng.integers(N)), int(rng.integers(K, max(K + 1, H - K))), int(rng.integers(K, max(K + 1, W - K))))
                   for _ in range(npts)]
            win = np.stack([datagen.gen_dy(N, F, Ho, Wo, n=(n, n + 1), h=(u - P, u + P + 1), w=(v - P, v + P + 1))[0]
                            for n, u, v in pts])                                                  # pts x F x K x K
            # local "same" problem of extent K: its centre dx is the global dx[u, v]
            ref = oracle.conv_bwd_data(win, w, K, K, 1, P)[:, :, P, P]                            # pts x C
            Sb = oracle.conv_bwd_data(np.abs(win), aw, K, K, 1, P)[:, :, P, P]
            idx = torch.tensor(pts, device="cuda")
            got = dx[idx[:, 0], idx[:, 1], idx[:, 2], :C].double().cpu().numpy()
            assert_elementwise(f"{name}: dx at {npts} interior points", got, ref,
                               elementwise_bound(ref, Sb, F * K * K, 16, True))
            del win

        # ---- >= 1024 dW entries: all K x K taps of enough (c, f) pairs,
        # each an N Ho Wo dot product over whole channels (Eq. 2) ----
        dwh = dw.double().cpu().numpy()  # F K K C
        pairs = -(-min(1024, F * C * K * K) // (K * K))   # (c, f) pairs for >= 1024 entries
        nf = min(F, max(1, int(np.ceil(np.sqrt(pairs)))))
        nc = min(C, -(-pairs // nf))
        nf = min(F, -(-pairs // nc))
        cs = sorted(set(int(c) for c in np.linspace(0, C - 1, nc).round()))
        fs = sorted(set(int(f) for f in np.linspace(0, F - 1, nf).round()))
        gen_dev = dict(dtype=torch.float64, device="cuda")
        # the selected channels of x and dy, stacked: ONE oracle call computes
        # every (f, c) pair (Eq. 2 is independent per pair; its OpenMP loop
        # runs over the pairs)
        xs = np.concatenate([datagen.gen_block_nhwc_torch((N, C, H, W), datagen.SEED, datagen.TID_X, c=(c, c + 1),
                                                          **gen_dev).permute(0, 3, 1, 2).cpu().numpy() for c in cs], 1)
        dys = np.concatenate([datagen.gen_block_nhwc_torch((N, F, Ho, Wo), datagen.SEED, datagen.TID_DY,
                                                           c=(f, f + 1), **gen_dev).permute(0, 3, 1, 2).cpu().numpy()
                              for f in fs], 1)
        ref = oracle.conv_bwd_filter(xs, dys, K, S, P)                     # nf x nc x K x K
        Sb = oracle.conv_bwd_filter(np.abs(xs), np.abs(dys), K, S, P)
        del xs, dys
        nent = 0
        for a_, f in enumerate(fs):
            for b_, c in enumerate(cs):
                got = dwh[f, :, :, c]
                assert_elementwise(f"{name}: dW[{f}, {c}]", got, ref[a_, b_],
                                   elementwise_bound(ref[a_, b_], Sb[a_, b_], N * Ho * Wo, 16, False, extra_adds=300))
                nent += K * K
        assert nent >= min(1024, F * C * K * K)
    finally:
        dc.dc_plan_destroy(plan)


"""Pins of the fp64 CPU oracle against things other than itself (paper worked
values, closed forms, library special cases, adjointness, finite
differences, brute force in the paper's own notation, partition invariance).
CPU only."""
import itertools
import json
import os

import numpy as np
import pytest
import torch

import oracle
from oracle import partition as part
from oracle import perfmodel as pm
import datagen

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_values.json")))
rng = np.random.default_rng(1903)


def _fixture_tensor(spec, shape):
    if spec == "ones":
        return np.ones(shape)
    return np.array(spec, dtype=np.float64).reshape(shape)


@pytest.mark.parametrize("name", ["ones_3x3_same", "asymmetric_xcorr"])
def test_worked_values(name):
    g = GOLD[name]
    x = _fixture_tensor(g["x"], (g["N"], g["C"], g["H"], g["W"]))
    w = _fixture_tensor(g["w"], (g["F"], g["C"], g["K"], g["K"]))
    y = oracle.conv_fwd(x, w, g["S"], g["P"])
    np.testing.assert_array_equal(y[0, 0], np.array(g["y"], dtype=np.float64))


def test_identity_and_zero_filters():
    # K=1, w=1 -> y == x; w = 0 -> y = 0
    x = rng.standard_normal((2, 1, 5, 4))
    np.testing.assert_array_equal(oracle.conv_fwd(x, np.ones((1, 1, 1, 1)), 1, 0), x)
    assert not oracle.conv_fwd(x, np.zeros((3, 1, 3, 3)), 1, 1).any()
    # identity 1x1 -> dx == dy
    dy = rng.standard_normal((2, 1, 5, 4))
    np.testing.assert_array_equal(oracle.conv_bwd_data(dy, np.ones((1, 1, 1, 1)), 5, 4, 1, 0), dy)


def test_dw_scalar_special_case():
    # N=C=F=1, K=1 -> dw = sum x * dy
    x = rng.standard_normal((1, 1, 2, 2))
    dy = rng.standard_normal((1, 1, 2, 2))
    dw = oracle.conv_bwd_filter(x, dy, 1, 1, 0)
    assert dw.shape == (1, 1, 1, 1)
    assert abs(dw[0, 0, 0, 0] - float((x * dy).sum())) < 1e-15


def _eq1_bruteforce(x, w):
    """Eq. 1 exactly as printed: S = 1, same padding,
    a, b in [-O, O], w index a+O, out-of-range x = 0."""
    N, C, H, W = x.shape
    F, _, K, _ = w.shape
    O = K // 2
    y = np.zeros((N, F, H, W))
    for k, f, i, j in itertools.product(range(N), range(F), range(H), range(W)):
        s = 0.0
        for c in range(C):
            for a in range(-O, O + 1):
                for b in range(-O, O + 1):
                    if 0 <= i + a < H and 0 <= j + b < W:
                        s += x[k, c, i + a, j + b] * w[f, c, a + O, b + O]
        y[k, f, i, j] = s
    return y


def _eq2_bruteforce(x, dy, K):
    """Eq. 2 as printed, S=1 same padding, a,b in [0,K)."""
    N, C, H, W = x.shape
    F = dy.shape[1]
    O = K // 2
    dw = np.zeros((F, C, K, K))
    for f, c, a, b in itertools.product(range(F), range(C), range(K), range(K)):
        s = 0.0
        for k in range(N):
            for i in range(H):
                for j in range(W):
                    if 0 <= i + a - O < H and 0 <= j + b - O < W:
                        s += dy[k, f, i, j] * x[k, c, i + a - O, j + b - O]
        dw[f, c, a, b] = s
    return dw


def _eq3_bruteforce(dy, w):
    """Eq. 3 as printed, S=1 same padding, a,b in [-O,O]."""
    N, F, H, W = dy.shape
    _, C, K, _ = w.shape
    O = K // 2
    dx = np.zeros((N, C, H, W))
    for k, c, i, j in itertools.product(range(N), range(C), range(H), range(W)):
        s = 0.0
        for f in range(F):
            for a in range(-O, O + 1):
                for b in range(-O, O + 1):
                    if 0 <= i - a < H and 0 <= j - b < W:
                        s += dy[k, f, i - a, j - b] * w[f, c, a + O, b + O]
        dx[k, c, i, j] = s
    return dx


@pytest.mark.parametrize("K", [1, 3, 5])
def test_brute_force_paper_notation(K):
    x = rng.standard_normal((2, 3, 6, 5))
    w = rng.standard_normal((2, 3, K, K))
    dy = rng.standard_normal((2, 2, 6, 5))
    np.testing.assert_allclose(oracle.conv_fwd(x, w, 1, K // 2), _eq1_bruteforce(x, w), rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.conv_bwd_filter(x, dy, K, 1, K // 2), _eq2_bruteforce(x, dy, K), rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.conv_bwd_data(dy, w, 6, 5, 1, K // 2), _eq3_bruteforce(dy, w), rtol=0, atol=1e-12)


SHAPES = [  # (N, C, H, W, F, K, S, P)
    (2, 3, 9, 7, 4, 3, 1, 1), (1, 2, 11, 10, 3, 3, 2, 1), (2, 2, 12, 9, 2, 5, 1, 2),
    (1, 3, 15, 13, 2, 7, 2, 3), (2, 4, 7, 8, 3, 1, 1, 0), (1, 2, 10, 9, 3, 3, 1, 0),
    (1, 2, 9, 9, 2, 3, 2, 0), (1, 1, 8, 8, 1, 1, 2, 0),
]


@pytest.mark.parametrize("shape", SHAPES)
def test_against_torch_fp64(shape):
    """Library special case: torch CPU float64 conv2d and its autograd are an
    independent implementation of the same cross-correlation."""
    N, C, H, W, F, K, S, P = shape
    x = rng.standard_normal((N, C, H, W))
    w = rng.standard_normal((F, C, K, K))
    y = oracle.conv_fwd(x, w, S, P)
    tx = torch.tensor(x, requires_grad=True)
    tw = torch.tensor(w, requires_grad=True)
    ty = torch.nn.functional.conv2d(tx, tw, stride=S, padding=P)
    np.testing.assert_allclose(y, ty.detach().numpy(), rtol=0, atol=1e-12)
    g = rng.standard_normal(y.shape)
    ty.backward(torch.tensor(g))
    np.testing.assert_allclose(oracle.conv_bwd_data(g, w, H, W, S, P), tx.grad.numpy(), rtol=0, atol=1e-12)
    np.testing.assert_allclose(oracle.conv_bwd_filter(x, g, K, S, P), tw.grad.numpy(), rtol=0, atol=1e-11)


@pytest.mark.parametrize("shape", SHAPES)
def test_adjoint_identities(shape):
    """<conv(x), g> = <x, conv^T(g)> = <w, dW(x, g)> (north_star)."""
    N, C, H, W, F, K, S, P = shape
    x = rng.standard_normal((N, C, H, W))
    w = rng.standard_normal((F, C, K, K))
    y = oracle.conv_fwd(x, w, S, P)
    g = rng.standard_normal(y.shape)
    a = float((y * g).sum())
    b = float((x * oracle.conv_bwd_data(g, w, H, W, S, P)).sum())
    c = float((w * oracle.conv_bwd_filter(x, g, K, S, P)).sum())
    scale = max(abs(a), 1.0)
    assert abs(a - b) / scale < 1e-10
    assert abs(a - c) / scale < 1e-10


def test_finite_differences():
    """Central FD of L = sum y*g, step 1e-6, rel err <= 1e-6."""
    N, C, H, W, F, K, S, P = 1, 2, 5, 5, 2, 3, 1, 1
    x = rng.standard_normal((N, C, H, W))
    w = rng.standard_normal((F, C, K, K))
    g = rng.standard_normal((N, F, 5, 5))
    L = lambda xx, ww: float((oracle.conv_fwd(xx, ww, S, P) * g).sum())
    dw = oracle.conv_bwd_filter(x, g, K, S, P)
    dx = oracle.conv_bwd_data(g, w, H, W, S, P)
    h = 1e-6
    for idx in [(0, 0, 0, 0), (1, 1, 2, 1), (0, 1, 1, 2)]:
        e = np.zeros_like(w); e[idx] = h
        fd = (L(x, w + e) - L(x, w - e)) / (2 * h)
        assert abs(fd - dw[idx]) <= 1e-6 * max(1.0, abs(dw[idx]))
    for idx in [(0, 0, 0, 0), (0, 1, 4, 2), (0, 0, 2, 2)]:
        e = np.zeros_like(x); e[idx] = h
        fd = (L(x + e, w) - L(x - e, w)) / (2 * h)
        assert abs(fd - dx[idx]) <= 1e-6 * max(1.0, abs(dx[idx]))


def test_row_range_and_entry_match_full():
    N, C, H, W, F, K, S, P = 2, 3, 10, 9, 4, 3, 2, 1
    x = rng.standard_normal((N, C, H, W)); w = rng.standard_normal((F, C, K, K))
    y = oracle.conv_fwd(x, w, S, P)
    yr = oracle.conv_fwd(x, w, S, P, rows=(1, 3))
    np.testing.assert_array_equal(yr[:, :, 1:3], y[:, :, 1:3])
    g = rng.standard_normal(y.shape)
    dw = oracle.conv_bwd_filter(x, g, K, S, P)
    assert oracle.conv_bwd_filter_entry(x, g, K, S, P, 3, 2, 1, 0) == dw[3, 2, 1, 0]
    dx = oracle.conv_bwd_data(g, w, H, W, S, P)
    dxr = oracle.conv_bwd_data(g, w, H, W, S, P, rows=(4, 7))
    np.testing.assert_array_equal(dxr[:, :, 4:7], dx[:, :, 4:7])


# ---------------- halo / partition pins ----------------

def test_halo_examples_from_paper_and_spec():
    g = GOLD["halo_2x2_grid"]
    lo, hi = part.halo_rows(g["ph"], 0, g["H"], g["K"], g["S"], g["P"])
    assert sorted(lo) == g["rank00_rows_lo"] and sorted(hi) == g["rank00_rows_hi"]
    for key in ("halo_stride2", "halo_conv1_2way"):
        g = GOLD[key]
        for r in range(g["parts"]):
            lo, hi = part.halo_rows(g["parts"], r, g["H"], g["K"], g["S"], g["P"])
            assert sorted(lo) == g[f"rank{r}_lo"], (key, r)
            assert sorted(hi) == g[f"rank{r}_hi"], (key, r)


@pytest.mark.parametrize("parts", [2, 3, 4])
def test_k1_needs_no_halo(parts):
    # PAPER.md:139 "when K=1, O=0 and no halo is needed"
    for r in range(parts):
        for t in ("x", "dy"):
            assert part.halo_rows(parts, r, 13, 1, 1, 0, t) == (set(), set())


def test_blocked_examples():
    # SPEC.md:124-126
    assert [part.blocked(8, 2, i) for i in range(2)] == [(0, 4), (4, 8)]
    assert [part.blocked(7, 2, i) for i in range(2)] == [(0, 4), (4, 7)]
    assert part.blocked(5, 1, 0) == (0, 5)


GRIDS = [(1, 1, 1), (1, 2, 1), (1, 1, 2), (2, 2, 1), (1, 2, 2), (1, 3, 2), (2, 1, 3), (1, 4, 1)]


@pytest.mark.parametrize("shape", SHAPES[:6])
@pytest.mark.parametrize("grid", GRIDS)
def test_partition_invariance(shape, grid):
    """the partitioned algorithm 'exactly replicates convolution
    as if it were performed on a single GPU'. In fp64 with the same summation
    order y and dx are bitwise equal; dW (different reduction tree) to 1e-12."""
    N, C, H, W, F, K, S, P = shape
    if grid[0] > N:
        pytest.skip("p_N > N")
    Ho, Wo = oracle.out_extent(H, K, S, P), oracle.out_extent(W, K, S, P)
    if grid[1] > Ho or grid[2] > Wo:
        pytest.skip("more parts than output rows")
    x = rng.standard_normal((N, C, H, W)); w = rng.standard_normal((F, C, K, K))
    dy = rng.standard_normal((N, F, Ho, Wo))
    np.testing.assert_array_equal(part.partitioned_fwd(x, w, S, P, grid), oracle.conv_fwd(x, w, S, P))
    np.testing.assert_array_equal(part.partitioned_bwd_data(dy, w, H, W, S, P, grid),
                                  oracle.conv_bwd_data(dy, w, H, W, S, P))
    np.testing.assert_allclose(part.partitioned_bwd_filter(x, dy, K, S, P, grid),
                               oracle.conv_bwd_filter(x, dy, K, S, P), rtol=0, atol=1e-12)


def test_partition_detects_a_missing_halo_row():
    """The pin has teeth: drop one needed halo row and y changes."""
    N, C, H, W, F, K, S, P = 1, 2, 8, 6, 2, 3, 1, 1
    x = rng.standard_normal((N, C, H, W)); w = rng.standard_normal((F, C, K, K))
    need = part.fwd_needed(0, 4, K, S, P, H) - {4}
    xs = part._mask_rows_cols(x, need, set(range(W)))
    assert not np.array_equal(oracle.conv_fwd(xs, w, S, P)[:, :, :4], oracle.conv_fwd(x, w, S, P)[:, :, :4])


# ---------------- BN statistics pins ----------------

def test_bn_stats_pins():
    t = rng.standard_normal((3, 4, 5, 6))
    mu, var = oracle.bn_stats(t)
    # library special case: numpy mean / var(ddof=0)
    np.testing.assert_allclose(mu, t.mean(axis=(0, 2, 3)), rtol=0, atol=1e-14)
    np.testing.assert_allclose(var, t.var(axis=(0, 2, 3)), rtol=0, atol=1e-14)
    # constant input -> var 0, mean = constant
    mu, var = oracle.bn_stats(np.full((2, 3, 4, 4), 0.75))
    assert np.all(mu == 0.75) and np.all(var == 0)


@pytest.mark.parametrize("grid", [(1, 2, 1), (1, 2, 2), (2, 3, 1), (1, 1, 3)])
def test_bn_spatial_equals_serial(grid):
    # spatially aggregated stats equal serial stats to 1e-12
    t = rng.standard_normal((4, 3, 9, 7))
    for iN, (mu, var) in enumerate(part.spatial_bn_stats(t, grid)):
        n0, n1 = part.blocked(4, grid[0], iN)
        m2, v2 = oracle.bn_stats(t[n0:n1])
        np.testing.assert_allclose(mu, m2, rtol=0, atol=1e-12)
        np.testing.assert_allclose(var, v2, rtol=0, atol=1e-12)


# ---------------- perf-model pins ----------------

def test_perfmodel_closed_forms():
    g = GOLD["perfmodel_sr"]
    assert abs(pm.sr(g["n"], g["alpha"], g["beta"], g["word_bytes"]) - g["seconds"]) < 1e-15
    assert pm.sr(0, 1e-6, 1e-9) == 1e-6
    assert pm.ar(1, 1e6, 1e-6, 1e-9) == 0.0
    assert abs(pm.ar(2, 1e6, 1e-6, 1e-9, 4) - (1e-6 + 4e-3)) < 1e-15
    g = GOLD["perfmodel_halo_words_conv1"]
    Hl = part.blocked(g["H"], 2, 0)[1]
    O = g["K"] // 2
    assert O * g["N"] * g["C"] * Hl == g["words_ew"]
    g = GOLD["mesh_sample_bytes"]
    assert g["H"] * g["W"] * g["C"] * g["word_bytes"] / 2 ** 20 == g["mib"]


def test_perfmodel_halo_branches_pinned():
    """halo_terms' east/west, north/south and corner branches against the
    hand-priced SPEC.md:370 / PAPER.md:193-194 messages (golden values)."""
    g = GOLD["perfmodel_halo_ew_conv1"]
    a = (g["N"], g["C"], g["H_l"], g["W_l"], g["O"])
    kw = dict(alpha=g["alpha"], beta=g["beta"], word_bytes=g["word_bytes"])
    ew = pm.halo_terms(*a, h_split=False, w_split=True, **kw)
    ns = pm.halo_terms(*a, h_split=True, w_split=False, **kw)
    both = pm.halo_terms(*a, h_split=True, w_split=True, **kw)
    assert abs(ew - g["seconds_ew_only"]) < 1e-15
    assert abs(ns - g["seconds_ns_only"]) < 1e-15
    assert abs(both - g["seconds_both"]) < 1e-15
    assert abs((both - ew - ns) - g["seconds_corners"]) < 1e-15
    # the strided extra latency lands on the 2 e/w and 4 corner messages only
    aw = 3e-6
    assert abs(pm.halo_terms(*a, True, True, alpha_w=aw, **kw) - (g["seconds_both"] + 6 * aw)) < 1e-15
    assert abs(pm.halo_terms(*a, True, False, alpha_w=aw, **kw) - g["seconds_ns_only"]) < 1e-15


def test_perfmodel_allreduce_ring_pinned():
    """AR picks the ring at n = 1e7, p = 64 with the hand value."""
    g = GOLD["perfmodel_ar_ring"]
    t = pm.ar(g["p"], g["n"], g["alpha"], g["beta"], g["word_bytes"])
    assert abs(t - g["seconds"]) < 1e-12
    assert abs(t - g["seconds_ring"]) < 1e-12 and t < g["seconds_rd"]
    # p = 2: recursive doubling (alpha + n beta') beats the ring (2 alpha + n beta') -- SPEC.md:360
    assert abs(pm.ar(2, 1e6, 1e-6, 1e-9, 4) - (1e-6 + 4e-3)) < 1e-15


def test_perfmodel_layer_cost_pinned():
    """layer_cost's FP/BP composition against hand-priced values: P = 1 ->
    C + Cx + Cw; pure sample parallelism -> no halo, plus BPa
    (SPEC.md:368), with and without the R16 overlap; a 2-way H split adds
    2 SR(O N_l C W_l) to FP and the F-channel dy halo to BP (R13)."""
    g = GOLD["perfmodel_layer_cost"]
    cost = lambda op, *a: g["costs"][op]
    L, al, be = g["layer"], g["alpha"], g["beta"]
    for ov in (True, False):
        assert abs(pm.layer_cost(L, (1, 1, 1), cost, al, be, overlap=ov)["total"] - g["p1_total"]) < 1e-15
    s = pm.layer_cost(L, (4, 1, 1), cost, al, be, overlap=False)
    assert s["halo_x"] == 0.0 and s["halo_dy"] == 0.0
    assert abs(s["bpa"] - g["sample4_bpa"]) < 1e-15
    assert abs(s["total"] - g["sample4_total_plain"]) < 1e-15
    assert abs(pm.layer_cost(L, (4, 1, 1), cost, al, be, overlap=True)["total"] - g["sample4_total_overlap"]) < 1e-15
    sp = pm.layer_cost(L, (1, 2, 1), cost, al, be, overlap=False)
    assert abs(sp["halo_x"] - g["spatial2_halo_x"]) < 1e-15
    assert abs(sp["halo_dy"] - g["spatial2_halo_x"]) < 1e-15
    assert abs(sp["bpa"] - g["spatial2_bpa"]) < 1e-15
    assert abs(sp["total"] - g["spatial2_total_plain"]) < 1e-15
    # a 2-way W split of the square layer prices the same message through the
    # east/west branch, O N_l C H_l with H_l = 256 (W_l = 128 would differ)
    sw = pm.layer_cost(L, (1, 1, 2), cost, al, be, overlap=False)
    assert abs(sw["halo_x"] - g["spatial2_halo_x"]) < 1e-15
    assert abs(sw["total"] - g["spatial2_total_plain"]) < 1e-15
    # without the allreduce the plain total drops exactly BPa
    nar = pm.layer_cost(L, (1, 2, 1), cost, al, be, overlap=False, include_allreduce=False)
    assert abs(sp["total"] - nar["total"] - g["spatial2_bpa"]) < 1e-15


def _flops_cost(op, n, c, h, w, f, K=3):
    return 2.0 * n * c * h * w * f * K * K / 1e15


def test_perfmodel_structure():
    layer = dict(N=8, C=64, H=256, W=256, F=64, K=3, S=1, P=1)
    # undivided W removes e/w and corners; K=1 -> no halo
    assert pm.halo_terms(1, 64, 128, 256, 1, True, False, 1e-6, 1e-9, 2) == 2 * pm.sr(256 * 64, 1e-6, 1e-9, 2)
    assert pm.halo_terms(1, 64, 128, 256, 0, True, True, 1e-6, 1e-9, 2) == 0.0
    # sample-only FP <= spatial FP for the same local compute
    flat = lambda op, *a: 1e-3
    s = pm.layer_cost(layer, (4, 1, 1), flat, 1e-6, 1e-9, overlap=False)
    sp = pm.layer_cost(layer, (1, 4, 1), flat, 1e-6, 1e-9, overlap=False)
    assert s["fp"] <= sp["fp"]
    # argmin equals brute-force enumeration with the tie-break
    best = pm.choose(layer, 8, _flops_cost, 1e-6, 1e-9)
    allc = [(pm.layer_cost(layer, g, _flops_cost, 1e-6, 1e-9)["total"], g)
            for g in pm.candidates(8) if pm.valid(layer, g)]
    tmin = min(t for t, _ in allc)
    assert best[1] == tmin
    assert best[0] == max((g for t, g in allc if t == tmin), key=lambda g: (g[0], g[1], g[2]))


def test_validity_rejects_degenerate():
    # PAPER.md:145 spatial extent ~ kernel size; reading R22
    assert not pm.valid(dict(N=1, C=1, H=8, W=8, F=1, K=7, S=1, P=3), (1, 4, 1))
    assert pm.valid(dict(N=1, C=1, H=8, W=8, F=1, K=3, S=1, P=1), (1, 4, 1))
    assert not pm.valid(dict(N=2, C=1, H=8, W=8, F=1, K=3), (4, 1, 1))


# ---------------- generator ----------------

def test_generator_is_partition_independent_and_bf16_exact():
    full = datagen.gen_x(2, 3, 9, 7)
    blk = datagen.gen_x(2, 3, 9, 7, n=(1, 2), h=(3, 8), w=(2, 5))
    np.testing.assert_array_equal(blk, full[1:2, :, 3:8, 2:5])
    t = torch.tensor(full).to(torch.bfloat16).double().numpy()
    np.testing.assert_array_equal(t, full)
    w = datagen.gen_w(4, 3, 3)
    np.testing.assert_array_equal(torch.tensor(w).to(torch.bfloat16).double().numpy(), w)
    assert np.abs(full).max() <= 1.0 and len(np.unique(full)) > 100

"""GPU parity of the fp32 path (DC_FP32_3XTF32: fp32 activations and weights,
three tf32 tensor-core products per term, fp32 accumulation; reading R18,
PAPER.md:32 "single-precision") against the fp64 oracle, on fp32-exact
24-bit inputs (datagen kind "act24"; the oracle consumes the same numbers).

Tolerances:
  * north_star's fp32 bar on every output: max|g - o| / max|o| <= 1e-4;
  * element by element, the derived bound |g - o| <= (2^-20 + (n/8) 2^-24) S
    with S = the same sum over |operands| (the oracle run on |x|, |w|, |dy|)
    and n the terms per output (x3 for the three products): the split drops
    x_lo w_lo and truncates each lo to tf32 (<= 3 2^-22 |x w| per term), the
    fp32 accumulator adds one partial per K = 8 step.
Partitioned runs are bitwise equal to the 1-GPU fp32 result (north_star)."""
import numpy as np
import pytest
import torch

import datagen
import oracle

pytestmark = pytest.mark.gpu
TOL = 1e-4


@pytest.fixture(scope="module")
def dc():
    from paper_1903_06681_b200 import build
    build.build()
    import paper_1903_06681_b200 as dc
    torch.cuda.init()
    return dc


def inputs(shape):
    N, C, H, W, F, K, S, P = shape
    Ho, Wo = oracle.out_extent(H, K, S, P), oracle.out_extent(W, K, S, P)
    x = datagen.gen_x(N, C, H, W, kind="act24")
    w = datagen.gen_w(F, C, K, kind="act24")
    dy = datagen.gen_dy(N, F, Ho, Wo, kind="act24")
    return x, w, dy


def nhwc32(t):
    """fp64 NCHW -> dense NHWC fp32 device tensor (exact: 24-bit values)."""
    return torch.tensor(np.ascontiguousarray(t.transpose(0, 2, 3, 1)), dtype=torch.float32, device="cuda")


def full_split_buffer(dc, shape, tensor, glob):
    """The unpartitioned margined buffer of `tensor` (x or dy) filled by the
    library's import (the [hi | lo] split), for slicing shard windows."""
    N, C, H, W, F, K, S, P = shape
    plan = dc.dc_plan_create_virtual(N, C, H, W, F, K, S, P, (1, 1, 1), 0, dtype=dc.DC_FP32_3XTF32)
    try:
        d = dc.dc_plan_query(plan, tensor)
        buf = torch.zeros((d["n"], d["hb"], d["wb"], d["c_pad"]), dtype=torch.float32, device="cuda")
        dc.dc_tensor_import(plan, tensor, nhwc32(glob), buf)
        torch.cuda.synchronize()
        return buf
    finally:
        dc.dc_plan_destroy(plan)


def shard_of(full, d):
    """A shard's margined buffer = the global split buffer's window (data movement only)."""
    r0, c0 = d["h0"] - d["halo_n"], d["w0"] - d["halo_w"]
    return full[d["n0"]:d["n0"] + d["n"], r0:r0 + d["hb"], c0:c0 + d["wb"]].contiguous()


def weights32(w, cp):
    F, C, K, _ = w.shape
    out = np.zeros((F, K, K, cp))
    out[..., :C] = w.transpose(0, 2, 3, 1)
    return torch.tensor(out, dtype=torch.float32, device="cuda")


def run(dc, shape, grid=(1, 1, 1), rank=0, x=None, w=None, dy=None, fx=None, fdy=None):
    N, C, H, W, F, K, S, P = shape
    plan = dc.dc_plan_create_virtual(N, C, H, W, F, K, S, P, grid, rank, dtype=dc.DC_FP32_3XTF32)
    try:
        q = {t: dc.dc_plan_query(plan, t) for t in (dc.DC_X, dc.DC_Y, dc.DC_DY, dc.DC_DX, dc.DC_W)}
        xb, dyb = shard_of(fx, q[dc.DC_X]), shard_of(fdy, q[dc.DC_DY])
        wb = weights32(w, q[dc.DC_W]["c_pad"])
        yd, dxd = q[dc.DC_Y], q[dc.DC_DX]
        y = torch.full((yd["n"], yd["h"], yd["w"], yd["c_pad"]), float("nan"), device="cuda")
        dx = torch.full((dxd["n"], dxd["h"], dxd["w"], dxd["c_pad"]), float("nan"), device="cuda")
        dw = torch.full((F, K, K, C), float("nan"), device="cuda")
        dc.dc_conv_fwd(plan, xb, wb, y, 0)
        dc.dc_conv_bwd_data(plan, dyb, wb, dx, 0)
        dc.dc_conv_bwd_filter(plan, xb, dyb, dw, 0)
        torch.cuda.synchronize()
        return dict(y=y, dx=dx, dw=dw, q=q)
    finally:
        dc.dc_plan_destroy(plan)


def nchw(t, C):
    return t[..., :C].double().cpu().numpy().transpose(0, 3, 1, 2)


def check(name, got, ref, S, n):
    assert np.isfinite(got).all(), f"{name}: non-finite"
    err = np.abs(got - ref)
    rel = err.max() / max(np.abs(ref).max(), 1e-300)
    assert rel <= TOL, f"{name}: max rel err {rel:.3e} > {TOL}"
    bound = (2.0 ** -20 + (n / 8.0) * 2.0 ** -24) * S + 1e-30
    bad = err > bound
    assert not bad.any(), f"{name}: {bad.sum()} elements over the derived bound (worst {(err / bound).max():.2f}x)"
    return rel


SHAPES = [  # (N, C, H, W, F, K, S, P)
    (1, 2, 16, 16, 4, 3, 1, 1),        # C1 (BASELINE configs[0]): C, F padded to 8
    (2, 16, 20, 18, 32, 3, 1, 1),
    (1, 64, 24, 40, 64, 3, 1, 1),      # 64-channel groups (two 32-channel tf32 atoms in wgrad)
    (2, 32, 17, 23, 48, 3, 2, 1),      # stride 2, ragged, F = 48 (not a multiple of 32)
    (1, 3, 30, 30, 64, 7, 2, 3),       # conv1-like (C=3 -> 8, K=7 S=2)
    (2, 128, 14, 14, 256, 1, 1, 0),    # 1x1: wgrad M tiles of 4 channel groups
    (1, 18, 33, 35, 64, 3, 2, 1),      # mesh conv1_1-like (C = 18 -> 24)
    (1, 24, 19, 21, 16, 5, 1, 2),      # K=5
    (1, 64, 12, 12, 320, 3, 1, 1),     # F > 256: two N tiles
    (1, 512, 16, 18, 256, 3, 1, 1),    # deep layer: split-K
    (3, 16, 9, 9, 16, 3, 1, 0),        # P = 0
]


@pytest.mark.parametrize("shape", SHAPES)
def test_fp32_parity(dc, shape):
    """y (Eq. 1), dx (Eq. 3), dW (Eq. 2) of the 3xTF32 path vs the fp64 oracle,
    element by element and at north_star's 1e-4 bar."""
    N, C, H, W, F, K, S, P = shape
    x, w, dy = inputs(shape)
    fx, fdy = full_split_buffer(dc, shape, dc.DC_X, x), full_split_buffer(dc, shape, dc.DC_DY, dy)
    r = run(dc, shape, x=x, w=w, dy=dy, fx=fx, fdy=fdy)
    ax, aw, ady = np.abs(x), np.abs(w), np.abs(dy)
    check("y", nchw(r["y"], F), oracle.conv_fwd(x, w, S, P), oracle.conv_fwd(ax, aw, S, P), 3 * C * K * K)
    check("dx", nchw(r["dx"], C), oracle.conv_bwd_data(dy, w, H, W, S, P),
          oracle.conv_bwd_data(ady, aw, H, W, S, P), 3 * F * K * K)
    Ho, Wo = oracle.out_extent(H, K, S, P), oracle.out_extent(W, K, S, P)
    check("dw", r["dw"].double().cpu().numpy().transpose(0, 3, 1, 2), oracle.conv_bwd_filter(x, dy, K, S, P),
          oracle.conv_bwd_filter(ax, ady, K, S, P), 3 * N * Ho * Wo)
    # padded output channels are zeros
    assert float(r["y"][..., F:].abs().max()) == 0.0 if r["y"].shape[-1] > F else True
    assert float(r["dx"][..., C:].abs().max()) == 0.0 if r["dx"].shape[-1] > C else True


@pytest.mark.parametrize("shape", [SHAPES[0], SHAPES[2], SHAPES[3], SHAPES[4], SHAPES[6]])
@pytest.mark.parametrize("grid", [(1, 2, 1), (1, 1, 2), (1, 2, 2), (2, 2, 1)])
def test_fp32_partition_bitwise(dc, shape, grid):
    """Each rank's y and dx from its own margined fp32 shard are bitwise the
    1-GPU fp32 result; the per-rank dW sum matches within the fp32 bar."""
    N, C, H, W, F, K, S, P = shape
    try:
        dc.dc_plan_destroy(dc.dc_plan_create_virtual(N, C, H, W, F, K, S, P, grid, 0, dtype=dc.DC_FP32_3XTF32))
    except dc.DCError:
        pytest.skip("grid invalid for this shape")
    x, w, dy = inputs(shape)
    fx, fdy = full_split_buffer(dc, shape, dc.DC_X, x), full_split_buffer(dc, shape, dc.DC_DY, dy)
    full = run(dc, shape, x=x, w=w, dy=dy, fx=fx, fdy=fdy)
    dw_sum = torch.zeros_like(full["dw"])
    for rank in range(grid[0] * grid[1] * grid[2]):
        r = run(dc, shape, grid, rank, x=x, w=w, dy=dy, fx=fx, fdy=fdy)
        yd, dxd = r["q"][dc.DC_Y], r["q"][dc.DC_DX]
        ys = full["y"][yd["n0"]:yd["n0"] + yd["n"], yd["h0"]:yd["h0"] + yd["h"], yd["w0"]:yd["w0"] + yd["w"]]
        assert torch.equal(r["y"], ys), f"rank {rank}: y differs from 1 GPU"
        dxs = full["dx"][dxd["n0"]:dxd["n0"] + dxd["n"], dxd["h0"]:dxd["h0"] + dxd["h"],
                         dxd["w0"]:dxd["w0"] + dxd["w"]]
        assert torch.equal(r["dx"], dxs), f"rank {rank}: dx differs from 1 GPU"
        dw_sum += r["dw"]
    e = float((dw_sum - full["dw"]).abs().max() / full["dw"].abs().max())
    assert e <= TOL, e


def test_fp32_import_split_exact(dc):
    """dc_tensor_import of an fp32 tensor into an fp32 plan's margined buffer:
    hi + lo == x exactly, hi is a tf32 value (low 13 mantissa bits zero), the
    padded channels and the margins are zero."""
    N, C, H, W, F, K, S, P = 2, 18, 12, 10, 8, 3, 1, 1
    x = datagen.gen_x(N, C, H, W, kind="act24")
    plan = dc.dc_plan_create_virtual(N, C, H, W, F, K, S, P, (1, 2, 1), 1, dtype=dc.DC_FP32_3XTF32)
    try:
        d = dc.dc_plan_query(plan, dc.DC_X)
        buf = torch.zeros((d["n"], d["hb"], d["wb"], d["c_pad"]), dtype=torch.float32, device="cuda")
        own = x[:, :, d["h0"]:d["h0"] + d["h"], d["w0"]:d["w0"] + d["w"]]
        dc.dc_tensor_import(plan, dc.DC_X, nhwc32(own), buf)
        torch.cuda.synchronize()
        cp = d["c_pad"] // 2
        hi, lo = buf[..., :cp].double(), buf[..., cp:].double()
        blk = slice(d["halo_n"], d["halo_n"] + d["h"])
        assert torch.equal((hi + lo)[:, blk, :, :C].cpu(), torch.tensor(own.transpose(0, 2, 3, 1)))
        assert int((buf[..., :cp].view(torch.int32) & 0x1FFF).abs().max()) == 0
        assert float(buf[:, :d["halo_n"]].abs().max()) == 0.0 and float(buf[..., C:cp].abs().max()) == 0.0
    finally:
        dc.dc_plan_destroy(plan)


def test_fp32_bn_stats(dc):
    """Spatial BN statistics of an fp32 y (fp64 accumulation) vs the oracle."""
    N, C, H, W, F, K, S, P = 2, 8, 20, 24, 48, 3, 1, 1
    plan = dc.dc_plan_create_virtual(N, C, H, W, F, K, S, P, (1, 1, 1), 0, dtype=dc.DC_FP32_3XTF32)
    try:
        t = datagen.gen_block((N, F, H, W), 7, 9, kind="act24")
        cp = dc.dc_plan_query(plan, dc.DC_Y)["c_pad"]
        tt = torch.zeros((N, H, W, cp), dtype=torch.float32, device="cuda")
        tt[..., :F] = nhwc32(t)
        mean = torch.zeros(F, dtype=torch.float64, device="cuda")
        var = torch.zeros(F, dtype=torch.float64, device="cuda")
        dc.dc_bn_spatial_stats(plan, tt, mean, var, dc.DC_BN_LOCAL)
        torch.cuda.synchronize()
        m_ref, v_ref = oracle.bn_stats(t)
        np.testing.assert_allclose(mean.cpu().numpy(), m_ref, rtol=0, atol=1e-12)
        np.testing.assert_allclose(var.cpu().numpy(), v_ref, rtol=0, atol=1e-12)
    finally:
        dc.dc_plan_destroy(plan)

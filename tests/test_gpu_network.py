"""GPU parity of the NEXT-1 layers: batch-norm apply with
the spatially aggregated statistics (+ residual, ReLU) written into the next
layer's margined input, and its backward with the group sums (PAPER.md:149,
234-236), against oracle/network.py (fp64) on the same bf16-exact inputs --
on one GPU and on loopback ranks of 2x2 / hybrid grids.

Tolerances: apply -- the fp32 evaluation a y + b (+ r) is
within 4 u (|a y| + |b| + |r|) of the exact value, then the bf16 store adds
2^-8 |out|; backward -- dy = k (g - m1 - y_hat m2) evaluated in fp32 from
fp64 group sums: within 8 u |k| (|g| + |m1| + |y_hat| |m2|) + 2^-8 |dy|;
dgamma, dbeta (fp32 sums of <= 4 pixels, then fp64): within 6 u sum |g y_hat|,
5 u sum |g| (u = 2^-24)."""
import numpy as np
import pytest
import torch

import datagen
import oracle
from oracle import network as net
from tests.gpu_util import fill_buffer

pytestmark = pytest.mark.gpu
U = 2.0 ** -24


@pytest.fixture(scope="module")
def dc():
    from paper_1903_06681_b200 import build
    build.build()
    import paper_1903_06681_b200 as dc
    torch.cuda.init()
    return dc


def nhwc(t, cp, dtype=torch.bfloat16):
    """fp64 NCHW -> dense NHWC device tensor with channels padded to cp."""
    N, C, H, W = t.shape
    out = np.zeros((N, H, W, cp))
    out[..., :C] = t.transpose(0, 2, 3, 1)
    return torch.tensor(out, dtype=dtype, device="cuda")


def nchw(t, C):
    return t[..., :C].double().cpu().numpy().transpose(0, 3, 1, 2)


def params(F):
    g = datagen.gen_block((1, F, 1, 1), 5, 11).ravel() + 1.25   # bf16-exact, positive and negative scales
    b = datagen.gen_block((1, F, 1, 1), 5, 12).ravel() * 0.5
    return g, b


CASES = [  # layer (N, C, H, W, F, K, S, P) whose output is normalised; grid
    ((2, 16, 24, 20, 32, 3, 1, 1), (1, 1, 1)),
    ((1, 64, 33, 30, 64, 3, 1, 1), (1, 1, 1)),
    ((2, 16, 24, 20, 48, 3, 1, 1), (1, 2, 2)),
    ((4, 16, 18, 20, 32, 3, 1, 1), (2, 2, 1)),
    ((1, 32, 40, 24, 64, 3, 1, 1), (1, 4, 1)),
]


def stats_of(dc, plan, y, F, stream=None):
    mean = torch.zeros(F, dtype=torch.float64, device="cuda")
    var = torch.zeros(F, dtype=torch.float64, device="cuda")
    dc.dc_bn_spatial_stats(plan, y, mean, var, 0, stream)
    return mean, var


def check_apply(got, y, m, v, g, b, res, relu, store=2.0 ** -8):
    ref = net.bn_relu_forward(y, m, v, g, b, 1e-5, residual=res, relu=relu)
    a = g / np.sqrt(v + 1e-5)
    mag = np.abs(a[None, :, None, None] * y) + np.abs((b - a * m))[None, :, None, None]
    if res is not None:
        mag = mag + np.abs(res)
    bound = 4 * U * mag + store * np.abs(ref) + 1e-30
    err = np.abs(got - ref)
    assert (err <= bound).all(), f"BN apply: {(err > bound).sum()} elements over bound (worst {(err / bound).max():.2f}x)"


def check_backward(got_dy, got_dg, got_db, dout, y, m, v, g, b, res, relu, store=2.0 ** -8):
    dy, dgam, dbet, gm = net.bn_relu_backward(dout, y, m, v, g, b, 1e-5, residual=res, relu=relu)
    M = y.shape[0] * y.shape[2] * y.shape[3]
    k = g / np.sqrt(v + 1e-5)
    yh = (y - m[None, :, None, None]) / np.sqrt(v + 1e-5)[None, :, None, None]
    mag = np.abs(k)[None, :, None, None] * (np.abs(gm) + np.abs(dbet / M)[None, :, None, None]
                                            + np.abs(yh) * np.abs(dgam / M)[None, :, None, None])
    bound = 8 * U * mag + store * np.abs(dy) + 1e-30
    err = np.abs(got_dy - dy)
    assert (err <= bound).all(), f"BN bwd dy: {(err > bound).sum()} over bound (worst {(err / bound).max():.2f}x)"
    # per-thread fp32 sums over a trip of <= 4 pixels (4 fused adds), then fp64
    # (DESIGN.md §7): <= 4 u sum|term|, plus the final fp32 rounding of the sum
    tg = 6 * U * np.abs(gm * yh).sum(axis=(0, 2, 3)) + 1e-12
    tb = 5 * U * np.abs(gm).sum(axis=(0, 2, 3)) + 1e-12
    assert (np.abs(got_dg - dgam) <= tg).all(), "dgamma"
    assert (np.abs(got_db - dbet) <= tb).all(), "dbeta"


# many chunks per block (the staged kernels' ring of stages wraps, ragged last chunk)
BIG = ((2, 16, 256, 250, 64, 3, 1, 1), (1, 1, 1))


@pytest.mark.parametrize("relu,use_res", [(True, False), (True, True), (False, False)])
@pytest.mark.parametrize("case", CASES[:2] + [BIG])
def test_bn_apply_backward_one_gpu(dc, case, relu, use_res):
    (N, C, H, W, F, K, S, P), _ = case
    Ho, Wo = oracle.out_extent(H, K, S, P), oracle.out_extent(W, K, S, P)
    plan = dc.dc_plan_create(N, C, H, W, F, K, S, P, (1, 1, 1), dc.DC_BF16, None)
    nxt = dc.dc_plan_create(N, F, Ho, Wo, 16, 3, 1, 1, (1, 1, 1), dc.DC_BF16, None)
    try:
        yd, dyd = dc.dc_plan_query(plan, dc.DC_Y), dc.dc_plan_query(plan, dc.DC_DY)
        cp = yd["c_pad"]
        y = datagen.gen_block((N, F, Ho, Wo), 21, 1)
        res = datagen.gen_block((N, F, Ho, Wo), 21, 2) if use_res else None
        dout = datagen.gen_block((N, F, Ho, Wo), 21, 3)
        g, b = params(F)
        yt = nhwc(y, cp)
        rt = nhwc(res, cp) if use_res else None
        mean, var = stats_of(dc, plan, yt, F)
        gt, bt = torch.tensor(g, dtype=torch.float32, device="cuda"), torch.tensor(b, dtype=torch.float32, device="cuda")
        flags = dc.DC_RELU if relu else 0
        out = torch.full_like(yt, float("nan"))
        dc.dc_bn_apply(plan, yt, mean, var, gt, bt, 1e-5, rt, flags, None, out)
        # straight into the next layer's margined input: the same values in its owned block
        xd = dc.dc_plan_query(nxt, dc.DC_X)
        xb = torch.zeros((xd["n"], xd["hb"], xd["wb"], xd["c_pad"]), dtype=torch.bfloat16, device="cuda")
        dc.dc_bn_apply(plan, yt, mean, var, gt, bt, 1e-5, rt, flags, nxt, xb)
        dyb = torch.full((dyd["n"], dyd["hb"], dyd["wb"], dyd["c_pad"]), float("nan"), dtype=torch.bfloat16,
                         device="cuda")
        dg = torch.zeros(F, device="cuda")
        db = torch.zeros(F, device="cuda")
        dres = torch.zeros_like(yt) if use_res else None
        dc.dc_bn_backward(plan, nhwc(dout, cp), yt, mean, var, gt, bt, dyb, 1e-5, rt, flags, dg, db, dres)
        torch.cuda.synchronize()
        m, v = oracle.bn_stats(y)
        check_apply(nchw(out, F), y, m, v, g, b, res, relu)
        own = xb[:, xd["halo_n"]:xd["halo_n"] + xd["h"], xd["halo_w"]:xd["halo_w"] + xd["w"]]
        assert torch.equal(own, out), "dc_bn_apply into the next plan's margins differs from the dense result"
        ow = dyb[:, dyd["halo_n"]:dyd["halo_n"] + dyd["h"], dyd["halo_w"]:dyd["halo_w"] + dyd["w"]]
        check_backward(nchw(ow, F), dg.double().cpu().numpy(), db.double().cpu().numpy(), dout, y, m, v, g, b,
                       res, relu)
        if use_res:
            gm = net.bn_relu_backward(dout, y, m, v, g, b, 1e-5, residual=res, relu=relu)[3]
            assert np.array_equal(nchw(dres, F), gm), "dresidual = the ReLU-masked gradient (exact)"
    finally:
        dc.dc_plan_destroy(nxt)
        dc.dc_plan_destroy(plan)


@pytest.mark.parametrize("relu,use_res", [(True, True), (False, False)])
def test_bn_fp32_split(dc, relu, use_res):
    """fp32 plans (DC_FP32_3XTF32): BN apply / backward evaluate in fp32 and
    store the [hi | lo] halves into the next layer's margined input / this
    layer's margined dy; hi is tf32 and hi + lo the fp32 value (no bf16
    rounding: the bounds without the store term)."""
    N, C, H, W, F = 2, 16, 21, 19, 40
    plan = dc.dc_plan_create(N, C, H, W, F, 3, 1, 1, (1, 1, 1), dc.DC_FP32_3XTF32, None)
    nxt = dc.dc_plan_create(N, F, H, W, 16, 3, 1, 1, (1, 1, 1), dc.DC_FP32_3XTF32, None)
    try:
        yd, dyd, xd = dc.dc_plan_query(plan, dc.DC_Y), dc.dc_plan_query(plan, dc.DC_DY), dc.dc_plan_query(nxt, dc.DC_X)
        cp = yd["c_pad"]
        y = datagen.gen_block((N, F, H, W), 23, 1)
        res = datagen.gen_block((N, F, H, W), 23, 2) if use_res else None
        dout = datagen.gen_block((N, F, H, W), 23, 3)
        g, b = params(F)
        yt = nhwc(y, cp, torch.float32)
        rt = nhwc(res, cp, torch.float32) if use_res else None
        mean, var = stats_of(dc, plan, yt, F)
        gt, bt = torch.tensor(g, dtype=torch.float32, device="cuda"), torch.tensor(b, dtype=torch.float32, device="cuda")
        flags = dc.DC_RELU if relu else 0
        xb = torch.full((xd["n"], xd["hb"], xd["wb"], xd["c_pad"]), float("nan"), device="cuda")
        dc.dc_bn_apply(plan, yt, mean, var, gt, bt, 1e-5, rt, flags, nxt, xb)
        dyb = torch.full((dyd["n"], dyd["hb"], dyd["wb"], dyd["c_pad"]), float("nan"), device="cuda")
        dg, db = torch.zeros(F, device="cuda"), torch.zeros(F, device="cuda")
        dres = torch.zeros_like(yt) if use_res else None
        dc.dc_bn_backward(plan, nhwc(dout, cp, torch.float32), yt, mean, var, gt, bt, dyb, 1e-5, rt, flags, dg, db,
                          dres)
        torch.cuda.synchronize()

        def owned(buf, d):
            o = buf[:, d["halo_n"]:d["halo_n"] + d["h"], d["halo_w"]:d["halo_w"] + d["w"]]
            half = d["c_pad"] // 2
            hi, lo = o[..., :half], o[..., half:]
            assert (hi.view(torch.int32) & 0x1FFF == 0).all(), "hi half is not tf32"
            return hi + lo  # exact: lo = v - hi

        m, v = oracle.bn_stats(y)
        check_apply(nchw(owned(xb, xd), F), y, m, v, g, b, res, relu, store=U)
        check_backward(nchw(owned(dyb, dyd), F), dg.double().cpu().numpy(), db.double().cpu().numpy(), dout, y, m, v,
                       g, b, res, relu, store=U)
        if use_res:
            gm = net.bn_relu_backward(dout, y, m, v, g, b, 1e-5, residual=res, relu=relu)[3]
            assert np.array_equal(nchw(dres, F), gm), "dresidual = the ReLU-masked gradient (exact)"
    finally:
        dc.dc_plan_destroy(nxt)
        dc.dc_plan_destroy(plan)


@pytest.mark.parametrize("case", CASES[2:])
def test_bn_backward_spatial_group(dc, case):
    """Loopback ranks: each rank's dy from its shard with the GROUP sums
     matches the unpartitioned oracle; the mailbox
    sum runs once for the statistics and once for the backward sums."""
    (N, C, H, W, F, K, S, P), grid = case
    Ho, Wo = oracle.out_extent(H, K, S, P), oracle.out_extent(W, K, S, P)
    world = grid[0] * grid[1] * grid[2]
    y = datagen.gen_block((N, F, Ho, Wo), 22, 1)
    dout = datagen.gen_block((N, F, Ho, Wo), 22, 3)
    g, b = params(F)
    comms = dc.dc_comm_create_local(world, torch.cuda.current_device())
    R = []
    try:
        for r in range(world):
            plan = dc.dc_plan_create(N, C, H, W, F, K, S, P, grid, dc.DC_BF16, comms[r])
            yd, dyd = dc.dc_plan_query(plan, dc.DC_Y), dc.dc_plan_query(plan, dc.DC_DY)
            dyb = dc.wrap_device_buffer(dc.dc_buffer_alloc(plan, dc.DC_DY),
                                        (dyd["n"], dyd["hb"], dyd["wb"], dyd["c_pad"]))
            R.append(dict(plan=plan, yd=yd, dyd=dyd, dyb=dyb, s=torch.cuda.ExternalStream(dc.dc_comm_stream(comms[r])),
                          y=fill_buffer(y, yd), dout=fill_buffer(dout, yd),
                          mean=torch.zeros(F, dtype=torch.float64, device="cuda"),
                          var=torch.zeros(F, dtype=torch.float64, device="cuda"),
                          dg=torch.zeros(F, device="cuda"), db=torch.zeros(F, device="cuda")))
        gt, bt = torch.tensor(g, dtype=torch.float32, device="cuda"), torch.tensor(b, dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        for d in R:
            with torch.cuda.stream(d["s"]):
                dc.dc_bn_spatial_stats(d["plan"], d["y"], d["mean"], d["var"], 0, d["s"])
                dc.dc_bn_backward(d["plan"], d["dout"], d["y"], d["mean"], d["var"], gt, bt, d["dyb"], 1e-5, None,
                                  dc.DC_RELU, d["dg"], d["db"], None, d["s"])
        torch.cuda.synchronize()
        for r, d in enumerate(R):
            yd, dyd = d["yd"], d["dyd"]
            n0, n1 = yd["n0"], yd["n0"] + yd["n"]
            ys = y[n0:n1]                                    # the BN group: this rank's samples, whole space
            m, v = oracle.bn_stats(ys)
            dy_ref = net.bn_relu_backward(dout[n0:n1], ys, m, v, g, b)[0]
            blk = dy_ref[:, :, yd["h0"]:yd["h0"] + yd["h"], yd["w0"]:yd["w0"] + yd["w"]]
            got = nchw(d["dyb"][:, dyd["halo_n"]:dyd["halo_n"] + dyd["h"], dyd["halo_w"]:dyd["halo_w"] + dyd["w"]], F)
            err = np.abs(got - blk)
            assert (err <= 2.0 ** -8 * np.abs(blk) + 1e-4 * np.abs(blk).max() + 1e-30).all(), \
                f"rank {r}: dy (max err {err.max():.3e})"
            _, dgam, dbet, _ = net.bn_relu_backward(dout[n0:n1], ys, m, v, g, b)
            np.testing.assert_allclose(d["dg"].double().cpu().numpy(), dgam, rtol=1e-5, atol=1e-5)
            np.testing.assert_allclose(d["db"].double().cpu().numpy(), dbet, rtol=1e-5, atol=1e-5)
    finally:
        for d in R:
            dc.dc_plan_destroy(d["plan"])
        for c in comms:
            dc.dc_comm_destroy(c)
